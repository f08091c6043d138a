"""Per-source-line instruction counts and stall samples from an ncu report
(--page source --print-source cuda,sass).  usage: ncu_lines.py rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:  # a source line row with aggregated metrics
        try:
            ie = float(r[hdr.index("Instructions Executed")] or 0)
            te = float(r[hdr.index("Thread Instructions Executed")] or 0)
            sm = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        key = (fname, int(r[0]), r[1].strip()[:80])
        a = agg.setdefault(key, [0, 0, 0])
        a[0] += ie; a[1] += te; a[2] += sm
ti = sum(v[0] for v in agg.values()); ts = sum(v[2] for v in agg.values())
print(f"total warp inst {ti/1e6:.1f}M  samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{k[0][:14]:14s}:{k[1]:4d} samp {v[2]/ts*100:5.1f}% inst {v[0]/ti*100:5.1f}% thr/inst {v[1]/max(v[0],1):5.1f} | {k[2]}")
