"""Summarise an ncu --set full report (+ optional launch-list CSV) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_trace.ncu-rep gpurun_out/launches.csv profiles/r02_xxx \
        [--bench BUILD_ID_FILE]

--bench also writes profiles/ncu_summary.json, the pointer bench.py reads: the
first k_trace_packet launch's DRAM / L2 bytes and warp instructions, stamped
with the srt_build_id of the profiled library (tools/profile_trace.py writes it).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "l1tex__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__sass_average_branch_targets_threads_uniform.pct", "lts__t_sectors.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for i, name in enumerate(h):
            if name in KEYS or name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                d[name] = (v[i], u[i])
        kernels.append(d)
    return kernels


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[start + 1:]:
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(float(r[vi]))
    total = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "total_ns": sum(v), "share": sum(v) / total} for k, v in
            sorted(agg.items(), key=lambda kv: -sum(kv[1]))}


def main():
    rep, lcsv, outdir = sys.argv[1], sys.argv[2], Path(sys.argv[3])
    outdir.mkdir(parents=True, exist_ok=True)
    summary = {"full": raw(rep)}
    # achieved bandwidths of each profiled launch (DRAM, L2 = 32-B sectors)
    for k in summary["full"]:
        try:
            ms = float(k["gpu__time_duration.sum"][0]) * (1e-3 if k["gpu__time_duration.sum"][1] == "us" else 1.0)
            unit = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
            dr = sum(float(k[m][0]) * unit[k[m][1]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            l2 = float(k["lts__t_sectors.sum"][0]) * 32 / 1e6
            k["derived.dram_GBps"] = (f"{dr / ms:.1f}", "GB/s")
            k["derived.l2_GBps"] = (f"{l2 / ms:.1f}", "GB/s")
            k["derived.l2_bytes_per_launch"] = (f"{l2:.1f}", "Mbyte")
        except (KeyError, ValueError):
            pass
    if lcsv != "-":
        summary["launch_list"] = launches(lcsv)
    (outdir / "ncu_summary.json").write_text(json.dumps(summary, indent=1))
    lines = []
    for k in summary["full"]:
        lines.append(f"== {k['kernel'][:100]}")
        for name, (val, unit) in sorted((n, v) for n, v in k.items() if n != "kernel"):
            lines.append(f"  {name:75s} {val:>16s} {unit}")
    if "launch_list" in summary:
        lines.append("== launch list (ncu --metrics gpu__time_duration.sum, cold, serialised)")
        for name, d in summary["launch_list"].items():
            lines.append(f"  {name[:70]:70s} n={d['launches']:3d} total={d['total_ns']/1e3:10.1f} us share={d['share']:.3f}")
    (outdir / "ncu_summary.txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    if "--bench" in sys.argv:
        bid = Path(sys.argv[sys.argv.index("--bench") + 1]).read_text().strip()
        k = next(x for x in summary["full"] if "k_trace_packet" in x["kernel"])
        unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def val(m):
            return float(k[m][0]) * unit.get(k[m][1], 1.0)

        pointer = {
            "kernel": k["kernel"],
            "source": f"{outdir}/ncu_summary.json (ncu --set full --clock-control none, one launch of "
                      f"tools/profile_trace.py: C3-target 1080p, 2,073,600 walks)",
            "build_id": bid,
            "walks_per_launch": 2073600,
            "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "dram_read_bytes": val("dram__bytes_read.sum"),
            "dram_write_bytes": val("dram__bytes_write.sum"),
            "l2_bytes_per_launch": float(k["lts__t_sectors.sum"][0]) * 32,
            "warp_inst_per_launch": float(k["smsp__inst_executed.sum"][0]),
            "issue_active_pct": float(k["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
            "kernel_ms_ncu": float(k["gpu__time_duration.sum"][0]) * (1e-3 if k["gpu__time_duration.sum"][1] == "us"
                                                                       else 1.0),
        }
        (Path(__file__).resolve().parent.parent / "profiles" / "ncu_summary.json").write_text(
            json.dumps(pointer, indent=1) + "\n")


if __name__ == "__main__":
    main()
