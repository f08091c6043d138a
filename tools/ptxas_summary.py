"""Registers / spills per kernel from `nvcc -Xptxas -v` output (stdin):
    nvcc ... -Xptxas -v -c trace.cu 2>&1 | python tools/ptxas_summary.py [name-filter]"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    if flt in d:
        print(f"{rows[n].get('regs', '?'):>4} regs  spill {rows[n].get('spill', '?'):>9}  {d[:150]}")
