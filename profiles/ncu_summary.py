"""Markdown summary of one ncu --set full capture (key metrics + stall mix).
Usage: python profiles/ncu_summary.py report.ncu-rep "title" [alg_bytes_per_launch]"""
import csv
import os
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
here = os.path.dirname(os.path.abspath(__file__))
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(out.splitlines()))
hh = rr[0]
mi, vi, ui = hh.index("Metric Name"), hh.index("Metric Value"), hh.index("Metric Unit")
want = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Grid Size", "Block Size"]
vals = {}
for r in rr[1:]:
    if len(r) > ui and r[mi] in want and r[mi] not in vals:
        vals[r[mi]] = f"{r[vi]} {r[ui]}".strip()
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rh, units, rv = (list(csv.reader([raw[i]]))[0] for i in (0, 1, 2))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
dram = sum(float(rv[rh.index(m)].replace(",", "")) * scale.get(units[rh.index(m)], 1)
           for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
lines = [f"# {title}", "", "| metric | value |", "|---|---|"]
lines += [f"| {k} | {vals[k]} |" for k in want if k in vals]
lines.append(f"| dram bytes read+write | {dram:,.0f} B |")
if alg:
    lines.append(f"| algorithmic bytes (traffic.py) | {alg:,.0f} B |")
st = subprocess.run([sys.executable, os.path.join(here, "ncu_stalls.py"), rep, "12"], capture_output=True, text=True).stdout
lines += ["", "Warp-state samples (`profiles/ncu_stalls.py`):", "", "```", st.rstrip(), "```"]
print("\n".join(lines))
