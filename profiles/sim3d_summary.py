"""Summarise an ncu --set full capture of the 3-D env kernel into markdown.

    python profiles/sim3d_summary.py report.ncu-rep "title" > profiles/<round>_sim3d_env_kernel_<dtype>.md
"""
import csv
import re
import subprocess
import sys
from collections import Counter

rep, title = sys.argv[1], sys.argv[2]


def page(name, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout


det = list(csv.reader(page("details").splitlines()))
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Instructions", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Memory Throughput", "Compute (SM) Throughput"]
vals = {}
dh = det[0]
ni, ui, vi = dh.index("Metric Name"), dh.index("Metric Unit"), dh.index("Metric Value")
for r in det[1:]:
    if len(r) > vi and r[ni] in want and r[ni] not in vals:
        vals[r[ni]] = f"{r[vi]} {r[ui]}".strip()
src = list(csv.reader(page("source", ["--print-source", "cuda,sass"]).splitlines()))
lines, hdr, cur = [], None, None
stall_tot = Counter()
for r in src:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            e = int(r[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        code = r[hdr.index("Source")].strip() if "Source" in hdr else ""
        lines.append((s, e, cur.split("/")[-1] if cur else "?", int(r[0]), code))
        for i, c in enumerate(hdr):
            if c.startswith("stall_") and "Not Issued" not in c and i < len(r) and r[i]:
                try:
                    stall_tot[c] += int(r[i])
                except ValueError:
                    pass
tot = sum(x[0] for x in lines) or 1
print(f"# {title}\n")
print("| metric | value |\n|---|---|")
for k in want:
    if k in vals:
        print(f"| {k} | {vals[k]} |")
st = sum(stall_tot.values()) or 1
print("\n**Warp stall reasons** (share of samples): " +
      ", ".join(f"{k.replace('stall_', '')} {v / st * 100:.1f}%" for k, v in stall_tot.most_common(8)))
print("\n**Top source lines by stall samples**\n\n| samples | % | instructions | line | source |\n|---|---|---|---|---|")
for s, e, f, ln, code in sorted(lines, reverse=True)[:25]:
    code = re.sub(r"\|", "\\|", code)[:90]
    print(f"| {s} | {s / tot * 100:.1f} | {e} | {f}:{ln} | `{code}` |")
