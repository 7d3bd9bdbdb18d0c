"""Summarize an ncu --set full report: stall reasons by SASS opcode class and
top instructions. Usage: python profiles/ncu_summarize.py report.ncu-rep"""
import csv
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si = h.index("Source")
ns = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
by_op = defaultdict(Counter)
samples_by_op = Counter()
insts = []
for r in rows[1:]:
    if len(r) <= ns:
        continue
    sass = r[si].strip()
    op = sass.split()[0] if sass else "?"
    if op.startswith("@"):
        op = sass.split()[1]
    op = op.split(".")[0]
    s = int(r[ns] or 0)
    samples_by_op[op] += s
    for i in stall_cols:
        v = int(r[i] or 0)
        tot[h[i]] += v
        by_op[op][h[i]] += v
    insts.append((s, sass, int(r[ex] or 0)))
all_s = sum(samples_by_op.values())
print(f"total samples {all_s}")
print("stall reasons:", ", ".join(f"{k[6:]}={100*v/all_s:.1f}%" for k, v in tot.most_common(8)))
print("samples by opcode:")
for op, v in samples_by_op.most_common(15):
    top = ", ".join(f"{k[6:]}:{c}" for k, c in by_op[op].most_common(3))
    print(f"  {op:10s} {100*v/all_s:5.1f}%  ({top})")
n_exec = Counter()
for s, sass, e in insts:
    op = sass.split()[0]
    if op.startswith("@"):
        op = sass.split()[1]
    n_exec[op.split(".")[0]] += e
print("executed warp-instructions by opcode:", ", ".join(f"{k}={v}" for k, v in n_exec.most_common(14)))
print("top instructions by samples:")
for s, sass, e in sorted(insts, reverse=True)[:25]:
    print(f"  {s:6d} {sass[:90]}")
