"""Aggregate an ncu source-page capture of csrc/s3_kernel.cu by enclosing device function.

    python profiles/ncu_by_function.py report.ncu-rep
"""
import csv
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
src_path = "paper_2601_22074_b200/csrc/s3_kernel.cu"
lines_src = open(src_path).read().split("\n")
owner, name = {}, "?"
for i, l in enumerate(lines_src, 1):
    m = re.match(r"(?:template <class T>\s*)?(?:__global__|__device__)[^(]*?\b(\w+)\(", l)
    if m and not l.startswith(" "):
        name = m.group(1)
    owner[i] = name
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, cur = None, None
samp, inst = Counter(), Counter()
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur and cur.endswith("s3_kernel.cu") and r and r[0].isdigit():
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            e = int(r[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        f = owner.get(int(r[0]), "?")
        samp[f] += s
        inst[f] += e
tot = sum(samp.values()) or 1
for f, v in samp.most_common(30):
    print(f"{v / tot * 100:5.1f}%  inst {inst[f] / 1e6:8.1f}M  {f}")
