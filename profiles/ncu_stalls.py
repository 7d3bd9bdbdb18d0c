"""Stall-reason totals of an ncu report, overall and per source line.
Usage: python profiles/ncu_stalls.py report.ncu-rep [topN]"""
import collections
import csv
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if r and r[0] == "Line No")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
per_line = collections.defaultdict(collections.Counter)
src = {}
cur = line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = os.path.basename(r[1])
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:
        line = (cur, int(r[0]))
        src[line] = r[1].strip()[:70]
        continue
    if len(r) > max(cols) and r[2].startswith("0x"):
        for i in cols:
            v = int(r[i] or 0)
            tot[hdr[i]] += v
            per_line[line][hdr[i]] += v
T = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common(10)))
lines = sorted(per_line.items(), key=lambda kv: -sum(kv[1].values()))[:top]
for (f, ln), c in lines:
    s = sum(c.values())
    reasons = " ".join(f"{k[6:]}={v}" for k, v in c.most_common(3))
    print(f"{s:6d} {100 * s / T:4.1f}% {f}:{ln:<5d} [{reasons}]  {src.get((f, ln), '')}")
