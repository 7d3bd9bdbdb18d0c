"""Per-source-line stall samples from an ncu report (cuda,sass view).
Usage: python profiles/ncu_lines.py report.ncu-rep [topN]"""
import csv
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cur, hdr, agg = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].strip():
        continue
    try:
        s = int(r[4] or 0)
        ex = int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    agg.append((s, ex, cur, int(r[0]), r[1]))
tot = sum(a[0] for a in agg) or 1
src_cache = {}


def text(path, line, fallback):
    base = os.path.basename(path)
    local = os.path.join(here, "paper_2601_22074_b200", "csrc", base)
    if fallback.strip():
        return fallback.strip()
    if os.path.exists(local):
        lines = src_cache.setdefault(local, open(local).read().splitlines())
        return lines[line - 1].strip() if line - 1 < len(lines) else ""
    return ""


print(f"total samples {tot}")
for s, ex, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{s:5d} {100 * s / tot:5.1f}%  ex={ex:8d}  {os.path.basename(f)}:{ln}  {text(f, ln, src)[:90]}")
