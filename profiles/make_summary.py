"""Turn gpurun_out/ ncu artifacts into committed profile summaries.

    python profiles/make_summary.py <round> <launches.csv> <full.ncu-rep> <envs> [alg_bytes_per_world]

Writes profiles/<round>_launches.md (per-kernel launch list stats),
profiles/<round>_step_kernel.md (full-set summary of the fused step kernel)
and profiles/ncu_step_kernel.json (dram bytes per launch, read by bench.py).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

rnd, launches, rep, envs = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
alg = int(sys.argv[5]) if len(sys.argv) > 5 else 2197
here = os.path.dirname(os.path.abspath(__file__))

rows = list(csv.reader(open(launches)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)  # -> us
        agg[r[ki].split("(")[0][:70]].append(v)
lines = [f"# {rnd}: launch list of `python bench.py --steps 10 --warmup 3 --no-cpu --scale-envs 0 --no-e2e` (N=4096)",
         "", "ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares).", "",
         "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {100*sum(v)/tot:.1f} % |")
ours = {k: v for k, v in agg.items() if k.startswith(("ss_step", "rng_draw", "ss::", "randomize", "heights", "fk_"))}
t_ours = sum(sum(v) for v in ours.values())
lines += ["", f"Own kernels: {t_ours:.1f} us of {tot:.1f} us total; the rest is the bench's 512 MiB L2-flush "
          "fills before every timed step and torch fills/indexing at env setup and reset."]
open(os.path.join(here, f"{rnd}_launches.md"), "w").write("\n".join(lines) + "\n")

out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(out.splitlines()))
hh = rr[0]
si, mi, vi2, ui2 = hh.index("Section Name"), hh.index("Metric Name"), hh.index("Metric Value"), hh.index("Metric Unit")
want = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Ipc Active", "Executed Instructions", "Registers Per Thread", "Stack Size",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
        "Avg. Not Predicated Off Threads Per Warp", "Grid Size", "Block Size"]
vals = {}
for r in rr[1:]:
    if len(r) > ui2 and r[mi] in want and r[mi] not in vals:
        vals[r[mi]] = (r[vi2], r[ui2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rh = list(csv.reader(raw[:1]))[0]
rv = list(csv.reader(raw[2:3]))[0] if len(raw) > 2 else []
units = list(csv.reader(raw[1:2]))[0] if len(raw) > 1 else []
def rawv(name):
    i = rh.index(name)
    v = float(rv[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024**2}.get(u, 1)
    return v * scale
dram = rawv("dram__bytes_read.sum") + rawv("dram__bytes_write.sum")
dur = rawv("gpu__time_duration.sum")  # ncu reports usecond here
md = [f"# {rnd}: fused step kernel (`ss_step_jit`), ncu --set full", "",
      f"Captured on a timed step of `bench.py` (Velocity-Rough, N={envs}, L2 flushed before the step).", "",
      "| metric | value |", "|---|---|"]
for k in want:
    if k in vals:
        md.append(f"| {k} | {vals[k][0]} {vals[k][1]} |")
md.append(f"| dram bytes read+write | {dram:.0f} B ({dram/envs:.0f} B per world) |")
md.append(f"| algorithmic bytes (traffic.py) | {alg*envs} B ({alg} B per world) |")
st = subprocess.run([sys.executable, os.path.join(here, "ncu_stalls.py"), rep, "12"], capture_output=True, text=True).stdout
md += ["", "Warp-state samples (ncu source counters; `profiles/ncu_stalls.py`):", "", "```", st.rstrip(), "```"]
open(os.path.join(here, f"{rnd}_step_kernel.md"), "w").write("\n".join(md) + "\n")
json.dump({"round": rnd, "envs": envs, "dram_bytes_per_launch": dram, "ncu_duration_us": dur,
           "report": os.path.basename(rep)}, open(os.path.join(here, "ncu_step_kernel.json"), "w"), indent=1)
print("\n".join(lines[-8:]))
print("\n".join(md))
