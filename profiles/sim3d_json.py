"""Write profiles/ncu_sim3d_env_kernel.json (read by bench.py's 3-D leg) from the two ncu --set full
captures of the 3-D env kernel.

    python profiles/sim3d_json.py <f32.ncu-rep> <f64.ncu-rep>
"""
import csv
import json
import os
import subprocess
import sys

WANT = {"Duration": ("duration_ms", 1.0), "Executed Ipc Active": ("executed_ipc_active", 1.0),
        "Issue Slots Busy": ("issue_slots_busy_frac", 0.01), "Achieved Occupancy": ("achieved_occupancy_frac", 0.01),
        "DRAM Throughput": ("dram_throughput_frac", 0.01), "L1/TEX Hit Rate": ("l1_hit_frac", 0.01),
        "Registers Per Thread": ("registers_per_thread", 1.0),
        "Dynamic Shared Memory Per Block": ("smem_kb_per_block", 1.0),
        "Warp Cycles Per Issued Instruction": ("warp_cycles_per_issued_instruction", 1.0)}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    iname, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    got = {}
    for r in rows[1:]:
        if r[iname] in WANT and WANT[r[iname]][0] not in got:
            key, scale = WANT[r[iname]]
            v = float(r[ival].replace(",", ""))
            if r[iname] == "Duration":
                v = v / 1e3 if r[iunit] == "us" else (v / 1e6 if r[iunit] == "ns" else v)
            got[key] = round(v * scale, 4)
    return got


here = os.path.dirname(os.path.abspath(__file__))
doc = {"f32": metrics(sys.argv[1]), "f64": metrics(sys.argv[2]),
       "source": "ncu --set full --import-source on --clock-control none of tools/sim3d_env_profile.py <dtype> 4096 "
                 "(one fused control step, current defaults); summaries in profiles/r1_sim3d_env_kernel_<dtype>.md"}
with open(os.path.join(here, "ncu_sim3d_env_kernel.json"), "w") as fh:
    json.dump(doc, fh, indent=1)
print(json.dumps(doc, indent=1))
