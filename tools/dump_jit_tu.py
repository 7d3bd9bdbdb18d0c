"""Write the NVRTC translation unit of a task's specialized step kernel
(for offline ptxas/SASS inspection with tools/jit_offline.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_22074_b200 import jit  # noqa: E402
from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
os.makedirs(out, exist_ok=True)
for task in ("Velocity-Rough", "Velocity-Flat", "Velocity-Flat-Quad12", "Velocity-Rough-Humanoid10"):
    env = ManagerBasedRlEnv(make_env_cfg(task, num_envs=4096))
    env.reset()
    with open(os.path.join(out, f"jit_tu_{task}.cu"), "w") as fh:
        fh.write(jit.kernel_source(env._get_desc()))
    print(task, "ok")
