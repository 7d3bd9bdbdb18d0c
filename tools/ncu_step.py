"""Profiling target: the bench's headline step exactly (Velocity-Rough, fused random policy, a 512 MiB L2
flush before each step). Launches: 1 reset + WARM warm-up steps + PROF profiled steps of ss_step_jit, so
`ncu -k regex:ss_step_jit -s <1 + WARM> -c 1` captures a steady-state step.
    N=4096 WARM=11 PROF=3 python tools/ncu_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(os.environ.get("N", "4096"))
warm, prof = int(os.environ.get("WARM", "11")), int(os.environ.get("PROF", "3"))
env = ManagerBasedRlEnv(make_env_cfg(os.environ.get("TASK", "Velocity-Rough"), num_envs=n), "Velocity-Rough")
env.reset()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for i in range(warm + prof):
    flush.fill_(float(i))
    env.step(random_policy(env, i, fused=True))
torch.cuda.synchronize()
print(f"ok: {n} worlds, {warm + prof} steps, use_jit={env.use_jit}")
