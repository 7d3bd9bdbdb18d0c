"""Steady-state step for ncu: warm up W control steps (episodes desynchronize,
resets occur), then run P profiled steps. Also prints the CUDA-event time of
those steps when run without ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(os.environ.get("N", "4096"))
warm = int(os.environ.get("WARM", "200"))
prof = int(os.environ.get("PROF", "20"))
env = ManagerBasedRlEnv(make_env_cfg(os.environ.get("TASK", "Velocity-Rough"), num_envs=n))
env.reset()
for i in range(warm):
    env.step(random_policy(env, i))
torch.cuda.synchronize()
a = random_policy(env, 0)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(prof)]
for i in range(prof):
    ev[i][0].record()
    env.step(a)
    ev[i][1].record()
torch.cuda.synchronize()
ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
print(f"N={n} steady-state step (warm L2, back-to-back): median {ts[len(ts)//2]:.1f} us, min {ts[0]:.1f} us")
