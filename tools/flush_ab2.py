"""Where does the ~6 us between two events around an empty kernel come from after an L2 flush?
Variants before e0 (all untimed): 512 MiB write; the write + a 40 us GPU spin (torch.cuda._sleep) that
lets the flush's write-back drain; a 16 MiB write; a 40 us spin alone."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

big = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
small = torch.empty(16 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
SPIN = 80000  # cycles (~40 us)


def pre(mode, i):
    if mode in ("write", "write+spin"):
        big.fill_(float(i))
    if mode == "small-write":
        small.fill_(float(i))
    if mode in ("write+spin", "spin"):
        torch.cuda._sleep(SPIN)


def timed(fn, mode, steps=40):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        pre(mode, i)
        evs[i][0].record()
        fn(i)
        evs[i][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs[3:])
    return t[len(t) // 2], t[0]


tiny = torch.zeros(4, device="cuda")
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=4096, seed=0), "Velocity-Rough")
env.reset()
for i in range(5):
    env.step(random_policy(env, i, fused=True))
for name, fn in (("empty", lambda i: tiny.zero_()), ("step4096", lambda i: env.step(random_policy(env, i, fused=True)))):
    for mode in ("write", "write+spin", "small-write", "spin"):
        med, lo = timed(fn, mode)
        print(f"{name:10s} {mode:12s} median {med:7.2f} us  min {lo:7.2f} us", flush=True)
