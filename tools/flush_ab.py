"""A/B of the L2-flush protocol between timed steps (untimed flush; CUDA events around the step):
(a) a 512 MiB write only, (b) the write followed by a 256 MiB read, so the flush's own dirty lines are
written back before the events start; for an empty kernel (torch's zero_ of 16 B), the fused step at
4096 and at 262144 worlds."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

wbuf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
rbuf = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
sink = torch.empty(1, device="cuda")


def timed(fn, mode, steps=30):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        wbuf.fill_(float(i))
        if mode == "write+read":
            torch.sum(rbuf, dim=0, out=sink[0])
        evs[i][0].record()
        fn(i)
        evs[i][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs[3:])
    return t[len(t) // 2], sum(t) / len(t)


tiny = torch.zeros(4, device="cuda")
for n in (0, 4096, 262144):
    if n == 0:
        fn = lambda i: tiny.zero_()  # noqa: E731
        name = "empty (zero_ of 16 B)"
    else:
        env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n, seed=0), "Velocity-Rough")
        env.reset()
        for i in range(5):
            env.step(random_policy(env, i, fused=True))
        fn = lambda i, env=env: env.step(random_policy(env, i, fused=True))  # noqa: E731
        name = f"fused step N={n}"
    for mode in ("write", "write+read", "none"):
        if mode == "none":
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
            for i in range(30):
                evs[i][0].record()
                fn(i)
                evs[i][1].record()
            torch.cuda.synchronize()
            t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs[3:])
            med, mean = t[len(t) // 2], sum(t) / len(t)
        else:
            med, mean = timed(fn, mode)
        print(f"{name:28s} flush={mode:11s} median {med:8.2f} us  mean {mean:8.2f} us", flush=True)
