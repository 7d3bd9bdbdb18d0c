"""Is the e2e loop host-bound? The bench's step_async / step_wait loop (Velocity-Rough 4096, 300 steps)
with the host time split into step_async (enqueue), step_wait (blocking) and the rest, plus the same loop
with a bare D2H copy per step instead of the env step (the PCIe floor of the pipe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import PIPE_SLOTS, ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n, K = 4096, 300
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n), "Velocity-Rough")
env.reset()
A = env.action_manager.total_dim
acts = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(K, n, A))).pin_memory()
for rep in range(4):
    torch.cuda.synchronize()
    ta = tw = 0.0
    t0 = time.perf_counter()
    for i in range(K):
        a0 = time.perf_counter()
        env.step_async(acts[i])
        a1 = time.perf_counter()
        ta += a1 - a0
        if i >= PIPE_SLOTS - 1:
            v = env.step_wait()
            tw += time.perf_counter() - a1
            float(v["reward"][0])
    for _ in range(PIPE_SLOTS - 1):
        env.step_wait()
    tt = time.perf_counter() - t0
    print(f"rep {rep}: {tt / K * 1e6:.1f} us/step  step_async {ta / K * 1e6:.1f}  step_wait {tw / K * 1e6:.1f}  "
          f"-> {n * K / tt / 1e6:.1f} M env-steps/s", flush=True)

# the copies alone: one 1.58 MB D2H per step on a side stream, waited S steps later
nb = env.step_outputs.numel()
src = torch.empty(nb, dtype=torch.uint8, device="cuda")
hosts = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(PIPE_SLOTS + 1)]
s = torch.cuda.Stream()
evs = []
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(K):
    with torch.cuda.stream(s):
        hosts[i % len(hosts)].copy_(src, non_blocking=True)
        e = torch.cuda.Event()
        e.record(s)
    evs.append(e)
    if i >= PIPE_SLOTS - 1:
        evs[i - PIPE_SLOTS + 1].synchronize()
torch.cuda.synchronize()
tt = time.perf_counter() - t0
print(f"bare D2H copies of {nb} B: {tt / K * 1e6:.1f} us/step", flush=True)

# transfer size vs per-copy overhead: back-to-back D2H copies of k arenas (k = 1, 2, 4), per arena
for k in (1, 2, 4):
    big = torch.empty(k * nb, dtype=torch.uint8, device="cuda")
    hb = [torch.empty(k * nb, dtype=torch.uint8).pin_memory() for _ in range(3)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M = K // k
        with torch.cuda.stream(s):
            for i in range(M):
                hb[i % 3].copy_(big, non_blocking=True)
        torch.cuda.synchronize()
        tt = time.perf_counter() - t0
        print(f"k={k}: {tt / (M * k) * 1e6:.1f} us per arena ({k * nb * M / tt / 1e9:.1f} GB/s)", flush=True)
