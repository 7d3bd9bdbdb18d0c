"""Host cost of the e2e loop (step_async / step_wait), cProfile'd: where the ~21 us of Python per step go."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import PIPE_SLOTS, ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n, K = 4096, 600
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n), "Velocity-Rough")
env.reset()
A = env.action_manager.total_dim
acts = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(K, n, A))).pin_memory()


def loop():
    for i in range(K):
        env.step_async(acts[i])
        if i >= PIPE_SLOTS - 1:
            env.step_wait()
    for _ in range(PIPE_SLOTS - 1):
        env.step_wait()


loop()
torch.cuda.synchronize()
t0 = time.perf_counter()
ta = 0.0
for i in range(K):
    a0 = time.perf_counter()
    env.step_async(acts[i])
    ta += time.perf_counter() - a0
    if i >= PIPE_SLOTS - 1:
        env.step_wait()
for _ in range(PIPE_SLOTS - 1):
    env.step_wait()
print(f"{(time.perf_counter() - t0) / K * 1e6:.1f} us/step, step_async {ta / K * 1e6:.1f} us", flush=True)
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
