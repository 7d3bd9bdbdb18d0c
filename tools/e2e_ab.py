"""e2e A/B: the bench's step_async / step_wait loop (Velocity-Rough 4096, 200 steps) under the
environment's pipe knobs (SS_PIPE_SLOTS, SS_PIPE_OUT2), several repetitions."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import PIPE_SLOTS, ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n, K = 4096, 200
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n), "Velocity-Rough")
env.reset()
A = env.action_manager.total_dim
acts = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(K, n, A))).pin_memory()
for i in range(5):
    env.step_async(acts[i])
    env.step_wait()
res = []
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    chk = 0.0
    for i in range(K):
        env.step_async(acts[i])
        if i >= PIPE_SLOTS - 1:
            chk += float(env.step_wait()["reward"][0])
    for _ in range(PIPE_SLOTS - 1):
        env.step_wait()
    res.append((time.perf_counter() - t0) / K * 1e6)
knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SS_PIPE"))
print(f"[{knobs}] slots={PIPE_SLOTS}: us/step {' '.join(f'{r:.1f}' for r in res)} -> {n / min(res) * 1e6 / 1e6:.1f} M env-steps/s best")
