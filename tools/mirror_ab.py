"""GPU time of a zero-copy step (pinned actions in, host-mirrored outputs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(os.environ.get("N", "4096"))
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n))
env.reset()
A = env.action_manager.total_dim
pinned = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(n, A))).pin_memory()
mode = os.environ.get("MODE", "both")
if mode in ("both", "out"):
    env.enable_host_outputs()
if mode in ("out", "none"):
    pinned = pinned.cuda()
for _ in range(10):
    env.step(pinned)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
K = 100
spin = torch.empty(1, device="cuda")
for _ in range(K):
    torch.cuda._sleep(200000)  # keep the GPU busy so the launch is queued before e0 fires
    e0.record()
    env.step(pinned)
    e1.record()
    e1.synchronize()
    tot += e0.elapsed_time(e1)
gpu = 1e3 * tot / K
import time  # noqa: E402
t0 = time.perf_counter()
for _ in range(K):
    env.step(pinned)
    torch.cuda.current_stream().synchronize()
wall = 1e6 * (time.perf_counter() - t0) / K
print(f"{os.environ.get('TAG', '')} mode={mode}: zero-copy step GPU {gpu:.1f} us, closed loop {wall:.1f} us "
      f"({n / wall:.1f} M env-steps/s), {env.step_outputs.numel() / (gpu * 1e-6) / 1e9:.1f} GB/s out")
