"""Env-count sweep of the fused 3-D G1 velocity task (rough + height scan, random actions, L2 flushed
between steps): env-steps/s per world count and dtype -> markdown table on stdout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from bench import timed_steps  # noqa: E402
from paper_2601_22074_b200.sim3d import robots  # noqa: E402
from paper_2601_22074_b200.sim3d.task import VelocityEnv3D, VelocityTaskCfg  # noqa: E402

flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
print("| worlds | dtype | ms / control step | env-steps/s |\n|---|---|---|---|")
for dtype in ("f32", "f64"):
    for n in (1024, 4096, 16384, 65536):
        m = robots.g1_like(rough=True)
        cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
        env = VelocityEnv3D(m, cfg, n, dtype=dtype)
        env.reset()
        acts = torch.rand(8, n, m.nu, device="cuda", dtype=env.dm.tdtype) * 2 - 1
        for i in range(3):
            env.step(acts[i])
        t = timed_steps(env, 5, flush, stream, lambda i: acts[3 + i])
        print(f"| {n} | {dtype} | {1e3 * t / 5:.2f} | {n * 5 / t:.3e} |", flush=True)
        del env
