"""ms per control step of the fused 3-D G1 velocity task (rough + scan, random actions, L2 flushed between
steps) at N worlds, f32 and f64, under the environment's S3_* knobs (A/B driver: run once per setting).
    python tools/sim3d_task_time.py [N]"""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("S3_"))
out = []
for dtype in ("f32", "f64"):
    m = robots.g1_like(rough=True)
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
    env = VelocityEnv3D(m, cfg, n, dtype=dtype)
    env.reset()
    acts = torch.rand(16, n, m.nu, device="cuda", dtype=env.dm.tdtype) * 2 - 1
    for i in range(4):
        env.step(acts[i])
    t = timed_steps(env, 10, flush, stream, lambda i: acts[4 + i])
    out.append(f"{dtype} {1e3 * t / 10:.3f} ms")
    del env
print(f"[{knobs}] N={n}: " + ", ".join(out), flush=True)
