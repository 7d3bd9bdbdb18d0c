"""Newton vs CG (Opt.solver) on the fused 3-D G1 velocity task: ms per control step at 4096 worlds, f32 /
f64, L2 flushed between steps (bench protocol), default iteration caps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from bench import timed_steps  # noqa: E402
from paper_2601_22074_b200.sim3d import robots  # noqa: E402
from paper_2601_22074_b200.sim3d.model import Opt  # noqa: E402
from paper_2601_22074_b200.sim3d.task import VelocityEnv3D, VelocityTaskCfg  # noqa: E402

flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for dtype in ("f32", "f64"):
    for solver, iters in (("newton", 10), ("cg", 10), ("cg", 30)):
        m = robots.g1_like(rough=True, opt=Opt(solver=solver, iterations=iters))
        cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
        env = VelocityEnv3D(m, cfg, n, dtype=dtype)
        env.reset()
        acts = torch.rand(10, n, m.nu, device="cuda", dtype=env.dm.tdtype) * 2 - 1
        for i in range(3):
            env.step(acts[i])
        t = timed_steps(env, 5, flush, stream, lambda i: acts[3 + i])
        cost = env.solver_cost.float().mean().item() / 4 if env.solver_cost is not None else float("nan")
        print(f"{dtype} {solver:6s} cap {iters:2d}: {1e3 * t / 5:.2f} ms / control step, {n * 5 / t:.3e} env-steps/s, "
              f"{cost:.1f} solver iterations per substep", flush=True)
        del env
