"""Solver statistics of the 3-D G1 task under random actions (Newton iterations, contacts, rows)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.task import VelocityEnv3D, VelocityTaskCfg

dtype = sys.argv[1] if len(sys.argv) > 1 else "f32"
n = 4096
m = robots.g1_like(rough=True)
cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
env = VelocityEnv3D(m, cfg, n, dtype=dtype)
env.reset()
for k in range(40):
    a = torch.rand(n, m.nu, device="cuda", dtype=env.dm.tdtype) * 2 - 1
    env.step(a)
    if k % 10 == 9:
        d = env.data
        d.ctrl.copy_(torch.as_tensor(cfg.default_qpos[m.actuator_qposadr], device="cuda") + 0.25 * env.action)
        saved = (d.qpos.clone(), d.qvel.clone(), d.qacc_warmstart.clone())
        out = d.step(1, outputs=True)
        d.qpos.copy_(saved[0]); d.qvel.copy_(saved[1]); d.qacc_warmstart.copy_(saved[2])
        it = out["solver_niter"].float(); nc = out["ncon"].float(); ne = out["nefc"].float()
        print(f"step {k+1}: niter mean {it.mean():.2f} max {it.max():.0f} hist {torch.bincount(out['solver_niter'].long(), minlength=11).tolist()} "
              f"ncon mean {nc.mean():.2f} max {nc.max():.0f} nefc mean {ne.mean():.1f} dropped {out['ndropped'].float().mean():.2f} "
              f"term {env.terminated.float().mean():.3f} z {d.qpos[:,2].float().mean():.3f}", flush=True)
