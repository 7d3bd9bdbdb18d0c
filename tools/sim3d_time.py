"""Time the 3-D step kernel (G1-like, 4 substeps per launch) at a few world counts."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.device import Data, DeviceModel

for name, make, table in (("g1_flat", lambda: robots.g1_like(), robots.G1_DEFAULT_JOINTS),
                          ("g1_rough", lambda: robots.g1_like(rough=True), robots.G1_DEFAULT_JOINTS),
                          ("go1_flat", lambda: robots.go1_like(), robots.GO1_DEFAULT_JOINTS)):
    for dtype in ("f64", "f32"):
        m = make()
        dm = DeviceModel(m, dtype)
        dm.set_const()
        for n in (4096, 16384):
            d = Data(dm, n)
            q0 = robots.default_qpos(m, table)
            d.qpos.copy_(torch.as_tensor(np.tile(q0, (n, 1))))
            d.ctrl.copy_(torch.as_tensor(np.tile(q0[m.actuator_qposadr], (n, 1))))
            for _ in range(3):
                d.step(4)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            K = 10
            for _ in range(K):
                d.step(4)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            out = d.step(1, outputs=True)
            torch.cuda.synchronize()
            print(f"{name} {dtype} N={n} wpb={dm.layout.warps_per_block} smem/world={dm.layout.elems_per_world*(8 if dtype=='f64' else 4)}B "
                  f"ms/step(4 sub)={ms:.3f} env-steps/s={n/ms*1e3:.3e} ncon_mean={out['ncon'].float().mean().item():.2f} "
                  f"niter_mean={out['solver_niter'].float().mean().item():.2f} z_mean={d.qpos[:,2].float().mean().item():.3f}", flush=True)
