"""One 3-D control step (4 substeps) of N worlds after warm-up: the ncu target.
usage: python tools/sim3d_profile.py [robot] [dtype] [N]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.device import Data, DeviceModel

robot = sys.argv[1] if len(sys.argv) > 1 else "g1"
dtype = sys.argv[2] if len(sys.argv) > 2 else "f64"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
m = robots.g1_like() if robot == "g1" else robots.go1_like()
table = robots.G1_DEFAULT_JOINTS if robot == "g1" else robots.GO1_DEFAULT_JOINTS
dm = DeviceModel(m, dtype)
dm.set_const()
d = Data(dm, n)
q0 = robots.default_qpos(m, table)
d.qpos.copy_(torch.as_tensor(np.tile(q0, (n, 1))))
d.ctrl.copy_(torch.as_tensor(np.tile(q0[m.actuator_qposadr], (n, 1))))
for _ in range(20):
    d.step(4)
torch.cuda.synchronize()
d.step(4)
torch.cuda.synchronize()
print("done", d.qpos[:, 2].float().mean().item())
