"""One fused 3-D control step (G1-like rough + height scan, N worlds) after warm-up: the ncu target.
usage: python tools/sim3d_env_profile.py [dtype] [N]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.task import VelocityEnv3D, VelocityTaskCfg

dtype = sys.argv[1] if len(sys.argv) > 1 else "f32"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
m = robots.g1_like(rough=True)
cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
env = VelocityEnv3D(m, cfg, n, dtype=dtype)
env.reset()
acts = torch.rand(12, n, m.nu, device="cuda", dtype=env.dm.tdtype) * 2 - 1
for i in range(11):
    env.step(acts[i])
torch.cuda.synchronize()
env.step(acts[11])
torch.cuda.synchronize()
print("done", env.reward.float().mean().item())
