"""clock64() phase probes of world 0 inside the JIT step (SS_PROBES=1)."""
import os
import sys

os.environ["SS_PROBES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(os.environ.get("N", "4096"))
cfg = make_env_cfg(os.environ.get("TASK", "Velocity-Rough"), num_envs=n)
if os.environ.get("NO_NOISE"):  # experiment: observation noise off
    from paper_2601_22074_b200.config import NoiseCfg
    for g in cfg.observations.values():
        for t in g.terms.values():
            t.noise = NoiseCfg()
if os.environ.get("NO_SCAN"):  # experiment: no height scan term
    cfg.observations["critic"].terms.pop("height_scan", None)
if os.environ.get("NO_CRITIC"):  # experiment: policy group only
    cfg.observations.pop("critic", None)
env = ManagerBasedRlEnv(cfg)
probe = torch.zeros(16, dtype=torch.int64, device="cuda")
env.reset()
env._probe_ptr = probe.data_ptr()
env._invalidate()
names = ["start", "loads+params", "action", "sub0", "sub1", "sub2", "sub3", "post-sim", "term", "reward",
         "cur+reset", "cmd+events", "obs", "stores"]
acc = [0.0] * 14
span = 0.0
K = 50
probe[14] = 2**62
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if os.environ.get("FLUSH") else None
for i in range(200 + K):
    if flush is not None:
        flush.fill_(float(i))  # cold L2 (as bench.py): code and data come from HBM
    if i >= 200:
        probe[14] = 2**62
        probe[15] = 0
    env.step(random_policy(env, i, fused=True))
    if i >= 200:
        torch.cuda.synchronize()
        p = probe.cpu().tolist()
        span += (p[15] - p[14]) / 1e3
        probe[14] = 2**62
        probe[15] = 0
        for j in range(1, 14):
            acc[j] += p[j] - p[j - 1]
tot = sum(acc)
print(f"kernel span (globaltimer, first warp start -> last warp end): {span / K:.1f} us")
print(f"N={n} world-0 phase cycles (mean of {K} steps), total {tot / K:.0f} cycles = {tot / K / 1.965e3:.1f} us at 1.965 GHz")
for j in range(1, 14):
    print(f"  {names[j - 1]:>12s} -> {names[j]:<12s} {acc[j] / K:8.0f} cycles  {100 * acc[j] / tot:5.1f} %")
