"""Upper bounds for splitting the post-physics stages of the 4096-world step over several lanes per world:
the headline step timed (bench protocol: L2 flush before every step, events around each, fused policy
draw) with a stage's work removed from the config -- observation noise off, the critic's height scan
off, both, and terminations that never fire (no reset path). The step is the slowest warp's chain, so a
stage that costs little when removed cannot gain much when parallelised."""
import copy
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.config import NoiseCfg  # noqa: E402
from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timed(cfg, K=200):
    env = ManagerBasedRlEnv(cfg, "Velocity-Rough")
    env.reset()
    st = torch.cuda.current_stream()
    for i in range(10):
        env.step(random_policy(env, i, fused=True))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for i in range(K):
        flush.fill_(float(i))
        evs[i][0].record(st)
        env.step(random_policy(env, 10 + i, fused=True))
        evs[i][1].record(st)
        if i >= 2:
            evs[i - 2][1].synchronize()
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) * 1e3 for a, b in evs])
    resets = float(env.termination_manager.terminated.float().mean() + env.termination_manager.truncated.float().mean())
    del env
    return np.median(t), t.mean(), resets


def variant(name):
    cfg = make_env_cfg("Velocity-Rough", num_envs=4096, seed=0)
    if "nonoise" in name:
        for t in cfg.observations["policy"].terms.values():
            t.noise = NoiseCfg(kind="none", scale=0.0)
    if "noscan" in name:
        del cfg.observations["critic"].terms["height_scan"]
    if "noreset" in name:
        for t in cfg.terminations.values():
            t.params = dict(t.params)
        cfg.terminations["base_height_below"].params["min_height"] = -1e9
        cfg.terminations["pitch_beyond"].params["max_pitch"] = 1e9
        cfg.episode_length_s = 1e6
    return cfg


for rep in range(2):
    for name in ("base", "nonoise", "noscan", "nonoise+noscan", "noreset", "nonoise+noscan+noreset"):
        try:
            med, mean, r = timed(variant(name))
            print(f"{name:26s} median {med:6.2f} us  mean {mean:6.2f} us  (reset fraction last step {r:.4f})", flush=True)
        except Exception as e:  # a config knob this variant needs is missing: say so
            print(f"{name:26s} skipped: {e}", flush=True)
