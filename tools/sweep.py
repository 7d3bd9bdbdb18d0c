"""Env-count scaling sweep on one B200 (BASELINE configs[4] restated):
env-steps/s of policy+step per task and N, warm back-to-back and with the
L2 flushed before each step, plus algorithmic GB/s of the fused kernel.
Writes a markdown table to stdout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402
from paper_2601_22074_b200.traffic import step_bytes_per_world  # noqa: E402

tasks = sys.argv[1].split(",") if len(sys.argv) > 1 else ["Velocity-Rough"]
sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1024", "4096", "16384", "65536", "262144"])]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
try:
    import json

    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    PEAK = 6650.0
print("Fused random policy (one launch per control step, `random_policy(env, i, fused=True)`).")
print()
print(f"| task | N | step us (warm) | env-steps/s (warm) | step us (L2 flushed) | env-steps/s (flushed) | B/env-step | "
      f"GB/s (flushed) | frac of {PEAK:.0f} GB/s |")
print("|---|---|---|---|---|---|---|---|---|")
for task in tasks:
    for n in sizes:
        env = ManagerBasedRlEnv(make_env_cfg(task, num_envs=n))
        env.reset()
        for i in range(60):
            env.step(random_policy(env, i, fused=True))
        torch.cuda.synchronize()
        K = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(K):
            env.step(random_policy(env, i, fused=True))
        e1.record()
        torch.cuda.synchronize()
        warm = e0.elapsed_time(e1) * 1e3 / K
        tot = 0.0
        for i in range(20):
            flush.fill_(float(i))
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            env.step(random_policy(env, 60 + K + i, fused=True))
            a1.record()
            a1.synchronize()
            tot += a0.elapsed_time(a1) * 1e3
        tot /= 20
        b = step_bytes_per_world(env, fused_policy=True)["total"]
        gbs = b * n / (tot * 1e-6) / 1e9
        print(f"| {task} | {n} | {warm:.1f} | {n / warm * 1e6:,.0f} | {tot:.1f} | {n / tot * 1e6:,.0f} | {b} | {gbs:,.0f} | "
              f"{gbs / PEAK:.3f} |", flush=True)
        del env
        torch.cuda.empty_cache()
