"""Kernel A/B: fused-step time (fused random policy, L2 flushed before each step, CUDA events) per task
and world count, under the environment's JIT knobs (run once per knob setting).
    python tools/kab.py [Velocity-Rough] [4096,262144]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402
from paper_2601_22074_b200.traffic import step_bytes_per_world  # noqa: E402

tasks = sys.argv[1].split(",") if len(sys.argv) > 1 else ["Velocity-Rough"]
sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4096", "262144"])]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SS_"))
for task in tasks:
    for n in sizes:
        env = ManagerBasedRlEnv(make_env_cfg(task, num_envs=n), task)
        env.reset()
        for i in range(10):
            env.step(random_policy(env, i, fused=True))
        K = 60 if n <= 65536 else 30
        ts = []
        for i in range(K):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            env.step(random_policy(env, 10 + i, fused=True))
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        med = ts[len(ts) // 2]
        mean = sum(ts) / len(ts)
        bpw = step_bytes_per_world(env, fused_policy=True)["total"]
        print(f"[{knobs}] {task} N={n}: median {med:.2f} us mean {mean:.2f} us  {bpw * n / mean / 1e3:.0f} GB/s "
              f"({bpw * n / mean / 1e3 / 6535.1:.3f})", flush=True)
        del env
        torch.cuda.empty_cache()
