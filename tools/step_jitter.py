"""Per-step device time distribution of the headline step (Velocity-Rough 4096, fused policy draw, L2 flushed
before every step, CUDA events on the launching stream): is a slow bench run a slow process or a few slow steps?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(os.environ.get("N", "4096"))
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n, seed=0), "Velocity-Rough")
env.reset()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for i in range(10):
    env.step(random_policy(env, i, fused=True))
if os.environ.get("SAMPLER") == "1":  # an nvidia-smi sampler beside the timed loop (as bench.py runs one)
    import subprocess
    import time

    q = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(float(os.environ.get("SAMPLER_DELAY", "0.5")))
for rep in range(int(os.environ.get("REPS", "6"))):
    K = 100
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for i in range(K):
        flush.fill_(float(i))
        evs[i][0].record(st)
        env.step(random_policy(env, 10 + rep * K + i, fused=True))
        evs[i][1].record(st)
        if i >= 2:
            evs[i - 2][1].synchronize()
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) * 1e3 for a, b in evs])
    q = np.percentile(t, [0, 10, 50, 90, 100])
    print(f"rep {rep}: mean {t.mean():.2f} us  min/p10/p50/p90/max " + " ".join(f"{x:.2f}" for x in q), flush=True)
