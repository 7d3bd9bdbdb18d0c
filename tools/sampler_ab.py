"""Does the nvidia-smi clock sampler perturb the headline step? 20-step timed windows (bench protocol: L2
flush before each step, events around each) right after starting a sampler the way bench.py does (wait for
its first sample), after an extra delay, and with no sampler; 12 trials each."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=4096, seed=0), "Velocity-Rough")
env.reset()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
ctr = [0]


def window(K=20):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for i in range(K):
        flush.fill_(float(i))
        evs[i][0].record(st)
        env.step(random_policy(env, ctr[0], fused=True))
        ctr[0] += 1
        evs[i][1].record(st)
        if i >= 2:
            evs[i - 2][1].synchronize()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) * 1e3 for a, b in evs])


FULL = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
        "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
        "clocks_event_reasons.sw_power_cap")
NOPOWER = FULL.replace("power.draw,", "")
CLOCKS = "index,clocks.sm,clocks.max.sm"
BENCH = "index,clocks.sm,clocks.max.sm,clocks_event_reasons.active"  # bench.py's sampler


def sampler(period_ms, q=FULL):
    path = "/tmp/smi.csv"
    p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                          "-lms", str(period_ms)], stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    t0 = time.time()
    while time.time() - t0 < 5.0:
        with open(path) as fh:
            if sum(1 for _ in fh):
                break
        time.sleep(0.05)
    return p


for i in range(10):
    window()
for name, period, delay, q in (("none", 0, 0, FULL), ("recipe line, 100 ms", 100, 0, FULL),
                               ("recipe line, 200 ms", 200, 0, FULL), ("100 ms no power", 100, 0, NOPOWER),
                               ("100 ms clocks only", 100, 0, CLOCKS), ("bench: 4 fields, 200 ms + 0.5 s", 200, 0.5, BENCH),
                               ("none", 0, 0, FULL)):
    means = []
    for trial in range(12):
        p = sampler(period, q) if period else None
        time.sleep(delay)
        t = window()
        means.append(t.mean())
        if p is not None:
            p.terminate()
            p.wait()
    means = np.array(means)
    print(f"{name:24s}: window means {' '.join(f'{m:.1f}' for m in means)}  (slow: {(means > 22.5).sum()})",
          flush=True)
