"""Measure host-side (Python) cost per env.step vs GPU time; cProfile the step."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n))
env.reset()
for i in range(20):
    env.step(random_policy(env, i))
torch.cuda.synchronize()
K = 500
t0 = time.perf_counter()
for i in range(K):
    env.step(random_policy(env, i))
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"N={n}: host enqueue {1e6*(t1-t0)/K:.1f} us/step, wall incl. drain {1e6*(t2-t0)/K:.1f} us/step, "
      f"{n*K/(t2-t0)/1e6:.1f} M env-steps/s back-to-back")
a = random_policy(env, 0)
t0 = time.perf_counter()
for i in range(K):
    env.step(a)
torch.cuda.synchronize()
print(f"step only: {1e6*(time.perf_counter()-t0)/K:.1f} us/step")
t0 = time.perf_counter()
for i in range(K):
    random_policy(env, i)
torch.cuda.synchronize()
print(f"policy only: {1e6*(time.perf_counter()-t0)/K:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for i in range(200):
    env.step(random_policy(env, i))
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# ---- end-to-end loop breakdown (bench.py e2e: pinned H2D -> step -> one D2H of step_outputs)
import numpy as np  # noqa: E402

A = env.action_manager.total_dim
host_actions = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(n, A))).pin_memory()
host_out = torch.empty(env.step_outputs.numel(), dtype=torch.uint8).pin_memory()
dev_actions = torch.empty((n, A), dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()


def timed(label, fn, k=300):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    print(f"{label:<40s} {1e6 * (time.perf_counter() - t0) / k:7.1f} us")


timed("H2D actions + sync", lambda: (dev_actions.copy_(host_actions, non_blocking=True), stream.synchronize()))
timed("D2H step_outputs + sync", lambda: (host_out.copy_(env.step_outputs, non_blocking=True), stream.synchronize()))
timed("step + sync", lambda: (env.step(dev_actions), stream.synchronize()))
timed("e2e (H2D, step, D2H, sync)", lambda: (dev_actions.copy_(host_actions, non_blocking=True), env.step(dev_actions),
                                             host_out.copy_(env.step_outputs, non_blocking=True), stream.synchronize()))
t0 = time.perf_counter()
for _ in range(300):
    dev_actions.copy_(host_actions, non_blocking=True)
    env.step(dev_actions)
    host_out.copy_(env.step_outputs, non_blocking=True)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"{'e2e host enqueue only':<40s} {1e6 * (t1 - t0) / 300:7.1f} us")
print("D2H bytes", env.step_outputs.numel())

# ---- zero-copy host I/O (enable_host_outputs + pinned actions read in place)
host_views = env.enable_host_outputs()
pinned = host_actions
env.step(pinned)
torch.cuda.synchronize()
timed("zero-copy e2e (step(pinned), sync)", lambda: (env.step(pinned), stream.synchronize()))
t0 = time.perf_counter()
for _ in range(300):
    env.step(pinned)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"{'zero-copy host enqueue only':<40s} {1e6 * (t1 - t0) / 300:7.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for _ in range(100):
    e0.record()
    env.step(pinned)
    e1.record()
    e1.synchronize()
    tot += e0.elapsed_time(e1)
print(f"{'zero-copy step GPU time (events, host-bound)':<40s} {10 * tot:7.1f} us")
