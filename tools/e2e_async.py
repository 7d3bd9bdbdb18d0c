"""Timeline probes of the step_async pipeline (planar Velocity-Rough, 4096 worlds)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2601_22074_b200.env import PIPE_SLOTS, ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n, K = 4096, 300
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n), "Velocity-Rough")
env.reset()
A = env.action_manager.total_dim
acts = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(K, n, A))).pin_memory()
dacts = acts[:20].cuda()
st = torch.cuda.current_stream()


def run(label, fn):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        fn(i)
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / K * 1e6:.1f} us/step", flush=True)


run("step(device actions), no sync", lambda i: env.step(dacts[i % 20]))
run("step(pinned actions), no sync", lambda i: env.step(acts[i]))
state = {"n": 0}


def async_only(i):
    env.step_async(acts[i])
    state["n"] += 1
    if state["n"] >= PIPE_SLOTS:
        env.step_wait()
        state["n"] -= 1


run("step_async + step_wait(prev)", async_only)
while state["n"]:
    env.step_wait()
    state["n"] -= 1


t0 = time.perf_counter()
for i in range(K):
    env.step_async(acts[i])
    env.step_wait()
print(f"step_async + immediate step_wait: {(time.perf_counter() - t0) / K * 1e6:.1f} us/step")
# host-side cost breakdown of the pipelined loop
ta = tw = 0.0
n_p = 0
for i in range(K):
    t0 = time.perf_counter()
    env.step_async(acts[i])
    t1 = time.perf_counter()
    n_p += 1
    if n_p >= PIPE_SLOTS:
        env.step_wait()
        n_p -= 1
    t2 = time.perf_counter()
    ta += t1 - t0
    tw += t2 - t1
while n_p:
    env.step_wait()
    n_p -= 1
print(f"host: step_async {ta / K * 1e6:.1f} us/call, step_wait {tw / K * 1e6:.1f} us/call")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for i in range(100):
    env.step_async(acts[i])
    env.step_wait()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)

# floors: back-to-back D2H of the arena (pinned), H2D of the actions, and both at once
nb = env.step_outputs.numel()
hb = torch.empty(nb, dtype=torch.uint8).pin_memory()
ha = acts[0]
da = torch.empty_like(ha, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
run("D2H arena only", lambda i: hb.copy_(env.step_outputs, non_blocking=True))
run("H2D actions only", lambda i: da.copy_(ha, non_blocking=True))


def both(i):
    with torch.cuda.stream(s1):
        hb.copy_(env.step_outputs, non_blocking=True)
    with torch.cuda.stream(s2):
        da.copy_(ha, non_blocking=True)


run("D2H + H2D on two streams", both)
