"""Where the end-to-end step time goes (pinned host actions in, results to pinned host memory).

Prints per-step: (a) the bench's e2e loop (step + stream sync), (b) host enqueue cost of env.step alone,
(c) device time of the kernel with host outputs (events), (d) device time with device outputs only,
(e) e2e with device outputs + one explicit D2H copy of the arena, (f) a plain 1.58 MB D2H copy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
K = 300
env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n), "Velocity-Rough")
env.reset()
A = env.action_manager.total_dim
acts = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(K, n, A))).pin_memory()
st = torch.cuda.current_stream()


def loop(sync=True, copy_out=None):
    for i in range(10):
        env.step(acts[i])
        st.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        env.step(acts[i])
        if copy_out is not None:
            copy_out.copy_(env.step_outputs, non_blocking=True)
        if sync:
            st.synchronize()
    st.synchronize()
    return (time.perf_counter() - t0) / K * 1e6


def dev_time():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.synchronize()
    e0.record()
    for i in range(K):
        env.step(acts[i])
    e1.record()
    st.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


print(f"arena bytes {env.step_outputs.numel()}  actions bytes {n * A * 8}")
print(f"(d) device outputs, pinned actions: device {dev_time():.1f} us/step, e2e loop {loop():.1f} us/step")
host = torch.empty(env.step_outputs.numel(), dtype=torch.uint8).pin_memory()
print(f"(e) device outputs + explicit D2H copy: e2e {loop(copy_out=host):.1f} us/step")
env.enable_host_outputs()
for i in range(5):
    env.step(acts[i])
st.synchronize()
print(f"(c) host outputs (kernel writes pinned host): device {dev_time():.1f} us/step")
print(f"(a) bench e2e loop: {loop():.1f} us/step")
t0 = time.perf_counter()
for i in range(K):
    env.step(acts[i])
t1 = time.perf_counter()
st.synchronize()
print(f"(b) host enqueue only: {(t1 - t0) / K * 1e6:.1f} us/step")
dev = torch.empty(env.step_outputs.numel(), dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(K):
    host.copy_(dev, non_blocking=True)
e1.record()
st.synchronize()
print(f"(f) plain D2H copy of the arena: {e0.elapsed_time(e1) / K * 1e3:.1f} us "
      f"({env.step_outputs.numel() / (e0.elapsed_time(e1) / K * 1e-3) / 1e9:.1f} GB/s)")
