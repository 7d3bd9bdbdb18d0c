"""Soak run: long stretches of every production path on one B200 -- the planar step (20,000 control steps,
fused policy draw), the step_async pipe (5,000 steps), the 3-D velocity / motion tasks (2,000 steps each,
float32) -- checking that outputs stay finite, device memory stays flat and nothing fails. Prints a
markdown table."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import PIPE_SLOTS, ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

rows = []


def record(name, steps, t, ok, mem0, mem1, extra=""):
    rows.append(f"| {name} | {steps} | {t:.1f} | {'yes' if ok else 'NO'} | {mem0 / 2**20:.1f} → {mem1 / 2**20:.1f} | {extra} |")


env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=4096, seed=0), "Velocity-Rough")
env.reset()
env.step(random_policy(env, 0, fused=True))
torch.cuda.synchronize()
m0 = torch.cuda.memory_allocated()
t0 = time.time()
ok = True
resets = 0
for i in range(1, 20001):
    env.step(random_policy(env, i, fused=True))
    if i % 1000 == 0:
        ok &= bool(torch.isfinite(env.step_outputs.view(torch.uint8)[: 8].float()).all())
        tm = env.termination_manager
        resets += int((tm.terminated | tm.truncated).sum())
        ok &= bool(all(torch.isfinite(env.observation_manager._out[g]).all() for g in env.observation_manager._out))
torch.cuda.synchronize()
record("planar Velocity-Rough 4096, fused policy", 20000, time.time() - t0, ok, m0, torch.cuda.memory_allocated(),
       f"{resets} resets sampled; trigger counts {dict(env.termination_manager.trigger_counts)}")

A = env.action_manager.total_dim
acts = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(64, 4096, A))).pin_memory()
m0 = torch.cuda.memory_allocated()
t0 = time.time()
ok = True
for i in range(5000):
    env.step_async(acts[i % 64])
    if i >= PIPE_SLOTS - 1:
        v = env.step_wait()
        if i % 500 == 0:
            ok &= bool(np.isfinite(v["obs/policy"].numpy()).all())
for _ in range(PIPE_SLOTS - 1):
    env.step_wait()
torch.cuda.synchronize()
record("planar step_async / step_wait pipe", 5000, time.time() - t0, ok, m0, torch.cuda.memory_allocated())
del env

from paper_2601_22074_b200.sim3d import robots  # noqa: E402
from paper_2601_22074_b200.sim3d.motion import synthetic_walk_clip  # noqa: E402
from paper_2601_22074_b200.sim3d.task import MotionTrackingCfg, VelocityEnv3D, VelocityTaskCfg  # noqa: E402

for name, make_cfg in (
        ("3-D G1 velocity (curriculum, scan, events), f32, 4096",
         lambda m, dq: VelocityTaskCfg(dq, height_scan=True, curriculum=(5, 6, 8.0))),
        ("3-D G1 motion imitation, f32, 4096",
         lambda m, dq: MotionTrackingCfg(dq, *synthetic_walk_clip(m, dq)))):
    m = robots.g1_like(rough="curriculum" if "velocity" in name else False)
    dq = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    e3 = VelocityEnv3D(m, make_cfg(m, dq), 4096, dtype="f32")
    e3.reset()
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_allocated()
    t0 = time.time()
    ok = True
    nt = 0
    for i in range(2000):
        a = torch.rand(4096, m.nu, device="cuda") * 2 - 1
        o, r, te, tr = e3.step(a)
        if i % 200 == 0:
            ok &= bool(torch.isfinite(o).all() and torch.isfinite(r).all())
            nt += int(te.sum())
    torch.cuda.synchronize()
    record(name, 2000, time.time() - t0, ok, m0, torch.cuda.memory_allocated(), f"{nt} terminations sampled")
    del e3

print("| path | steps | wall s | finite | device MiB (start → end) | notes |\n|---|---|---|---|---|---|")
print("\n".join(rows))
