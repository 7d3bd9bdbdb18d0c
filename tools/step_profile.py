"""cProfile of the host side of env.step (device actions, fused random policy)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import RandomActions  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=4096))
env.reset()
a = torch.zeros((4096, 4), dtype=torch.float64, device="cuda")
pinned = torch.zeros((4096, 4), dtype=torch.float64).pin_memory()
for arg, name in ((a, "device"), (RandomActions(), "fused"), (pinned, "pinned")):
    for _ in range(50):
        env.step(arg)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(200):
        torch.cuda._sleep(5_000_000)  # GPU busy: launches queue, the host never waits
        t0 = time.perf_counter()
        for _ in range(4):  # within the nonfinite lag: no event wait
            env.step(arg)
        tot += time.perf_counter() - t0
        torch.cuda.synchronize()
    print(f"{name}: host {1e6 * tot / 800:.1f} us/step (GPU kept busy)")
# raw cost of the pieces
d = env._get_desc()
la = env._la
la.stages = 0x3DFF
la.nsub = 4
la.actions = a.data_ptr()
la.policy_slot = -1
la.poll_keep = 4
la.groups_mask = 3
lib = env._lib
h = env._jit_handle
s = torch._C._cuda_getCurrentRawStream(0)
torch.cuda.synchronize()
for label, fn in (("ss_rt_launch (ctypes)", lambda: lib.ss_rt_launch(env._desc_ref, env._rt_ref, env._la_ref, h, s)),
                  ("raw stream query", lambda: torch._C._cuda_getCurrentRawStream(0)),
                  ("om.begin", lambda: env.observation_manager.begin(list(env.observation_manager.groups))),
                  ("check_actions(pinned)", lambda: env.action_manager.check_actions(pinned)),
                  ("check_actions(device)", lambda: env.action_manager.check_actions(a))):
    tot = 0.0
    for _ in range(200):
        torch.cuda._sleep(5_000_000)
        t0 = time.perf_counter()
        for _ in range(4):
            fn()
        tot += time.perf_counter() - t0
        torch.cuda.synchronize()
    print(f"{label:<28s} {1e6 * tot / 800:6.2f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    env.step(a)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
