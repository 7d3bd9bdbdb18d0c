"""How much of the 4096-world step is cold code? The bench protocol flushes L2 (512 MiB write) before each
timed step, which also evicts the kernel's ~85 KB of SASS. Here a second env of the same task and size (the
same specialized module) is stepped after the flush and before the timed step of the first: its launch pulls
the code into L2 and the SMs' instruction caches while the first env's state stays cold. The difference to
the plain protocol bounds what instruction fetch costs the timed step (not a bench mode: diagnosis only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.policies import random_policy  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

n = 4096
a = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n, seed=0), "Velocity-Rough")
b = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n, seed=1), "Velocity-Rough")
for e in (a, b):
    e.reset()
    for i in range(5):
        e.step(random_policy(e, i, fused=True))
assert a._jit_handle == b._jit_handle, "same module expected"
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for rep in range(3):
    for warm in (False, True):
        K = 100
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        torch.cuda.synchronize()
        for i in range(K):
            flush.fill_(float(i))
            if warm:
                b.step(random_policy(b, 100 + rep * K + i, fused=True))
            evs[i][0].record(st)
            a.step(random_policy(a, 100 + rep * 2 * K + i + (K if warm else 0), fused=True))
            evs[i][1].record(st)
            if i >= 2:
                evs[i - 2][1].synchronize()
        torch.cuda.synchronize()
        t = np.array([x.elapsed_time(y) * 1e3 for x, y in evs])
        print(f"rep {rep} {'code warmed by a sibling env' if warm else 'plain protocol         '}: mean {t.mean():.2f} us",
              flush=True)
