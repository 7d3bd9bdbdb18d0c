"""Back-to-back D2H copies of one output arena (1.58 MB) on a side stream: plain, with an event per copy,
with host syncs lagging 3 / 8 copies, with a cross-stream wait -- all ~31.3 us per copy (the pipe's floor)."""
import time, torch
nb = 1581056
K = 300
s = torch.cuda.Stream()
src = torch.empty(nb, dtype=torch.uint8, device="cuda")
hosts = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(5)]
def run(name, rec, sync_lag, wait_ev=False):
    evs = []
    other = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        if wait_ev:
            e0 = torch.cuda.Event(); e0.record(other); s.wait_event(e0)
        with torch.cuda.stream(s):
            hosts[i % 5].copy_(src, non_blocking=True)
            if rec:
                e = torch.cuda.Event(); e.record(s); evs.append(e)
        if sync_lag and i >= sync_lag:
            evs[i - sync_lag].synchronize()
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
    print(f"{name}: {tt / K * 1e6:.1f} us/copy", flush=True)
for r in range(2):
    run("plain", False, 0)
    run("event per copy", True, 0)
    run("event + sync lag 3", True, 3)
    run("event + sync lag 8", True, 8)
    run("wait_event + event + lag 3", True, 3, True)
