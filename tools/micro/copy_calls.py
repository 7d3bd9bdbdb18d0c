import time, torch
nb = 1581056
src = torch.empty(nb, dtype=torch.uint8, device="cuda")
dev = torch.empty(nb, dtype=torch.uint8, device="cuda")
host = torch.empty(nb, dtype=torch.uint8).pin_memory()
cs = torch.cuda.Stream()
ev = torch.cuda.Event(); ev2 = torch.cuda.Event()
main = torch.cuda.current_stream()
def t(label, fn, K=300):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: host {(t1-t0)/K*1e6:.1f} us, wall {(t2-t0)/K*1e6:.1f} us", flush=True)
t("D2D copy_", lambda: dev.copy_(src, non_blocking=True))
t("D2H copy_ (main)", lambda: host.copy_(dev, non_blocking=True))
def f():
    with torch.cuda.stream(cs):
        host.copy_(dev, non_blocking=True)
t("D2H copy_ in stream ctx", f)
t("event record", lambda: ev.record(main))
t("wait_event", lambda: cs.wait_event(ev))
t("stream ctx only", lambda: torch.cuda.stream(cs).__enter__() or torch.cuda.set_stream(main))
