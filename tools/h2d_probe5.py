"""Is the pinned H2D rate tied to the host buffer being freshly written by
the CPU? (development probe)"""
import time
import torch
n = 16257024 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
def one(buf):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); d.copy_(buf, non_blocking=True); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)
for rnd in range(3):
    h.fill_(1.0 + rnd)
    r1 = [one(h) for _ in range(8)]
    r2 = []
    for k in range(8):
        h.fill_(float(k)); r2.append(one(h))
    t0 = time.perf_counter(); h2.copy_(h); t1 = time.perf_counter()
    r3 = [one(h2) for _ in range(4)]
    time.sleep(0.05)
    r4 = [one(h) for _ in range(4)]
    f = lambda r: " ".join(f"{x:.2f}" for x in r)
    print(f"no-write: {f(r1)}\nwrite-each: {f(r2)}\nfresh copy ({(t1-t0)*1e3:.1f} ms host): {f(r3)}\nafter 50ms sleep: {f(r4)}", flush=True)
