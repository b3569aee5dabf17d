"""Per-copy times of back-to-back 16 MB pinned H2D copies after nothing, a
spin kernel, or an HBM kernel on another stream (development probe)."""
import torch
n = 16257024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
big = torch.empty(2**28, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
def run(mode, k=6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
    torch.cuda.synchronize()
    if mode == "sleep":
        torch.cuda._sleep(4_000_000)
    elif mode == "hbm":
        big.mul_(1.0000001)
    with torch.cuda.stream(s):
        ev[0].record(s)
        for i in range(k):
            d.copy_(h, non_blocking=True)
            ev[i + 1].record(s)
    torch.cuda.synchronize()
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(k)]
    print(f"{mode:6s}: " + " ".join(f"{t:.3f}" for t in ts), flush=True)
for m in ("idle", "sleep", "hbm") * 2:
    run(m)
