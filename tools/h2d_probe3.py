"""Does any SM activity lift the idle-GPU H2D rate? 16 MB pinned H2D alone,
beside torch.cuda._sleep (one spinning thread), and beside an HBM kernel
(development probe)."""
import torch
n = 16257024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
big = torch.empty(2**28, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
def run(mode):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(10):
        torch.cuda.synchronize()
        if mode == "sleep":
            torch.cuda._sleep(2_000_000)  # ~1 ms at 1.965 GHz
        elif mode == "hbm":
            big.mul_(1.0000001)
        with torch.cuda.stream(s):
            a.record(s)
            d.copy_(h, non_blocking=True)
            b.record(s)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / 10
    print(f"{mode:6s}: {ms:.3f} ms = {n * 8 / ms / 1e6:.1f} GB/s", flush=True)
for m in ("idle", "sleep", "hbm", "idle", "sleep", "hbm"):
    run(m)
