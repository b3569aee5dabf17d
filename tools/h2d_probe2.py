"""H2D of the C3 design vector (16 MB) in 1 / 8 / 32 chunks, alone and under a
running HBM-bound kernel (development probe)."""
import torch
n = 16257024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
big = torch.empty(2**28, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
def run(chunks, busy):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if busy:
        big.mul_(1.0000001)  # ~2 GB r+w on the default stream
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(10):
            for c in range(chunks):
                lo, hi = n * c // chunks, n * (c + 1) // chunks
                d[lo:hi].copy_(h[lo:hi], non_blocking=True)
        b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"chunks={chunks:3d} busy={busy}: {ms:.3f} ms = {n * 8 / ms / 1e6:.1f} GB/s", flush=True)
for busy in (False, True):
    for ch in (1, 8, 32):
        run(ch, busy); run(ch, busy)
