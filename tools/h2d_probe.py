"""Pinned host->device copy bandwidth on this box (development probe): the
e2e step's design upload is bounded by it."""
import torch
for mb in (16, 64, 256):
    n = mb * 2**20 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"H2D {mb} MiB: {ms:.3f} ms = {mb * 2**20 / ms / 1e6:.1f} GB/s")
