"""Pinned H2D rate of the 16 MB design vector against the NUMA placement of
the host buffer: the allocating thread pinned to each node's CPUs in turn
(development probe)."""
import os
import glob
import torch
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
def cpus_of(nd):
    out = []
    for part in open(nd + "/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out
print("cpus", os.cpu_count(), "nodes", [(os.path.basename(n), cpus_of(n)) for n in nodes])
try:
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("gpu0 numa", open(f"/sys/bus/pci/devices/{pynvml.nvmlDeviceGetPciInfo(hd).busId.lower()[4:]}/numa_node").read().strip()
          if True else "")
except Exception as ex:  # noqa
    print("nvml", ex)
n = 16257024 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
all_cpus = os.sched_getaffinity(0)
for nd in nodes:
    cp = cpus_of(nd)
    if not cp:
        continue
    os.sched_setaffinity(0, cp)
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    h.fill_(1.0)
    for placement in ("same", "all"):
        os.sched_setaffinity(0, cp if placement == "same" else all_cpus)
        ts = []
        for _ in range(12):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts = sorted(ts)[2:-2]
        ms = sum(ts) / len(ts)
        print(f"{os.path.basename(nd)} buffer, thread {placement}: {ms:.3f} ms = {n*8/ms/1e6:.1f} GB/s", flush=True)
    os.sched_setaffinity(0, all_cpus)
