#!/usr/bin/env python
"""Benchmark: LBM primal + discrete-adjoint sweep throughput on B200.

Metric (BASELINE.json): MLUPS of the primal and adjoint sweeps, with the
achieved HBM GB/s against the measured peak. One "step" = one primal sweep
(primal_step, collision.cpp:308-363) followed by one adjoint sweep against the
new state (adjoint_step, adjoint.cpp:206-254) over the whole lattice of
BASELINE config C3 (mixer3d preset at 256x128x128: D3Q19 flow + D3Q7
temperature, FMRT, FP64, 4,194,304 nodes per GPU). value = lattice node
updates of the step pair per second, i.e. nodes*K/T in millions.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): every rank owns one C3-sized x-slab of
the mixer3d lattice N times as long, (256 N) x 128 x 128 with the design span
scaled alike (weak scaling): decompose's x-slabs, halos over
NCCL (boundary columns first, the exchange overlapped with the interior
columns), residuals reduced across ranks.

Timing: W untimed step pairs, then exactly K timed pairs bracketed by a
barrier and device synchronisation, CUDA events on the engine's stream
(between every sweep, so the primal and adjoint shares are measured in the
same region), max over ranks. Each sweep streams 2x872 MB (primal) / 3x872 MB
(adjoint) at FP64 — far more than the 126 MB L2, so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_ID = "C3"
WORKLOAD = (f"{CONFIG_ID}: mixer3d preset 256x128x128 per GPU, D3Q19+D3Q7 FMRT, "
            "primal sweep + adjoint sweep per step")
BYTES_PRIMAL = lambda m, s: 2 * m * s  # SURVEY.md §8(d) canonical bytes / LUP
BYTES_ADJOINT = lambda m, s: 3 * m * s
BYTES_PAIR = lambda m, s: 4 * m * s  # fused adjoint k + primal k+1: f read once


def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, local_rank: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = vis.split(",")[local_rank] if vis else str(local_rank)
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.cmd = ["nvidia-smi", "-i", idx, f"--query-gpu={self.FIELDS}",
                    "--format=csv,noheader,nounits", "-lms", "20"]
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(self.cmd, stdout=self.tmp, stderr=subprocess.DEVNULL)
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        self.tmp.flush()
        self.tmp.seek(0)
        rows = [r.split(", ") for r in self.tmp.read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for name, flag in zip(names, r[4:8]):
                if flag.strip().lower() in ("active", "1"):
                    reasons.add(name)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(cfg_text: str, nodes: int) -> dict:
    """The reference itself (oracle/_ref: compiled from its own sources) on this
    box's host cores: one primal + one adjoint sweep of the same C3 lattice
    through its thread-per-slab PartitionedRun (partition.cpp:93-188) with all
    host threads."""
    from oracle import oracle as O
    cores = len(os.sched_getaffinity(0))
    r = O.RefOracle(cfg_text)
    r.init_state()
    tp = r.time_steps(0, cores, 1)
    ta = r.time_steps(1, cores, 1)
    r.close()
    return {"value": nodes / (tp + ta) / 1e6, "unit": "MLUPS", "cores": cores,
            "kind": "reference",
            "sample": f"1 primal + 1 adjoint sweep of the full {CONFIG_ID} lattice "
                      f"({nodes} nodes, FP64) via PartitionedRun x{cores} threads",
            "primal_mlups": nodes / tp / 1e6, "adjoint_mlups": nodes / ta / 1e6}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    from paper_1501_04741_b200.presets import config_text
    from oracle import oracle as O
    txt = config_text(CONFIG_ID)
    cores = len(os.sched_getaffinity(0))
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    r = O.RefOracle(txt)
    nodes = r.n
    r.init_state()
    # bounded CPU sample: <= 3 warm-up and <= 3 timed pairs (~0.8 s each at C3)
    warm, steps = min(max(args.warmup, 3), 3), max(1, min(args.steps, 3))
    for _ in range(warm):
        r.time_steps(0, cores, 1)
        r.time_steps(1, cores, 1)
    tp = sum(r.time_steps(0, cores, 1) for _ in range(steps))
    ta = sum(r.time_steps(1, cores, 1) for _ in range(steps))
    value = nodes * steps / (tp + ta) / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MLUPS",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": (tp + ta) / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": nodes},
        "primal_mlups": nodes * steps / tp / 1e6, "adjoint_mlups": nodes * steps / ta / 1e6,
        "cpu_baseline": {"value": value, "unit": "MLUPS", "cores": cores, "kind": "reference",
                         "sample": f"{steps} primal+adjoint sweep pairs of the full lattice, "
                                   f"PartitionedRun x{cores} threads"},
        "e2e": {"value": value, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


METRIC = "MLUPS primal & adjoint at 1/2/4/8 B200; achieved HBM GB/s vs peak"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.impl == "reference":
        run_reference(args, rank)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import numpy as np
    import torch

    import paper_1501_04741_b200 as P
    from paper_1501_04741_b200.presets import config_text

    if world == 1:
        txt = config_text(CONFIG_ID)
        eng = P.Engine.from_config(txt, device=local)
        nodes = eng.n
    else:
        txt = config_text(CONFIG_ID, {"lattice.nx": 256 * world, "tags.design_x0": 64 * world,
                                      "tags.design_x1": 192 * world - 1})
        eng = P.Engine.slab_from_config(txt, None, world, rank, device=local)
        uid = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.attach_nccl(uid[0], world, rank)
        sl = eng.slab()
        nodes = sl["span"] * eng.shape[1] * eng.shape[2]  # owned nodes of this rank
    m, s = eng.m, 8 if eng.precision == 64 else 4
    eng.init_state()
    # develop a non-trivial flow before timing (the pressure wave enters)
    eng.primal_step(20, residual=False)
    fused = eng.precision == 64  # lbgpu_pair_steps fuses adjoint k + primal k+1 at FP64
    eng.time_pair_steps(args.warmup)
    eng.time_pairs(args.warmup)

    def barrier():
        torch.cuda.synchronize(local)
        if dist:
            dist.barrier()

    def max_over_ranks(*vals):
        if not dist:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return tuple(t.tolist())

    # the headline: K steps of primal sweep + adjoint sweep through
    # lbgpu_pair_steps (one fused k_pair launch per step at FP64)
    barrier()
    launches0 = eng.sweep_launches()
    with ClockSampler(local) as clk:
        ms_tot = eng.time_pair_steps(args.steps)
    barrier()
    launches = eng.sweep_launches() - launches0
    (ms_tot,) = max_over_ranks(ms_tot)
    # explanation: the two sweeps apart, CUDA events between every sweep
    barrier()
    _, ms_p, ms_a = eng.time_pairs(args.steps)
    barrier()
    # the fused sweep alone (roofline of the dominant kernel)
    ms_k = eng.time_sweeps(2, args.steps) if fused else None
    barrier()
    ms_p, ms_a = max_over_ranks(ms_p, ms_a)
    if ms_k is not None:
        (ms_k,) = max_over_ranks(ms_k)
    # SURVEY.md §8d C3 protocol for the adjoint alone: the base frozen (the
    # steady solve_adjoint path, moment cache built once inside the timing)
    eng.time_sweeps(1, args.warmup)
    barrier()
    ms_f = eng.time_sweeps(1, args.steps)
    barrier()
    (ms_f,) = max_over_ranks(ms_f)
    K = args.steps
    value = world * nodes * K / (ms_tot / 1e3) / 1e6
    primal_mlups = world * nodes * K / (ms_p / 1e3) / 1e6
    adjoint_mlups = world * nodes * K / (ms_a / 1e3) / 1e6
    pk = peaks()
    bp, ba = BYTES_PRIMAL(m, s), BYTES_ADJOINT(m, s)
    bk = BYTES_PAIR(m, s)
    ach_a = ba * nodes / (ms_a / K / 1e3) / 1e9  # per-GPU GB/s, adjoint sweep alone
    ach_p = bp * nodes / (ms_p / K / 1e3) / 1e9
    ach_k = bk * nodes / (ms_k / K / 1e3) / 1e9 if ms_k else None

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        traffic = tj.get("pair_bytes_per_launch" if fused else "adjoint_bytes_per_launch")

    # e2e through the public C ABI with host buffers: each step uploads the
    # design vector (DesignField::nodes order, as a host-side optimizer such as
    # the reference's MMA update produces it, optimizer.cpp:200-202) from
    # pinned host memory, runs one primal sweep, then one adjoint sweep
    # against the new state (optimizer.cpp:33-34), and reads the step's
    # result, the objective J of the new state (evaluate_raw), back to the
    # host — one call, lbgpu_pair_step_with_design, which overlaps the upload,
    # the primal z-chunks and the adjoint z-chunks. Like the reference's
    # one-shot loop the sweeps skip the optional step_residual; the call still
    # returns its status (the rho <= 0 check) synchronously. The same step as
    # three calls (primal_step_with_design + adjoint_step + objective) is
    # reported beside it.
    w_host = torch.from_numpy(eng.design_values()).pin_memory()
    w_np = w_host.numpy()
    eng.set_design_values(w_np)

    def e2e_step():
        return eng.pair_step_with_design(w_np, residual=False)[2]

    def e2e_step_apart():
        eng.primal_step_with_design(w_np, 1, residual=False)
        eng.adjoint_step(1, residual=False)
        return eng.objective()

    def e2e_time(fn):
        # untimed warm-up, at least 30 steps: pinned H2D on these boxes runs at
        # 10-20 GB/s for a while after the copy engine idles (tools/h2d_probe5.py)
        # and at 48-54 GB/s once copies stream back to back
        for _ in range(max(args.warmup, 30)):
            fn()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            fn()
        torch.cuda.synchronize(local)
        s_ = time.perf_counter() - t0
        if dist:
            t = torch.tensor([s_], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s_ = t.item()
        return world * nodes * args.e2e_steps / s_ / 1e6

    e2e_apart = e2e_time(e2e_step_apart)
    e2e = {"value": e2e_time(e2e_step), "unit": "MLUPS",
           # J (8 B) + the call's status words (4 x 8 B)
           "h2d_bytes_per_step": int(8 * eng.n_design), "d2h_bytes_per_step": 8 + 32,
           "steps": args.e2e_steps,
           "path": "lbgpu_pair_step_with_design(pinned host w; J to the host)",
           "three_calls_mlups": e2e_apart}

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(txt, nodes)
        except Exception as exc:  # reported, never silently substituted
            cpu = {"error": str(exc)}

    line = {
        "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_tot / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD,
                   "path": "lbgpu_pair_steps: adjoint sweep k fused with primal sweep k+1 "
                           "(k_pair) at FP64",
                   "nodes_per_gpu": nodes,
                   "parallelism": (f"{world} x-slabs of a ({256 * world})x128x128 lattice, NCCL halo "
                                   "exchange overlapped with interior columns") if world > 1 else "1 GPU",
                   "l2": "no flush: each sweep streams >= 1.7 GB, 14x the 126 MB L2"},
        "primal_mlups": primal_mlups, "adjoint_mlups": adjoint_mlups,
        "primal_hbm_gbs": ach_p, "adjoint_hbm_gbs": ach_a,
        "adjoint_frozen_base_mlups": world * nodes * K / (ms_f / 1e3) / 1e6,
        "roofline": ({"bound": "hbm", "kernel": "k_pair (fused adjoint k + primal k+1, FMRT, FP64)",
                      "achieved": ach_k, "peak": pk["hbm_gbs"], "unit": "GB/s",
                      "frac": ach_k / pk["hbm_gbs"], "traffic": traffic,
                      "bytes_per_lup": bk, "peak_source": pk["source"],
                      "share_of_step": (ms_k / K) / (ms_tot / K)} if fused else
                     {"bound": "hbm", "kernel": "k_adjoint", "achieved": ach_a,
                      "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach_a / pk["hbm_gbs"],
                      "traffic": traffic, "bytes_per_lup": ba, "peak_source": pk["source"]}),
        "sweeps_apart": {"primal": {"mlups": primal_mlups, "achieved": ach_p,
                                    "frac": ach_p / pk["hbm_gbs"], "bytes_per_lup": bp},
                         "adjoint": {"mlups": adjoint_mlups, "achieved": ach_a,
                                     "frac": ach_a / pk["hbm_gbs"], "bytes_per_lup": ba},
                         "pair_mlups": world * nodes / ((ms_p + ms_a) / K / 1e3) / 1e6},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
