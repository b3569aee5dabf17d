#!/usr/bin/env python
"""Development probes on the GPU box (not the bench contract; bench.py is).

  python tools/probe.py rates [C3 overrides key=value ...] [streaming=aa]
      sweep / pair rates of one C3 variant (CUDA events)
  python tools/probe.py geom
      fused-pair rate with and without pressure faces (tags.geometry=periodic)
  python tools/probe.py variants DIR
      `rates` for every variant library DIR/*.so (built by
      `LBGPU_NVCC_EXTRA=-D... LBGPU_BUILD_DIR=... LBGPU_LIB=DIR/x.so builder.py`),
      one subprocess per library
  python tools/probe.py aa
      rates of the double-buffered and the in-place (AA) engines, C3 FP64 / FP32
  python tools/probe.py e2e
      lbgpu_pair_step_with_design rate (with LBGPU_TRACE_PAIR=1 in the
      environment, each call's stage timeline on stderr)
  python tools/probe.py e2e_alt
      the same call alternating with and without J, each call timed (the cost of J)
  python tools/probe.py l2gran
      objective / pair / e2e rates under each cudaLimitMaxL2FetchGranularity
  python tools/probe.py ncu {pair,sweeps,gradient,aa,e2e,sweeps32}
      a short run to put under ncu
"""
from __future__ import annotations

import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _engine(ov: dict | None = None, cfg: str = "C3", streaming: str = "double"):
    import paper_1501_04741_b200 as P
    from paper_1501_04741_b200.presets import config_text
    e = P.Engine.from_config(config_text(cfg, ov or {}), streaming=streaming)
    e.init_state()
    e.primal_step(20, residual=False)
    return e


def rates(ov: dict, K: int = 100, streaming: str = "double") -> dict:
    e = _engine(ov, streaming=streaming)
    s = 8 if e.precision == 64 else 4
    m, n = e.m, e.n
    e.time_pairs(5)
    _, tp, ta = e.time_pairs(K)
    e.time_pair_steps(5)
    tpair = e.time_pair_steps(K)
    e.time_sweeps(1, 5)
    tf = e.time_sweeps(1, K)
    out = {"lib": os.path.basename(os.environ.get("LBGPU_LIB", "liblbgpu.so")), "ov": ov,
           "streaming": streaming,
           "primal_gbs": round(2 * m * s * n * K / tp / 1e6, 1),
           "adjoint_gbs": round(3 * m * s * n * K / ta / 1e6, 1),
           "pair_mlups": round(n * K / tpair / 1e3, 1),
           "pair_gbs": round((4 if s == 8 else 5) * m * s * n * K / tpair / 1e6, 1),
           "frozen_adjoint_mlups": round(n * K / tf / 1e3, 1)}
    e.close()
    return out


def kv(args):
    ov = {}
    for a in args:
        k, v = a.split("=", 1)
        ov[k] = v
    return ov


def main():
    cmd = sys.argv[1] if len(sys.argv) > 1 else "rates"
    if cmd == "rates":  # streaming=aa selects the in-place engine
        ov = kv(sys.argv[2:])
        st = ov.pop("streaming", "double")
        print(json.dumps(rates(ov, streaming=st)), flush=True)
    elif cmd == "geom":
        for ov in ({}, {"tags.geometry": "periodic"}):
            print(json.dumps(rates(ov)), flush=True)
    elif cmd == "variants":
        for lib in sorted(glob.glob(os.path.join(sys.argv[2], "*.so"))):
            env = dict(os.environ, LBGPU_LIB=os.path.abspath(lib))
            subprocess.run([sys.executable, __file__, "rates", *sys.argv[3:]], env=env, check=False)
    elif cmd == "aa":
        for prec in (64, 32):
            for st in ("double", "aa"):
                print(json.dumps(rates({"model.precision": prec}, streaming=st)), flush=True)
    elif cmd == "e2e":
        import time
        import numpy as np
        import torch
        e = _engine()
        w = torch.from_numpy(e.design_values()).pin_memory().numpy()
        for obj in (True, False, True, False, True, False):  # J read back, or not
            for _ in range(40):
                e.pair_step_with_design(w, residual=False, objective=obj)
            e.finish()
            K = 200
            t0 = time.perf_counter()
            for _ in range(K):
                e.pair_step_with_design(w, residual=False, objective=obj)
            e.finish()
            dt = (time.perf_counter() - t0) / K
            print(json.dumps({"objective": obj, "e2e_ms_per_step": dt * 1e3,
                              "e2e_mlups": e.n / dt / 1e6}), flush=True)
    elif cmd == "e2e_alt":  # calls alternating with / without J, each timed (drift cancels)
        import time
        import torch
        e = _engine()
        w = torch.from_numpy(e.design_values()).pin_memory().numpy()
        for _ in range(40):
            e.pair_step_with_design(w, residual=False)
        t = {True: [], False: []}
        for k in range(600):
            obj = k % 2 == 0
            t0 = time.perf_counter()
            e.pair_step_with_design(w, residual=False, objective=obj)
            t[obj].append(time.perf_counter() - t0)
        e.finish()
        import statistics as S
        print(json.dumps({"with_J_us": S.median(t[True]) * 1e6, "without_J_us": S.median(t[False]) * 1e6}),
              flush=True)
    elif cmd == "l2gran":  # cudaLimitMaxL2FetchGranularity vs the objective / pair / e2e
        import ctypes
        import time
        import torch
        torch.cuda.init()
        rt = None
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                rt = ctypes.CDLL(name)
                break
            except OSError:
                pass
        e = _engine()
        w = torch.from_numpy(e.design_values()).pin_memory().numpy()
        for gran in (None, 32, 64, 128):
            if gran is not None:
                r = rt.cudaDeviceSetLimit(0x05, ctypes.c_size_t(gran))
                assert r == 0, r
            v = ctypes.c_size_t(0)
            rt.cudaDeviceGetLimit(ctypes.byref(v), 0x05)
            for _ in range(20):
                e.objective()
            t0 = time.perf_counter()
            for _ in range(200):
                e.objective()
            tobj = (time.perf_counter() - t0) / 200
            e.time_pair_steps(5)
            tpair = e.time_pair_steps(50)
            for _ in range(20):
                e.pair_step_with_design(w, residual=False)
            e.finish()
            t0 = time.perf_counter()
            for _ in range(200):
                e.pair_step_with_design(w, residual=False)
            e.finish()
            dt = (time.perf_counter() - t0) / 200
            print(json.dumps({"gran": v.value, "objective_us": tobj * 1e6,
                              "pair_mlups": e.n * 50 / tpair / 1e3, "e2e_mlups": e.n / dt / 1e6}),
                  flush=True)
    elif cmd == "ncu":
        what = sys.argv[2]
        if what == "pair":
            e = _engine()
            e.pair_steps(4, residual=False)
        elif what == "sweeps":
            e = _engine()
            e.adjoint_step(3, residual=False)
        elif what == "gradient":
            import numpy as np
            e = _engine(cfg="C4")
            e.one_shot(np.full(3, 1e-4), np.zeros(3), record_interval=100)
        elif what == "aa":
            e = _engine(streaming="aa")
            e.pair_steps(4, residual=False)
        elif what == "sweeps32":  # FP32 pairs run as the two sweeps apart
            e = _engine({"model.precision": 32})
            e.pair_steps(4, residual=False)
        elif what == "e2e":
            e = _engine()
            w = e.design_values()
            for _ in range(4):
                e.pair_step_with_design(w, residual=False)
            e.finish()
        print("ok")


if __name__ == "__main__":
    main()
