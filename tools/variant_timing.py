"""Sweep rates of C3 (FP64 and FP32) for the library named by LBGPU_LIB
(development tool for build-knob sweeps)."""
import json
import os
import sys

sys.path.insert(0, "/root/repo")
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

precs = [int(p) for p in (sys.argv[1:] or ["64", "32"])]
for prec in precs:
    e = P.Engine.from_config(config_text("C3", {"model.precision": prec}))
    e.init_state()
    e.primal_step(20, residual=False)
    e.time_pairs(5)
    K = 100
    t, tp, ta = e.time_pairs(K)
    s = prec // 8
    e.adjoint_step(10, residual=False)
    import torch
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    e.adjoint_step(K, residual=False)
    tf = (time.perf_counter() - t0) * 1e3
    e.time_pair_steps(5)
    tpair = e.time_pair_steps(K)
    print(json.dumps({"lib": os.environ.get("LBGPU_LIB", "default"), "prec": prec,
                      "pair_mlups_separate": round(e.n * K / t / 1e3, 1),
                      "pair_mlups_fused": round(e.n * K / tpair / 1e3, 1),
                      "fused_pair_gbs": round(4 * e.m * s * e.n * K / tpair / 1e6, 1),
                      "primal_gbs": round(2 * e.m * s * e.n * K / tp / 1e6, 1),
                      "adjoint_gbs": round(3 * e.m * s * e.n * K / ta / 1e6, 1),
                      "adjoint_mlups": round(e.n * K / ta / 1e3, 1),
                      "frozen_base_adjoint_mlups": round(e.n * K / tf / 1e3, 1),
                      "frozen_base_adjoint_gbs": round((2 * e.m + 5) * s * e.n * K / tf / 1e6, 1)}))
    e.close()
