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
    print(json.dumps({"lib": os.environ.get("LBGPU_LIB", "default"), "prec": prec,
                      "primal_gbs": round(2 * e.m * s * e.n * K / tp / 1e6, 1),
                      "adjoint_gbs": round(3 * e.m * s * e.n * K / ta / 1e6, 1)}))
    e.close()
