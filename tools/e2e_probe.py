"""Breakdown of bench.py's e2e step (development probe)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

e = P.Engine.from_config(config_text("C3"))
e.init_state()
e.primal_step(20, residual=False)
w = torch.from_numpy(e.design_values()).pin_memory().numpy()
K = 50


def t(name, fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t0) / K * 1e3:.3f} ms", flush=True)


t("primal_step(1)", lambda: e.primal_step(1))
t("primal_step(1) no resid", lambda: e.primal_step(1, residual=False))
t("adjoint_step(1)", lambda: e.adjoint_step(1))
t("set_design_values", lambda: e.set_design_values(w))
t("set_design_values + primal_step", lambda: (e.set_design_values(w), e.primal_step(1)))
t("primal_step_with_design", lambda: e.primal_step_with_design(w, 1))
t("adjoint_step(1) no resid", lambda: e.adjoint_step(1, residual=False))
t("objective", lambda: e.objective())
t("e2e step (residuals)", lambda: (e.primal_step_with_design(w, 1), e.adjoint_step(1)))
t("e2e step (J)", lambda: (e.primal_step_with_design(w, 1, residual=False),
                           e.adjoint_step(1, residual=False), e.objective()))
t("pair_step_with_design (J)", lambda: e.pair_step_with_design(w, residual=False))
t("pair_step_with_design (no J)", lambda: e.pair_step_with_design(w, residual=False, objective=False))
t("primal+adjoint no design", lambda: (e.primal_step(1, residual=False), e.adjoint_step(1, residual=False)))
