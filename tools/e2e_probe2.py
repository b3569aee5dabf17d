"""The e2e step's upload in context: torch's own pinned copy of the same host
buffer vs the engine's set_design_values, interleaved with sweeps
(development probe)."""
import sys
import time
sys.path.insert(0, "/root/repo")
import torch
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

e = P.Engine.from_config(config_text("C3"))
e.init_state()
e.primal_step(20, residual=False)
wt = torch.from_numpy(e.design_values()).pin_memory()
w = wt.numpy()
dd = torch.empty_like(wt, device="cuda")
K = 30


def t(name, fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    torch.cuda.synchronize()
    print(f"{name:44s} {(time.perf_counter() - t0) / K * 1e3:.3f} ms", flush=True)


def tcopy():
    dd.copy_(wt, non_blocking=True)
    torch.cuda.synchronize()


for _ in range(2):
    t("torch copy of w (sync)", tcopy)
    t("set_design_values", lambda: e.set_design_values(w))
    t("torch copy + primal_step", lambda: (tcopy(), e.primal_step(1, residual=False)))
    t("torch copy + primal + adjoint", lambda: (tcopy(), e.primal_step(1, residual=False),
                                                 e.adjoint_step(1, residual=False)))
    t("pair_step_with_design (J)", lambda: e.pair_step_with_design(w, residual=False))
    t("primal_step_with_design", lambda: e.primal_step_with_design(w, 1, residual=False))
