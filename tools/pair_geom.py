"""Fused-pair rate at C3 with and without pressure faces (tags.geometry =
periodic: no inlet/outlet lanes) — is the face path what holds k_pair back?
(development probe)"""
import sys
sys.path.insert(0, "/root/repo")
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

for ov in ({}, {"tags.geometry": "periodic"}):
    e = P.Engine.from_config(config_text("C3", ov))
    e.init_state()
    e.primal_step(20, residual=False)
    e.time_pair_steps(5)
    K = 100
    ms = e.time_pair_steps(K)
    t, tp, ta = e.time_pairs(K)
    print(ov, "pair fused MLUPS", round(e.n * K / ms / 1e3), "GB/s", round(832 * e.n * K / ms / 1e6),
          "| primal GB/s", round(416 * e.n * K / tp / 1e6), "adjoint GB/s", round(624 * e.n * K / ta / 1e6), flush=True)
    e.close()
