"""Sweep timing experiments (not part of the bench contract)."""
import sys, json
sys.path.insert(0, "/root/repo")
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text
variants = {
    "C3": {},
    "C3-periodic": {"tags.geometry": "periodic", "objective.kind": "mixing"},
    "C3-bgk": {"model.collision": "bgk"},
    "C3-fp32": {"model.precision": 32},
    "C1": None, "C2": None, "C4": None,
}
for name, ov in variants.items():
    txt = config_text(name if ov is None else "C3", ov or {})
    e = P.Engine.from_config(txt)
    e.init_state(); e.primal_step(20, residual=False)
    e.time_pairs(5)
    K = 50 if e.n > 1e6 else 400
    t, tp, ta = e.time_pairs(K)
    s = 8 if e.precision == 64 else 4
    bp, ba = 2 * e.m * s, 3 * e.m * s
    print(json.dumps({"case": name, "nodes": e.n, "primal_mlups": round(e.n*K/tp/1e3, 1), "adjoint_mlups": round(e.n*K/ta/1e3, 1),
                      "primal_gbs": round(bp*e.n*K/tp/1e6, 1), "adjoint_gbs": round(ba*e.n*K/ta/1e6, 1)}))
    e.close()
