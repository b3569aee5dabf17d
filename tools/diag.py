"""Ad-hoc GPU-vs-oracle diagnostics (prints where states first differ)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1501_04741_b200 as P
from oracle import oracle as O
from cases import case_text

def where(a, b, m, n, shape):
    d = np.abs(a - b)
    idx = np.argwhere(d > 0).ravel()
    if idx.size == 0:
        return "equal"
    out = []
    for i in idx[:6]:
        p, node = divmod(int(i), n)
        x = node % shape[0]; y = (node // shape[0]) % shape[1]; z = node // (shape[0] * shape[1])
        out.append(f"p={p} ({x},{y},{z}) gpu={a[i]!r} ora={b[i]!r}")
    return f"{idx.size} diffs, max {d.max():.3e}; " + "; ".join(out)

for name in sys.argv[1:] or ["grad2d", "bgk2d", "mix3d"]:
    for exact in (True, False):
        txt = case_text(name)
        e = P.Engine.from_config(txt, exact=exact); o = O.COracle(txt)
        e.init_state(); o.init_state()
        print(name, "exact" if exact else "fast", "init:", where(e.get_state(0), o.f, e.m, e.n, e.shape))
        e.primal_step(1); o.primal_steps(1)
        print("  primal1:", where(e.get_state(0), o.f, e.m, e.n, e.shape))
        e.primal_step(5); o.primal_steps(5)
        print("  primal6:", where(e.get_state(0), o.f, e.m, e.n, e.shape))
        e.adjoint_step(1); o.adjoint_steps(1)
        print("  adj1:", where(e.get_state(1), o.v, e.m, e.n, e.shape))
