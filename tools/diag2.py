import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1501_04741_b200 as P
from oracle import oracle as O
from cases import case_text
for name in sys.argv[1:]:
    txt = case_text(name)
    e = P.Engine.from_config(txt); o = O.COracle(txt)
    e.init_state(); o.init_state()
    e.primal_step(51); o.primal_steps(51)
    for k in (1, 20):
        e.adjoint_step(k); o.adjoint_steps(k)
        a, b = e.get_state(1), o.v
        d = np.abs(a - b); sc = np.abs(b).max()
        order = np.argsort(-d)[:8]
        t = e.tables()["tag"]
        print(name, "adj+", k, "maxrel", d.max() / sc, "scale", sc)
        for i in order:
            p, node = divmod(int(i), e.n)
            x = node % e.shape[0]; y = (node // e.shape[0]) % e.shape[1]
            print(f"   p={p} ({x},{y}) tag={t[node]} gpu={a[i]:.17g} ora={b[i]:.17g} d={d[i]:.3e}")
