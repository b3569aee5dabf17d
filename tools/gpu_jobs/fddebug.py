import sys, numpy as np
sys.path.insert(0, '.')
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text
txt = config_text("C3", {"tags.inlet_profile": "uniform", "tags.inlet_T": 0.0})
e = P.Engine.from_config(txt)
e.init_state(); e.primal_step(1000, residual=False)
f_w = e.get_state(0)
N = 200
J, g, gdp, fs = e.unsteady_adjoint(N, sum_objective=False, slots=16)
print("J", J, "gdp", gdp, "fsweeps", fs, "max|g|", np.abs(g).max())
e.set_state(0, f_w)
order = sorted(range(g.size), key=lambda i: (-abs(g[i]), i))[:6]
ords = [o for o in order for _ in (1e-5, 1e-6)] + [-1, -1]
hs = [1e-5, 1e-6] * (len(order) + 1)
fd = e.fd_gradient_batch(ords, hs, fixed_iters=N, from_state=True)
for k, (o, h) in enumerate(zip(ords, hs)):
    print(o, h, "adj", gdp if o < 0 else g[o], "fd", fd[k])
e.set_state(0, f_w)
print("single", e.fd_gradient(order[0], 1e-5, 0.0, N, fixed_iters=N))
# J by direct runs
e.set_state(0, f_w); e.primal_step(N, residual=False); print("J direct", e.objective())
