"""A short C3 sweep run to put under ncu (development tool).

  python tools/ncu_target.py [precision] [extra key=value ...]
"""
import sys

sys.path.insert(0, "/root/repo")
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ov = {"model.precision": prec}
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    ov[k] = v
e = P.Engine.from_config(config_text("C3", ov))
e.init_state()
e.primal_step(3, residual=False)
e.adjoint_step(3, residual=False)
print("ok")
