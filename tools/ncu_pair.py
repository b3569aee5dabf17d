"""A short C3 fused-pair run to put under ncu (development tool)."""
import sys

sys.path.insert(0, "/root/repo")
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

e = P.Engine.from_config(config_text("C3"))
e.init_state()
e.primal_step(3, residual=False)
e.pair_steps(4, residual=False)
print("ok")
