"""Stage timeline of lbgpu_pair_step_with_design at C3 (LBGPU_TRACE_PAIR=1;
development probe)."""
import os
import sys
os.environ["LBGPU_TRACE_PAIR"] = "1"
sys.path.insert(0, "/root/repo")
import torch
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

e = P.Engine.from_config(config_text("C3"))
e.init_state()
e.primal_step(20, residual=False)
w = torch.from_numpy(e.design_values()).pin_memory().numpy()
for _ in range(6):
    e.pair_step_with_design(w, residual=False)
