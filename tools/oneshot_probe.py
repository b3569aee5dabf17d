"""C4 one-shot iteration breakdown (development probe): per-iteration time of
lbgpu_one_shot at C4 next to the primal+adjoint pair; run under
`ncu --metrics gpu__time_duration.sum` for the per-kernel split."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1501_04741_b200 as P
from paper_1501_04741_b200.presets import config_text

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
e = P.Engine.from_config(config_text("C4", {"optimizer.zeta_stages": "0:0.0001"}))
e.init_state()
e.one_shot(np.full(5, 1e-4), np.zeros(5), record_interval=100)
t0 = time.perf_counter()
e.one_shot(np.full(K, 1e-4), np.zeros(K), record_interval=K)
dt = (time.perf_counter() - t0) / K
t, tp, ta = e.time_pairs(K)
print(f"one-shot {dt*1e3:.3f} ms/it   pair {t/K:.3f} ms (primal {tp/K:.3f} adjoint {ta/K:.3f})  "
      f"design nodes {e.design_values().size}")
