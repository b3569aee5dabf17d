# round 2, job 57: clocks and power during 100 back-to-back pairs at the C5 slab's shape and at C3
set -x
cat > /tmp/clk.py <<'PY'
import sys, json
sys.path.insert(0, '.')
import tools.probe as T
from bench import ClockSampler
big = sys.argv[1] == 'big'
ov = {"lattice.nx": "256", "lattice.ny": "512", "lattice.nz": "512", "tags.design_x0": "64", "tags.design_x1": "191"} if big else {}
e = T._engine(ov)
e.time_pair_steps(5)
K = 100 if big else 1600
with ClockSampler(0) as c:
    ms = e.time_pair_steps(K)
s = c.summary()
c.tmp.seek(0)
rows = [r.split(", ") for r in c.tmp.read().strip().splitlines()]
pw = [float(r[2]) for r in rows if len(r) > 2 and r[2].replace('.', '', 1).isdigit()]
print(json.dumps({"shape": sys.argv[1], "ms_per_pair": ms / K, "mlups": e.n * K / ms / 1e3, "clocks": s, "power_w_max": max(pw) if pw else None, "power_w_median": sorted(pw)[len(pw)//2] if pw else None}))
PY
python /tmp/clk.py big > gpurun_out/j57_big.log 2>&1
python /tmp/clk.py c3 > gpurun_out/j57_c3.log 2>&1
