# round 2, job 56: DRAM bytes of the fused pair at the C5 slab's shape vs C3
set -x
cat > /tmp/p.py <<'PY'
import sys
sys.path.insert(0, '.')
import tools.probe as T
ov = {} if sys.argv[1] == 'c3' else {"lattice.nx": "256", "lattice.ny": "512", "lattice.nz": "512", "tags.design_x0": "64", "tags.design_x1": "191"}
e = T._engine(ov)
e.pair_steps(4, residual=False)
print("ok")
PY
for w in c3 big; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_pair -s 2 -c 1 --csv --log-file gpurun_out/j56_$w.csv python /tmp/p.py $w > gpurun_out/j56_$w.log 2>&1; echo rc=$?
done
