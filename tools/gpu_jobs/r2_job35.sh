# round 2, job 35: per-config evidence (C1-C5) on the final build
set -x
timeout 3000 python tools/bench_configs.py r2 > gpurun_out/j35_configs.log 2>&1; echo cfg_rc=$?
cp profiles/r2_configs.json gpurun_out/j35_r2_configs.json
