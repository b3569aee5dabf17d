# round 2, job 51: per-config evidence refreshed on the final build (C3, C4, C5)
set -x
timeout 3000 python tools/bench_configs.py r2 C3 C4 C5 > gpurun_out/j51_configs.log 2>&1; echo cfg_rc=$?
cp profiles/r2_configs.json gpurun_out/j51_r2_configs.json
