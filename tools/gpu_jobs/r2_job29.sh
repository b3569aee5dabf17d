# round 2, job 29: e2e with / without J, alternating; the reference arm
set -x
python tools/probe.py e2e > gpurun_out/j29_e2e.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/j29_ref.log 2>&1; echo ref_rc=$?
