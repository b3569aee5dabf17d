# round 2, job 21: FP32 adjoint with v gathered before the base (5/6/8 blocks per SM)
set -x
python tools/probe.py rates model.precision=32 > gpurun_out/j21_main32.log 2>&1
python tools/probe.py variants variants model.precision=32 > gpurun_out/j21_var32.log 2>&1
