# round 2, job 15: FP32 in-place register bounds (primal 4/6/8, adjoint 4/5/6 blocks per SM)
set -x
python tools/probe.py variants variants streaming=aa model.precision=32 > gpurun_out/j15_var32.log 2>&1
