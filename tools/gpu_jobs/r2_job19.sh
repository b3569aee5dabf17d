# round 2, job 19: e2e host/GPU timeline (LBGPU_TRACE_PAIR with host clocks)
set -x
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j19_trace.log 2>&1
python tools/probe.py e2e > gpurun_out/j19_e2e.log 2>&1
