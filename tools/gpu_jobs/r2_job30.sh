# round 2, job 30: cost of J inside the design pair call (alternating calls)
python tools/probe.py e2e_alt > gpurun_out/j30.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e_alt > gpurun_out/j30_trace.log 2>&1
