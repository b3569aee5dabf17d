# round 2, job 20: J and the status words published by the call's last kernel (mapped memory)
set -x
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j20_trace.log 2>&1
python tools/probe.py e2e > gpurun_out/j20_e2e.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/j20_gpu.log 2>&1; echo gpu_rc=$?
