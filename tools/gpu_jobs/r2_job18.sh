# round 2, job 18: e2e with and without J; deferred-pair tests
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "deferred" > gpurun_out/j18_tests.log 2>&1; echo rc=$?
python tools/probe.py e2e > gpurun_out/j18_e2e.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j18_trace.log 2>&1
