# round 2, job 22: FP32 frozen-base adjoint with v gathered first; parity + in-place tests
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_aa.py -m gpu -q -p no:cacheprovider > gpurun_out/j22_tests.log 2>&1; echo rc=$?
python tools/probe.py aa > gpurun_out/j22_aa.log 2>&1
