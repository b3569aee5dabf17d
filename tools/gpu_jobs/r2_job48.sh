# round 2, job 48: FP32 in place at 8 blocks (default now); fused FP32 double-buffered pairs (variants)
set -x
timeout 900 python -m pytest tests/test_gpu_aa.py -m gpu -q -p no:cacheprovider > gpurun_out/j48_tests.log 2>&1; echo rc=$?
python tools/probe.py aa > gpurun_out/j48_main.log 2>&1
python tools/probe.py variants variants model.precision=32 > gpurun_out/j48_var.log 2>&1
