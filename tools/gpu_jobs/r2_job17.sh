# round 2, job 17: in-place tests (incl. C3 size), FP32 in-place bounds 4/6, FP32 adjoint variants
set -x
timeout 900 python -m pytest tests/test_gpu_aa.py -m gpu -q -p no:cacheprovider > gpurun_out/j17_aa_tests.log 2>&1; echo aa_rc=$?
python tools/probe.py aa > gpurun_out/j17_aa.log 2>&1
python tools/probe.py variants variants model.precision=32 > gpurun_out/j17_var32.log 2>&1
