# round 2, job 45: rematerialised in-place stores (default now) + 4-block variant; AA tests
set -x
timeout 900 python -m pytest tests/test_gpu_aa.py tests/test_gpu_slabs.py -m gpu -q -p no:cacheprovider > gpurun_out/j45_tests.log 2>&1; echo rc=$?
python tools/probe.py aa > gpurun_out/j45_main.log 2>&1
python tools/probe.py variants variants streaming=aa > gpurun_out/j45_m4_64.log 2>&1
python tools/probe.py variants variants streaming=aa model.precision=32 > gpurun_out/j45_m4_32.log 2>&1
