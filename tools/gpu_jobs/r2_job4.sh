# round 2, job 4: FD debug at C3, P2P group pairs, slab/AA tests
set -x
# (a one-off FD debug script ran here; removed since: tests/test_gpu_fdcheck.py covers it)
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_aa.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/j4_tests.log 2>&1; echo t_rc=$?
