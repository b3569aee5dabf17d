# round 2, job 4: FD debug at C3, P2P group pairs, slab/AA tests
set -x
python tools/gpu_jobs/fddebug.py > gpurun_out/j4_fddebug.log 2>&1; echo fd_rc=$?
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_aa.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/j4_tests.log 2>&1; echo t_rc=$?
