# round 2, job 40: slab boundary strips (32 coalesced columns) instead of boundary-column kernels
set -x
timeout 1800 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_aa.py -m gpu -q -p no:cacheprovider > gpurun_out/j40_tests.log 2>&1; echo rc=$?
LBGPU_BENCH_SLAB_RING=1 timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 10 --workload C3 > gpurun_out/j40_ring_c3.log 2>&1; echo c3_rc=$?
LBGPU_BENCH_SLAB_RING=1 timeout 1200 python bench.py --steps 5 --warmup 3 --e2e-steps 5 --workload C5 > gpurun_out/j40_ring_c5.log 2>&1; echo c5_rc=$?
