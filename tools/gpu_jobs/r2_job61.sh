# round 2, job 61: C5 at N = 1 (FP32 in place) on the final build, direct and through the N > 1 path
set -x
timeout 900 python bench.py --workload C5 --steps 5 --warmup 3 --e2e-steps 10 > gpurun_out/j61_c5.log 2>&1; echo c5_rc=$?
LBGPU_BENCH_SLAB_RING=1 timeout 1200 python bench.py --steps 5 --warmup 3 --e2e-steps 5 --workload C5 > gpurun_out/j61_ring_c5.log 2>&1; echo ring_rc=$?
