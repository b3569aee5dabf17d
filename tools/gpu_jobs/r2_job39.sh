# round 2, job 39: bench.py's N > 1 code path on one GPU (single-rank NCCL ring), C3 and C5
set -x
LBGPU_BENCH_SLAB_RING=1 timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 10 --workload C3 > gpurun_out/j39_ring_c3.log 2>&1; echo c3_rc=$?
LBGPU_BENCH_SLAB_RING=1 timeout 1200 python bench.py --steps 5 --warmup 3 --e2e-steps 5 --workload C5 > gpurun_out/j39_ring_c5.log 2>&1; echo c5_rc=$?
