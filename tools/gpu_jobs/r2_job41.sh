# round 2, job 41: column kernels removed (strips only): full gpu suite, bench, ring checks
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j41_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j41_bench.log 2>&1; echo bench_rc=$?
LBGPU_BENCH_SLAB_RING=1 timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 10 --workload C3 > gpurun_out/j41_ring_c3.log 2>&1; echo ring_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j41_smoke.log 2>&1; echo smoke_rc=$?
