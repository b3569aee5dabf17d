# round 2, job 46: in-place remat + 4-block bounds: full suite, bench, rates, C5 N=1, ring check
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j46_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j46_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py aa > gpurun_out/j46_aa.log 2>&1
timeout 900 python bench.py --workload C5 --steps 5 --warmup 3 --e2e-steps 10 > gpurun_out/j46_c5.log 2>&1; echo c5_rc=$?
LBGPU_BENCH_SLAB_RING=1 timeout 1200 python bench.py --steps 5 --warmup 3 --e2e-steps 5 --workload C5 > gpurun_out/j46_ring_c5.log 2>&1; echo ring_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j46_smoke.log 2>&1; echo smoke_rc=$?
