# round 2, job 25: full gpu suite on the current build, bench (C3), bench --workload C5 at N = 1
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j25_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j25_bench.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --workload C5 --steps 5 --warmup 3 --e2e-steps 10 > gpurun_out/j25_bench_c5.log 2>&1; echo c5_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j25_smoke.log 2>&1; echo smoke_rc=$?
