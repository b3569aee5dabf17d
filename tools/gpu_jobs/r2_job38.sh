# round 2, job 38: full gpu suite + bench + smoke on the current build
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j38_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j38_bench.log 2>&1; echo bench_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j38_smoke.log 2>&1; echo smoke_rc=$?
