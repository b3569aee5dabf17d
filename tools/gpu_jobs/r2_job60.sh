# round 2, job 60: final verification on the final build
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j60_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j60_bench.log 2>&1; echo bench_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j60_smoke.log 2>&1; echo smoke_rc=$?
