# round 2, job 50: final verification -- full suite, bench, rates, smoke
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j50_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j50_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py aa > gpurun_out/j50_aa.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j50_smoke.log 2>&1; echo smoke_rc=$?
