# round 2, job 14: 32-bit node offsets (Nbr): full gpu suite, bench, rates
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/j14_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j14_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py aa > gpurun_out/j14_aa.log 2>&1
python tools/probe.py e2e > gpurun_out/j14_e2e.log 2>&1
