# round 2, job 31: evaluate_raw as one fused launch (terms + leaf sums + tree by the last block)
set -x
python tools/probe.py e2e_alt > gpurun_out/j31_alt.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j31_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j31_bench.log 2>&1; echo bench_rc=$?
