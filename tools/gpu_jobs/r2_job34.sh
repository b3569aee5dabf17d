# round 2, job 34: J from the inbox the gated fused sweep fills
set -x
python tools/probe.py e2e_alt > gpurun_out/j34_alt.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j34_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j34_bench.log 2>&1; echo bench_rc=$?
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j34_trace.log 2>&1
