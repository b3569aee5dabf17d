# round 2, job 7: fused one-shot update, doubling upload slices, C1-C3 + C4 configs evidence
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "one_shot or deferred or design" > gpurun_out/j7_tests.log 2>&1; echo t_rc=$?
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j7_e2e_trace.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/j7_bench.log 2>&1; echo bench_rc=$?
cp profiles/r2_configs.json profiles/r2_configs.base.json
timeout 2400 python tools/bench_configs.py r2 C1 C2 C3 C4 > gpurun_out/j7_configs.log 2>&1; echo cfg_rc=$?
cp gpurun_out/r2_configs_part.json gpurun_out/j7_configs_part.json
