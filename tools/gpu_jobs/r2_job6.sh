# round 2, job 6: binomial checkpoint schedule, launch-first gated pair, FD tolerances, configs evidence
set -x
timeout 900 python -m pytest tests/test_gpu_unsteady.py tests/test_gpu_fdcheck.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "unsteady or schedule or fd or deferred or design" > gpurun_out/j6_tests.log 2>&1; echo t_rc=$?
python tools/probe.py e2e > gpurun_out/j6_e2e.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j6_e2e_trace.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/j6_bench.log 2>&1; echo bench_rc=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k c5 > gpurun_out/j6_c5.log 2>&1; echo c5_rc=$?
timeout 1500 python tools/bench_configs.py r2 C4 C5 > gpurun_out/j6_configs.log 2>&1; echo cfg_rc=$?
