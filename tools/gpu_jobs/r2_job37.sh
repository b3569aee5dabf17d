# round 2, job 37: unsteady back step with the gradient carried by the adjoint sweep
set -x
timeout 1800 python -m pytest tests/test_gpu_unsteady.py tests/test_gpu_fdcheck.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "unsteady or fd" > gpurun_out/j37_tests.log 2>&1; echo rc=$?
timeout 1800 python tools/bench_configs.py r2 C5 > gpurun_out/j37_c5.log 2>&1; echo c5_rc=$?
cp profiles/r2_configs.json gpurun_out/j37_r2_configs.json
