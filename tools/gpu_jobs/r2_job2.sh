set -x
timeout 600 python -m pytest tests/test_gpu_aa.py -q -x -p no:cacheprovider > gpurun_out/j2_aa.log 2>&1; echo aa_rc=$?
timeout 900 python -m pytest tests/test_integration.py tests/test_gpu_fdcheck.py -q -p no:cacheprovider --durations=10 > gpurun_out/j2_integ.log 2>&1; echo integ_rc=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --durations=10 > gpurun_out/j2_full.log 2>&1; echo full_rc=$?
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --deselect tests/test_gpu_aa.py > gpurun_out/j2_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j2_bench.log 2>&1; echo bench_rc=$?
python bench.py --steps 20 --warmup 5 --workload C5 > gpurun_out/j2_bench_c5.log 2>&1; echo c5_rc=$?
