# round 2, job 5: gated deferred pair, conditioning-aware full-size parity, FD at C3 scale
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "deferred or design or pair" > gpurun_out/j5_pair.log 2>&1; echo pair_rc=$?
timeout 600 python -m pytest tests/test_gpu_fdcheck.py tests/test_integration.py tests/test_gpu_slabs.py -q -p no:cacheprovider > gpurun_out/j5_fd.log 2>&1; echo fd_rc=$?
python tools/probe.py e2e > gpurun_out/j5_e2e.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/j5_bench.log 2>&1; echo bench_rc=$?
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/j5_full.log 2>&1; echo full_rc=$?
