# round 2, job 36: unsteady adjoint without per-step host syncs (J and inlet sums queued)
set -x
timeout 1800 python -m pytest tests/test_gpu_unsteady.py tests/test_gpu_fullsize.py tests/test_gpu_fdcheck.py -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/j36_tests.log 2>&1; echo rc=$?
