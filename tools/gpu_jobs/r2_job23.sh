# round 2, job 23: the gated upload's bounded wait (sentinel in the design vector)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "gated or deferred" > gpurun_out/j23_tests.log 2>&1; echo rc=$?
