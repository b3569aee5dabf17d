# round 2, job 28: primal_step_with_design parity (both precisions)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "primal_step_with_design or design_pairs or gated" > gpurun_out/j28_tests.log 2>&1; echo rc=$?
