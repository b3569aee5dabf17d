# round 2, job 63: fused pair as persistent blocks (variant): parity subset + rates
set -x
LBGPU_LIB=$PWD/variants/per.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pair or deferred or gated" > gpurun_out/j63_tests.log 2>&1; echo rc=$?
python tools/probe.py rates > gpurun_out/j63_main.log 2>&1
python tools/probe.py variants variants > gpurun_out/j63_var.log 2>&1
python tools/probe.py rates > gpurun_out/j63_main2.log 2>&1
LBGPU_LIB=$PWD/variants/per.so python tools/probe.py e2e > gpurun_out/j63_e2e_per.log 2>&1
python tools/probe.py e2e > gpurun_out/j63_e2e_main.log 2>&1
