# round 2, job 24: FP32 adjoint, two nodes per thread with the second's gathers prefetched
set -x
python tools/probe.py rates model.precision=32 > gpurun_out/j24_main32.log 2>&1
python tools/probe.py variants variants model.precision=32 > gpurun_out/j24_var32.log 2>&1
for lib in variants/pipe1.so variants/pipe2.so; do
  LBGPU_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_aa.py -m gpu -q -p no:cacheprovider -k "bitwise_equals and 32" > gpurun_out/j24_$(basename $lib .so)_aa.log 2>&1; echo rc=$?
done
