# round 2, job 64: the full gpu suite and the bench on a from-scratch build of HEAD
set -x
LBGPU_LIB=$PWD/variants/fresh.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j64_gpu.log 2>&1; echo gpu_rc=$?
LBGPU_LIB=$PWD/variants/fresh.so python bench.py --steps 20 --warmup 5 > gpurun_out/j64_bench.log 2>&1; echo bench_rc=$?
