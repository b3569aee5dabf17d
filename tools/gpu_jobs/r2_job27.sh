# round 2, job 27: upload-gated primal_step_with_design; objective() in one readback
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j27_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j27_bench.log 2>&1; echo bench_rc=$?
