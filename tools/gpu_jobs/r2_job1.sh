set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j1_smi.txt
python tools/probe.py variants variants > gpurun_out/j1_variants.log 2>&1
LBGPU_LIB=$PWD/variants/bx128.so python tools/probe.py geom > gpurun_out/j1_geom128.log 2>&1
LBGPU_LIB=$PWD/variants/bx32.so python tools/probe.py geom > gpurun_out/j1_geom32.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 -p no:cacheprovider > gpurun_out/j1_pytest.log 2>&1
echo pytest_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j1_bench.log 2>&1
echo bench_rc=$?
