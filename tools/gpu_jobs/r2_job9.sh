# round 2, job 9: the whole -m gpu suite on the current build, bench, e2e probe
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/j9_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j9_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py e2e > gpurun_out/j9_e2e.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j9_e2e_trace.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j9_smoke.log 2>&1; echo smoke_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j9_e2e_launches.csv python tools/probe.py ncu e2e > gpurun_out/j9_e2e_ncu.log 2>&1; echo ncu_rc=$?
