# round 2, job 11: per-node gated upload (sentinel values, one copy), one-block tree,
# in-place register bounds 3/3: full gpu suite, bench, e2e, L2 fetch granularity probe
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/j11_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j11_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py e2e > gpurun_out/j11_e2e.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j11_e2e_trace.log 2>&1
python tools/probe.py rates streaming=aa > gpurun_out/j11_aa.log 2>&1
python tools/probe.py l2gran > gpurun_out/j11_l2gran.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j11_smoke.log 2>&1; echo smoke_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j11_e2e_launches.csv python tools/probe.py ncu e2e > gpurun_out/j11_e2e_ncu.log 2>&1; echo ncu_rc=$?
