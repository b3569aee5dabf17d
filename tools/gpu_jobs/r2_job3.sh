# round 2, job 3: parity suite + full-size + bench + AA / e2e probes + ncu captures
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/j3_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j3_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py aa > gpurun_out/j3_aa.log 2>&1
python tools/probe.py e2e > gpurun_out/j3_e2e.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py ncu e2e > gpurun_out/j3_e2e_trace.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j3_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/j3_ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_pair -s 2 -c 1 -o gpurun_out/j3_pair python tools/probe.py ncu pair > gpurun_out/j3_ncu_pair.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_gradient -s 1 -c 1 -o gpurun_out/j3_grad python tools/probe.py ncu gradient > gpurun_out/j3_ncu_grad.log 2>&1; echo ncu3=$?
ncu --set full --clock-control none --import-source on -k regex:k_pair_aa -s 2 -c 1 -o gpurun_out/j3_pair_aa python tools/probe.py ncu aa > gpurun_out/j3_ncu_aa.log 2>&1; echo ncu4=$?
