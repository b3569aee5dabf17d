# round 2, job 8: FP32 occupancy / fusion variants; e2e slices; AA sweep split
set -x
python tools/probe.py variants variants model.precision=32 > gpurun_out/j8_variants.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j8_e2e_trace.log 2>&1
python tools/probe.py e2e > gpurun_out/j8_e2e.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j8_aa_launches.csv python tools/probe.py ncu aa > gpurun_out/j8_aa_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/j8_e2e_launches.csv python tools/probe.py ncu e2e > gpurun_out/j8_e2e_ncu.log 2>&1
