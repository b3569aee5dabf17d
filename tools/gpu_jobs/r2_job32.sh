LBGPU_TRACE_PAIR=1 python tools/probe.py e2e > gpurun_out/j32_trace.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j32_launches.csv python tools/probe.py ncu e2e > gpurun_out/j32_ncu.log 2>&1
