# round 2, job 47: FP32 in-place occupancy variants after the store rematerialisation
set -x
python tools/probe.py rates streaming=aa model.precision=32 > gpurun_out/j47_main.log 2>&1
python tools/probe.py variants variants streaming=aa model.precision=32 > gpurun_out/j47_var.log 2>&1
