# round 2, job 62: FP32 in-place pair with v staged and read in place (variant)
set -x
python tools/probe.py rates streaming=aa model.precision=32 > gpurun_out/j62_main.log 2>&1
python tools/probe.py variants variants streaming=aa model.precision=32 > gpurun_out/j62_var.log 2>&1
python tools/probe.py rates streaming=aa model.precision=32 > gpurun_out/j62_main2.log 2>&1
