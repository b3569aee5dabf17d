# round 2, job 42: in-place pair with 64x2 blocks
set -x
python tools/probe.py rates streaming=aa > gpurun_out/j42_main.log 2>&1
python tools/probe.py variants variants streaming=aa > gpurun_out/j42_var.log 2>&1
python tools/probe.py rates streaming=aa > gpurun_out/j42_main2.log 2>&1
