# round 2, job 13: in-place pair variants (register bound 3, 128-wide blocks, FP32 bound 4)
set -x
python tools/probe.py rates streaming=aa > gpurun_out/j13_main64.log 2>&1
python tools/probe.py rates streaming=aa model.precision=32 > gpurun_out/j13_main32.log 2>&1
python tools/probe.py variants variants streaming=aa > gpurun_out/j13_var64.log 2>&1
python tools/probe.py variants variants streaming=aa model.precision=32 > gpurun_out/j13_var32.log 2>&1
