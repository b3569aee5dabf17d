# round 2, job 58: FP64 split adjoint reading the staged v in place (variants, 4 / 5 blocks)
set -x
python tools/probe.py aa > gpurun_out/j58_main.log 2>&1
python tools/probe.py variants variants > gpurun_out/j58_var.log 2>&1
python tools/probe.py variants variants streaming=aa > gpurun_out/j58_var_aa.log 2>&1
