# round 2, job 59: fused pair's adjoint half reading the staged v in place (variant); adjoint VSMEM default
set -x
python tools/probe.py aa > gpurun_out/j59_main.log 2>&1
python tools/probe.py variants variants > gpurun_out/j59_var.log 2>&1
python tools/probe.py variants variants streaming=aa > gpurun_out/j59_var_aa.log 2>&1
python tools/probe.py aa > gpurun_out/j59_main2.log 2>&1
