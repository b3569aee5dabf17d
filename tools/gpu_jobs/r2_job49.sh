# round 2, job 49: FP32 gathering adjoint with v's gather offsets re-formed (variants)
set -x
python tools/probe.py rates model.precision=32 > gpurun_out/j49_main.log 2>&1
python tools/probe.py variants variants model.precision=32 > gpurun_out/j49_var.log 2>&1
