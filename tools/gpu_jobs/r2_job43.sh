# round 2, job 43: in-place rates, current build against the build of 83ba08a (same box)
set -x
python tools/probe.py aa > gpurun_out/j43_main.log 2>&1
LBGPU_LIB=$PWD/variants/old.so python tools/probe.py aa > gpurun_out/j43_old.log 2>&1
python tools/probe.py aa > gpurun_out/j43_main2.log 2>&1
