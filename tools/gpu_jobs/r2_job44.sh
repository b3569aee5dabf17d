# round 2, job 44: in-place stores with rematerialised neighbour offsets (variant)
set -x
python tools/probe.py aa > gpurun_out/j44_main.log 2>&1
LBGPU_LIB=$PWD/variants/remat.so python tools/probe.py aa > gpurun_out/j44_remat.log 2>&1
