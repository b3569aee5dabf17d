# round 2, job 16: 32-bit element offsets (LBGPU_OFF32=1 experiment) against the main build
set -x
python tools/probe.py aa > gpurun_out/j16_main.log 2>&1
LBGPU_LIB=$PWD/variants/o32.so python tools/probe.py aa > gpurun_out/j16_o32.log 2>&1
python tools/probe.py aa > gpurun_out/j16_main2.log 2>&1
