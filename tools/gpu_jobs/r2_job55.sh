# round 2, job 55: fused-pair block shapes at C3 and at the C5 slab's shape
set -x
for lib in liblbgpu.so variants/b64x2.so variants/b128.so; do
  if [ $lib = liblbgpu.so ]; then unset LBGPU_LIB; else export LBGPU_LIB=$PWD/$lib; fi
  python tools/probe.py rates >> gpurun_out/j55.log 2>&1
  python tools/probe.py rates lattice.nx=256 lattice.ny=512 lattice.nz=512 tags.design_x0=64 tags.design_x1=191 >> gpurun_out/j55.log 2>&1
done
