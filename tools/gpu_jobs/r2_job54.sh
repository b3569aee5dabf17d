# round 2, job 54: pair rate against lattice size (is the C5 slab's lower rate a size effect?)
set -x
for dims in "256 128 128" "256 256 256" "256 512 512" "512 512 256"; do
  set -- $dims
  python tools/probe.py rates lattice.nx=$1 lattice.ny=$2 lattice.nz=$3 tags.design_x0=64 tags.design_x1=191 >> gpurun_out/j54.log 2>&1
done
