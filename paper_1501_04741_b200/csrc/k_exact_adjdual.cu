// exact build, adjdual part (see kernels.cuh). Compiled with -fmad=false.
#define LBGPU_EXACT 1
#define LBGPU_PART_ADJDUAL
#include "kernels.cuh"
