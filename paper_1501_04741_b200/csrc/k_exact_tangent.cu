// exact build, tangent part (see kernels.cuh). Compiled with -fmad=false.
#define LBGPU_EXACT 1
#define LBGPU_PART_TANGENT
#include "kernels.cuh"
