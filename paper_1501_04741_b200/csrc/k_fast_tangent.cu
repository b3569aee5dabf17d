// fast build, tangent part (see kernels.cuh).
#define LBGPU_EXACT 0
#define LBGPU_PART_TANGENT
#include "kernels.cuh"
