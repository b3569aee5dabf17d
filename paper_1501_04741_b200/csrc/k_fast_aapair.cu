// fast build, in-place (AA) fused pair sweep (see kernels.cuh).
#define LBGPU_EXACT 0
#define LBGPU_PART_AAPAIR
#include "kernels.cuh"
