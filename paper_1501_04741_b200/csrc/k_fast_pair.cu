// fast build, fused primal/adjoint pair sweep (see kernels.cuh).
#define LBGPU_EXACT 0
#define LBGPU_PART_PAIR
#include "kernels.cuh"
