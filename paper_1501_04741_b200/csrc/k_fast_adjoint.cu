// fast build, adjoint part (see kernels.cuh). 
#define LBGPU_EXACT 0
#define LBGPU_PART_ADJOINT
#include "kernels.cuh"
