// fast build, primal part (see kernels.cuh). 
#define LBGPU_EXACT 0
#define LBGPU_PART_PRIMAL
#include "kernels.cuh"
