// fast build, aux part (see kernels.cuh). 
#define LBGPU_EXACT 0
#define LBGPU_PART_AUX
#include "kernels.cuh"
