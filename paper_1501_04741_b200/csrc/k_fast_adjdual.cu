// fast build, adjdual part (see kernels.cuh). 
#define LBGPU_EXACT 0
#define LBGPU_PART_ADJDUAL
#include "kernels.cuh"
