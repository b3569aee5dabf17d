// fast build, in-place (AA) streaming sweeps (see kernels.cuh).
#define LBGPU_EXACT 0
#define LBGPU_PART_AA
#include "kernels.cuh"
