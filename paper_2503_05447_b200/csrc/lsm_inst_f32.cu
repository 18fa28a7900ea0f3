// fp32 / tf32 (head_dim 64) instantiations of the LSM forward kernels.
#define LSM_T float
#define LSM_SUFFIX f32
#include "lsm_inst.cuh"
