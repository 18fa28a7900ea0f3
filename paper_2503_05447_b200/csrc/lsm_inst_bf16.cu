// bf16 (head_dim 128) instantiations of the LSM forward kernels.
#define LSM_T __nv_bfloat16
#define LSM_SUFFIX bf16
#include "lsm_inst.cuh"
