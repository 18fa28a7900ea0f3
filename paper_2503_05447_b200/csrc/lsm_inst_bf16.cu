// bf16 (head_dim 128) instantiations of the LSM forward kernels.
#define LSM_T __nv_bfloat16
#define LSM_SUFFIX bf16
#include "lsm_inst.cuh"

namespace lmoe_dev {
// local-state correction (lsm_kernels.cuh, bf16 only): ConstScalar / TokenScalar decays
cudaError_t launch_local_fix_bf16(int decay, dim3 grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& o,
                                  const LsmFwdParams& p) {
    auto go = [&](auto kern) -> cudaError_t {
        if (cudaError_t e = ensure_smem((const void*)kern, fix_smem()); e != cudaSuccess) return e;
        return launch_pdl(kern, grid, dim3(kFixThreads), fix_smem(), st, q, o, p);
    };
    if (decay == kDecayConst) return go(lsm_local_fix<kDecayConst>);
    if (decay == kDecayTokenScalar) return go(lsm_local_fix<kDecayTokenScalar>);
    return cudaErrorInvalidValue;
}
}  // namespace lmoe_dev
