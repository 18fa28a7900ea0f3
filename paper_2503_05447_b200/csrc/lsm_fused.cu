// lsm_fused.cu -- instantiation and launcher of the single-read persistent LSM forward
// (lsm_fused.cuh): bf16 / head_dim 128, DecayKind None / ConstScalar / TokenScalar, feature
// maps identity / elu+1 / squared, no normaliser.
#include "lsm_fused.cuh"
#include "lsm_launch.h"

namespace lmoe_dev {
namespace {
template <int DECAY, int FM>
cudaError_t fused_t(int grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                    const CUtensorMap& o, const LsmFwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_fused_fwd<DECAY, FM>, fused_smem()); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = fused_smem();
    cfg.stream = st;
    // the segment hand-off spins on other CTAs: all CTAs must be co-resident (grid <= #SMs,
    // one CTA per SM), which a cooperative launch guarantees (or refuses)
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, lsm_fused_fwd<DECAY, FM>, q, k, v, o, p);
}
}  // namespace

cudaError_t launch_fused_fwd_bf16(LsmVariant v, int grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& k,
                                  const CUtensorMap& val, const CUtensorMap& o, const LsmFwdParams& p) {
    if (v.norm || v.rev) return cudaErrorInvalidValue;
    switch (v.decay * 10 + v.fm) {
        case 0: return fused_t<0, 0>(grid, st, q, k, val, o, p);
        case 1: return fused_t<0, 1>(grid, st, q, k, val, o, p);
        case 2: return fused_t<0, 2>(grid, st, q, k, val, o, p);
        case 10: return fused_t<1, 0>(grid, st, q, k, val, o, p);
        case 11: return fused_t<1, 1>(grid, st, q, k, val, o, p);
        case 12: return fused_t<1, 2>(grid, st, q, k, val, o, p);
        case 20: return fused_t<2, 0>(grid, st, q, k, val, o, p);
        case 21: return fused_t<2, 1>(grid, st, q, k, val, o, p);
        case 22: return fused_t<2, 2>(grid, st, q, k, val, o, p);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace lmoe_dev
