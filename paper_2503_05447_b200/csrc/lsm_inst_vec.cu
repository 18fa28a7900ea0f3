// Instantiations + launchers of the TokenVector-decay (GLA / HGRN2 / RWKV6) LSM kernels.
#include "lsm_launch.h"
#include "lsm_vec_kernels.cuh"

namespace lmoe_dev {
namespace {

template <typename T, int FM, bool NORM, bool HG, bool REV = false>
cudaError_t spv(dim3 grid, cudaStream_t st, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& a,
                const LsmFwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_state_pass_vec<T, FM, NORM, HG, REV>, state_pass_vec_smem<T>());
        e != cudaSuccess)
        return e;
    return launch_pdl(lsm_state_pass_vec<T, FM, NORM, HG, REV>, grid, dim3(kStatePassVecThreads),
                      state_pass_vec_smem<T>(), st, k, v, a, p);
}

template <typename T, int FM, bool NORM, bool HG>
cudaError_t opv(dim3 grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                const CUtensorMap& a, const CUtensorMap& o, const LsmFwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_output_pass_vec<T, FM, NORM, HG>, output_pass_vec_smem<T>());
        e != cudaSuccess)
        return e;
    return launch_pdl(lsm_output_pass_vec<T, FM, NORM, HG>, grid, dim3(output_pass_vec_threads<T>()),
                      output_pass_vec_smem<T>(), st, q, k, v, a, o, p);
}

}  // namespace

#define VEC_VARIANTS(X, T, ...)                                                               \
    switch (v.hgrn2 * 100 + v.fm * 10 + v.norm) {                                             \
        case 0: return X<T, 0, false, false>(__VA_ARGS__);                                    \
        case 1: return X<T, 0, true, false>(__VA_ARGS__);                                     \
        case 10: return X<T, 1, false, false>(__VA_ARGS__);                                   \
        case 11: return X<T, 1, true, false>(__VA_ARGS__);                                    \
        case 20: return X<T, 2, false, false>(__VA_ARGS__);                                   \
        case 21: return X<T, 2, true, false>(__VA_ARGS__);                                    \
        case 100: return X<T, 0, false, true>(__VA_ARGS__);                                   \
        case 110: return X<T, 1, false, true>(__VA_ARGS__);                                   \
        case 120: return X<T, 2, false, true>(__VA_ARGS__);                                   \
        default: return cudaErrorInvalidValue;                                                \
    }

cudaError_t launch_state_pass_vec_bf16(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& k,
                                       const CUtensorMap& val, const CUtensorMap& a, const LsmFwdParams& p) {
    // backward adjoint states (lsm_vec_bwd.cu): feature map pre-applied, no normaliser
    if (v.rev) return spv<__nv_bfloat16, 0, false, false, true>(grid, st, k, val, a, p);
    VEC_VARIANTS(spv, __nv_bfloat16, grid, st, k, val, a, p)
}
cudaError_t launch_output_pass_vec_bf16(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& q,
                                        const CUtensorMap& k, const CUtensorMap& val, const CUtensorMap& a,
                                        const CUtensorMap& o, const LsmFwdParams& p) {
    VEC_VARIANTS(opv, __nv_bfloat16, grid, st, q, k, val, a, o, p)
}
cudaError_t launch_state_pass_vec_f32(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& k,
                                      const CUtensorMap& val, const CUtensorMap& a, const LsmFwdParams& p) {
    VEC_VARIANTS(spv, float, grid, st, k, val, a, p)
}
cudaError_t launch_output_pass_vec_f32(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& q,
                                       const CUtensorMap& k, const CUtensorMap& val, const CUtensorMap& a,
                                       const CUtensorMap& o, const LsmFwdParams& p) {
    VEC_VARIANTS(opv, float, grid, st, q, k, val, a, o, p)
}

cudaError_t launch_local_fix_vec_bf16(dim3 grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& a,
                                      const CUtensorMap& o, const LsmFwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_local_fix_vec<128>, fix_vec_smem()); e != cudaSuccess) return e;
    return launch_pdl(lsm_local_fix_vec<128>, grid, dim3(kFixVecThreads), fix_vec_smem(), st, q, a, o, p);
}

}  // namespace lmoe_dev
