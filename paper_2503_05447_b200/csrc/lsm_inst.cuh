// lsm_inst.cuh -- variant dispatch + instantiation of the LSM kernels for one element type
// (included by lsm_inst_bf16.cu / lsm_inst_f32.cu with LSM_T / LSM_SUFFIX defined).
#include "lsm_kernels.cuh"
#include "lsm_launch.h"

namespace lmoe_dev {
namespace {

template <typename T, int DECAY, int FM, bool NORM, bool REV>
cudaError_t sp_launch(dim3 grid, cudaStream_t st, const CUtensorMap& k, const CUtensorMap& v,
                      const LsmFwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_state_pass<T, DECAY, FM, NORM, REV>, state_pass_smem<T>());
        e != cudaSuccess)
        return e;
    return launch_pdl(lsm_state_pass<T, DECAY, FM, NORM, REV>, grid, dim3(kStatePassThreads), state_pass_smem<T>(),
                      st, k, v, p);
}

template <typename T, int DECAY, int FM, bool NORM, bool REV>
cudaError_t op_launch(dim3 grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& k,
                      const CUtensorMap& v, const CUtensorMap& o, const LsmFwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_output_pass<T, DECAY, FM, NORM, REV>, output_pass_smem<T>());
        e != cudaSuccess)
        return e;
    return launch_pdl(lsm_output_pass<T, DECAY, FM, NORM, REV>, grid, dim3(output_pass_threads<T>()),
                      output_pass_smem<T>(), st, q, k, v, o, p);
}

}  // namespace

#define LSM_VARIANTS(X, ...)                                                                  \
    switch (v.rev * 1000 + v.decay * 100 + v.fm * 10 + v.norm) {                              \
        case 0: return X<LSM_T, 0, 0, false, false>(__VA_ARGS__);                                    \
        case 1: return X<LSM_T, 0, 0, true, false>(__VA_ARGS__);                                     \
        case 10: return X<LSM_T, 0, 1, false, false>(__VA_ARGS__);                                   \
        case 11: return X<LSM_T, 0, 1, true, false>(__VA_ARGS__);                                    \
        case 20: return X<LSM_T, 0, 2, false, false>(__VA_ARGS__);                                   \
        case 21: return X<LSM_T, 0, 2, true, false>(__VA_ARGS__);                                    \
        case 100: return X<LSM_T, 1, 0, false, false>(__VA_ARGS__);                                  \
        case 101: return X<LSM_T, 1, 0, true, false>(__VA_ARGS__);                                   \
        case 110: return X<LSM_T, 1, 1, false, false>(__VA_ARGS__);                                  \
        case 111: return X<LSM_T, 1, 1, true, false>(__VA_ARGS__);                                   \
        case 120: return X<LSM_T, 1, 2, false, false>(__VA_ARGS__);                                  \
        case 121: return X<LSM_T, 1, 2, true, false>(__VA_ARGS__);                                   \
        case 200: return X<LSM_T, 2, 0, false, false>(__VA_ARGS__);                                  \
        case 210: return X<LSM_T, 2, 1, false, false>(__VA_ARGS__);                                  \
        case 220: return X<LSM_T, 2, 2, false, false>(__VA_ARGS__);                                  \
        case 1000: return X<LSM_T, 0, 0, false, true>(__VA_ARGS__);                           \
        case 1100: return X<LSM_T, 1, 0, false, true>(__VA_ARGS__);                           \
        case 1200: return X<LSM_T, 2, 0, false, true>(__VA_ARGS__);                           \
        default: return cudaErrorInvalidValue;                                                \
    }

#define LSM_CAT2(a, b) a##b
#define LSM_CAT(a, b) LSM_CAT2(a, b)

cudaError_t LSM_CAT(launch_state_pass_, LSM_SUFFIX)(LsmVariant v, dim3 grid, cudaStream_t st,
                                                    const CUtensorMap& k, const CUtensorMap& val,
                                                    const LsmFwdParams& p) {
    LSM_VARIANTS(sp_launch, grid, st, k, val, p)
}

cudaError_t LSM_CAT(launch_output_pass_, LSM_SUFFIX)(LsmVariant v, dim3 grid, cudaStream_t st,
                                                     const CUtensorMap& q, const CUtensorMap& k,
                                                     const CUtensorMap& val, const CUtensorMap& o,
                                                     const LsmFwdParams& p) {
    LSM_VARIANTS(op_launch, grid, st, q, k, val, o, p)
}

}  // namespace lmoe_dev
