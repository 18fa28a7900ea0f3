// lsm_launch.h -- host-callable launchers of the LSM forward kernels (one per dtype and
// phase), dispatching the compile-time (decay, feature map, normaliser) variant.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <utility>

#include "lsm_fwd.cuh"

namespace lmoe_dev {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `fn` on the CURRENT device, once per
// (kernel, device) pair: function attributes are per device, so a process driving several
// GPUs (one thread each) sets them on every device it launches on (common.cu).
cudaError_t ensure_smem(const void* fn, int bytes);

// Launch with programmatic stream serialization (PDL; see ptx.cuh pdl_wait / pdl_trigger).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}


struct LsmVariant {
    int decay;  // DecayMode
    int fm;     // 0 identity, 1 elu+1, 2 squared
    int norm;   // normaliser
    int hgrn2;  // TokenVector with keff = 1 - a (HGRN2)
    int rev = 0;  // reverse-time backward pass (fm = 0, norm = 0)
};

// local-state correction of the output pass (lsm_local_fix): grid (nseg - 1, H, B)
cudaError_t launch_local_fix_bf16(int decay, dim3 grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& o,
                                  const LsmFwdParams& p);
// the same for TokenVector decays (lsm_local_fix_vec, lsm_vec_kernels.cuh)
cudaError_t launch_local_fix_vec_bf16(dim3 grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& a,
                                      const CUtensorMap& o, const LsmFwdParams& p);
cudaError_t launch_state_pass_bf16(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& k,
                                   const CUtensorMap& val, const LsmFwdParams& p);
cudaError_t launch_output_pass_bf16(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& q,
                                    const CUtensorMap& k, const CUtensorMap& val,
                                    const CUtensorMap& o, const LsmFwdParams& p);
// single-read persistent forward (lsm_fused.cuh), grid = P * B * H CTAs
cudaError_t launch_fused_fwd_bf16(LsmVariant v, int grid, cudaStream_t st, const CUtensorMap& q, const CUtensorMap& k,
                                  const CUtensorMap& val, const CUtensorMap& o, const LsmFwdParams& p);
cudaError_t launch_state_pass_f32(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& k,
                                  const CUtensorMap& val, const LsmFwdParams& p);
cudaError_t launch_output_pass_f32(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& q,
                                   const CUtensorMap& k, const CUtensorMap& val,
                                   const CUtensorMap& o, const LsmFwdParams& p);

}  // namespace lmoe_dev

namespace lmoe_dev {
cudaError_t launch_seg_combine(dim3 grid, cudaStream_t st, const float* S, const float* zS,
                               const float* logD, const float* M0, const float* z0, float* Min,
                               float* zin, float* Mfin, float* zfin, float* logDtot, int fin_stride,
                               int nseg, int dk, int dv, int norm, int lw, int rev, int* err);
cudaError_t launch_sum_states(const float* gathered, int world, int BH, int nm, float* M, cudaStream_t st);
cudaError_t launch_rank_combine(dim3 grid, cudaStream_t st, const float* gathered, int P, int BH,
                                int rank, int dk, int dv, int norm, int lw, float* M0, float* z0);
cudaError_t launch_rank_seg_combine(const float* gathered, int P, int BH, int rank, const float* S, const float* zS,
                                    const float* logD, float* Min, float* zin, float* Mfin, float* zfin, int nseg,
                                    int dk, int dv, int norm, int lw, cudaStream_t st);
cudaError_t launch_rank_combine_rev(const float* gathered, int P, int BH, int rank, int world, int dk, int dv,
                                    int lw, float* X, cudaStream_t st);
// TokenVector decays (GLA / HGRN2 / RWKV6): variant {decay = 3, fm, norm, hgrn2 in bit 8 of fm}
cudaError_t launch_state_pass_vec_bf16(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& k,
                                       const CUtensorMap& val, const CUtensorMap& a, const LsmFwdParams& p);
cudaError_t launch_output_pass_vec_bf16(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& q,
                                        const CUtensorMap& k, const CUtensorMap& val, const CUtensorMap& a,
                                        const CUtensorMap& o, const LsmFwdParams& p);
cudaError_t launch_state_pass_vec_f32(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& k,
                                      const CUtensorMap& val, const CUtensorMap& a, const LsmFwdParams& p);
cudaError_t launch_output_pass_vec_f32(LsmVariant v, dim3 grid, cudaStream_t st, const CUtensorMap& q,
                                       const CUtensorMap& k, const CUtensorMap& val, const CUtensorMap& a,
                                       const CUtensorMap& o, const LsmFwdParams& p);
}  // namespace lmoe_dev

namespace lmoe_dev {
// backward helpers (lsm_bwd_kernels.cu)
cudaError_t launch_bwd_finish(bool bf16, int fm, bool mamba, const void* q, const void* k,
                              const float* dphq, const float* dkef, const float* b_pre, void* dq,
                              void* dk, float* dkf, int B, int N, int H, cudaStream_t st);
cudaError_t launch_mamba_dgate(bool bf16, const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                               const CUtensorMap& dO, const CUtensorMap& m, const CUtensorMap& dm,
                               const float* b_pre, const float* a_raw, const float* dkf, const void* dk,
                               float* db_pre, float* da_raw, int B, int N, int H, cudaStream_t st);
cudaError_t launch_transpose_states(const float* in, float* out, int BH, int D, cudaStream_t st);
cudaError_t launch_apply_fmap(bool bf16, int fm, const void* x, void* y, size_t n, cudaStream_t st);
// normaliser backward: op 0 fill e0 rows into a; op 1 (num b, den c, dO d) -> dO / den into e and
// -(dO . num) / den^2 e0 into f (err on |den| < 1e-12); op 2 a += b
cudaError_t launch_norm_helpers(int op, bool bf16, void* a, const void* b, const void* c, const void* d, void* e,
                                void* f, size_t rows, int D, int* err, cudaStream_t st);
}  // namespace lmoe_dev

namespace lmoe_dev {
// TokenVector backward (lsm_vec_bwd.cu), bf16 / head dim 128
struct VecBwdParams {
    int B, N, H;
    int seg_len, nseg, nchunk;           // nchunk = ceil(N / 128) chunks of the whole sequence
    const float* Min;                     // [BH][nseg][D][D] state entering each segment (carry)
    __nv_bfloat16* snap;                  // carry output [BH][nchunk + 1][D][D]
    const float* bd;                      // [BH][nchunk + 1][D] boundary dots
    const __nv_bfloat16* snap_fwd;        // REV carry: the forward snapshots (for the boundary dots)
    float* bd_out;                        // REV carry: boundary dots out
    void* dq;                             // [B, N, H, D] bf16, or fp32 when out_f32
    void* dk;
    __nv_bfloat16* dv;
    __nv_bfloat16* da;                    // [B, N, H, D]
    int out_f32;                          // dq / dk as fp32 d phi(q) / d keff (feature-map chain rule)
    int* err;                             // [2]: half-chunk decay span out of the fp32 range
    unsigned long long* trace;            // optional clock64 phase trace of one CTA [16 x 16]
    int pf_ahead;                         // lsm_vec_bwd_chunk: L2-prefetch the tiles of the CTA
                                          // this many launch slots ahead (one wave; 0 = off)
};
cudaError_t launch_vec_carry(bool hgrn2, bool rev, dim3 grid, cudaStream_t st, const CUtensorMap& x1,
                             const CUtensorMap& x2, const CUtensorMap& a, const VecBwdParams& p);
// tm = {q, k, v, dO, a_pre, snapM, snapX, dq, dk, dv, da} (dq / dk maps unused when out_f32)
cudaError_t launch_vec_bwd_chunk(bool hgrn2, dim3 grid, cudaStream_t st, const CUtensorMap* tm,
                                 const VecBwdParams& p);
}  // namespace lmoe_dev
