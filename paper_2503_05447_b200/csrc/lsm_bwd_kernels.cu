// lsm_bwd_kernels.cu -- elementwise / scan kernels around the three chunk passes of the LSM
// backward (lmoe_lsm_bwd, lsm_host.cu):
//
//   dphiq  = d/d phi(q)  from the dq pass   (forward-shaped:  q'=dO, k'=v,  v'=phi(k))
//   dkeff  = d/d keff    from the dk pass   (reverse-time:    q'=v,  k'=dO, v'=phi(q))
//   dv                   from the dv pass   (reverse-time:    q'=keff, k'=phi(q), v'=dO)
//
// and here the chain rule the reference tape applies (tensor.hpp:1178-1215 over the ops of
// lsm.hpp:483-598): dq = dphiq * phi'(q), dk = dkeff * kf * phi'(k) (kf = softplus(b) for
// Mamba2) and the keff-factor gradient dkf_t = phi(k_t).dkeff_t; the decay-gate gradients
// themselves come from lsm_dgate.cu.
#include "lsm_fwd.cuh"
#include "lsm_launch.h"

namespace lmoe_dev {

template <int FM>
__device__ __forceinline__ float fmap_grad_t(float x) {
    if constexpr (FM == 1) return x > 0.f ? 1.f : __expf(x);
    else if constexpr (FM == 2) return 2.f * x;
    else return 1.f;
}

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(*p);
    else return *p;
}
template <typename T>
__device__ __forceinline__ void st_f(T* p, float x) {
    if constexpr (sizeof(T) == 2) *p = __float2bfloat16_rn(x);
    else *p = x;
}

// One warp per (b, t, h) row of D elements; lane owns D/32 consecutive elements.
template <typename T, int D, int FM, bool MAMBA>
__global__ void __launch_bounds__(256) lsm_bwd_finish(const T* __restrict__ q, const T* __restrict__ k,
                                                      const float* __restrict__ dphq,
                                                      const float* __restrict__ dkef,
                                                      const float* __restrict__ b_pre, T* __restrict__ dq,
                                                      T* __restrict__ dk,
                                                      float* __restrict__ dkf, int N, int H) {
    constexpr int EPL = D / 32;
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int b = blockIdx.y;
    if (w >= (long long)N * H) return;
    const int t = (int)(w / H), h = (int)(w % H);
    const size_t row = ((size_t)b * N + t) * H + h;
    const size_t base = row * D + lane * EPL;
    float kf = 1.f;
    if constexpr (MAMBA) kf = softplus_f(__ldg(b_pre + row));
    float skf = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const float xq = ld_f(q + base + e), xk = ld_f(k + base + e);
        const float gq = dphq[base + e], gk = dkef[base + e];
        st_f(dq + base + e, gq * fmap_grad_t<FM>(xq));
        st_f(dk + base + e, gk * kf * fmap_grad_t<FM>(xk));
        if constexpr (MAMBA) {
            const float pk = fmap_t<FM>(xk);
            skf += pk * gk;
        }
    }
    if constexpr (MAMBA) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            skf += __shfl_xor_sync(0xFFFFFFFFu, skf, o);
        }
        if (lane == 0) {
            dkf[((size_t)b * H + h) * N + t] = skf;
        }
    }
}

// out[bh] = in[bh]^T for D x D fp32 matrices
__global__ void lsm_transpose_states(const float* __restrict__ in, float* __restrict__ out, int D) {
    const size_t bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= D * D) return;
    const int i = e / D, j = e % D;
    out[bh * D * D + (size_t)j * D + i] = in[bh * D * D + e];
}

template <typename T, int FM>
__global__ void lsm_apply_fmap(const T* __restrict__ x, T* __restrict__ y, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        st_f(y + i, fmap_t<FM>(ld_f(x + i)));
}

// ---------------------------------------------------------------- normaliser backward helpers
// o = num / den (chunk_forward_separable with the normaliser, lsm.hpp:584-596): the upstream
// gradient splits into dnum = dO / den and dden = -(dO . num) / den^2, the latter fed to an
// LSM whose value is e0 (den = column 0 of that LSM's output).
template <typename T>
__global__ void lsm_fill_e0(T* __restrict__ x, size_t rows, int D) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * D; i += (size_t)gridDim.x * blockDim.x)
        st_f(x + i, (i % D) == 0 ? 1.f : 0.f);
}

// one warp per (b, t, h) row
template <typename T, int D>
__global__ void __launch_bounds__(256) lsm_norm_prep(const T* __restrict__ num, const T* __restrict__ den_o,
                                                     const T* __restrict__ dO, T* __restrict__ dO1,
                                                     T* __restrict__ dO2, size_t rows, int* err) {
    constexpr int EPL = D / 32;
    const size_t row = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float den = ld_f(den_o + row * D);
    const float inv = 1.f / den;
    float dn = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const size_t i = row * D + lane * EPL + e;
        const float g = ld_f(dO + i);
        dn += g * ld_f(num + i);
        st_f(dO1 + i, g * inv);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dn += __shfl_xor_sync(0xFFFFFFFFu, dn, o);
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int c = lane * EPL + e;
        st_f(dO2 + row * D + c, c == 0 ? -dn * inv * inv : 0.f);
    }
    if (lane == 0 && fabsf(den) < 1e-12f) atomicOr(err, 1);
}

template <typename T>
__global__ void lsm_add_inplace(T* __restrict__ dst, const T* __restrict__ src, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        st_f(dst + i, ld_f(dst + i) + ld_f(src + i));
}

// ------------------------------------------------------------------------------- launchers
template <typename T, int D>
static cudaError_t finish_t(int fm, bool mamba, const void* q, const void* k, const float* dphq,
                            const float* dkef, const float* b_pre, void* dq, void* dk, float* dkf, int B, int N, int H, cudaStream_t st) {
    const dim3 grid((unsigned)(((long long)N * H + 7) / 8), B);
    const T* qq = static_cast<const T*>(q);
    const T* kk = static_cast<const T*>(k);
    T* oq = static_cast<T*>(dq);
    T* ok = static_cast<T*>(dk);
#define FIN(F, M) lsm_bwd_finish<T, D, F, M><<<grid, 256, 0, st>>>(qq, kk, dphq, dkef, b_pre, oq, ok, dkf, N, H)
    if (mamba) {
        if (fm == 0) FIN(0, true); else if (fm == 1) FIN(1, true); else FIN(2, true);
    } else {
        if (fm == 0) FIN(0, false); else if (fm == 1) FIN(1, false); else FIN(2, false);
    }
#undef FIN
    return cudaGetLastError();
}

cudaError_t launch_bwd_finish(bool bf16, int fm, bool mamba, const void* q, const void* k,
                              const float* dphq, const float* dkef, const float* b_pre, void* dq,
                              void* dk, float* dkf, int B, int N, int H, cudaStream_t st) {
    return bf16 ? finish_t<__nv_bfloat16, 128>(fm, mamba, q, k, dphq, dkef, b_pre, dq, dk, dkf, B, N, H, st)
                : finish_t<float, 64>(fm, mamba, q, k, dphq, dkef, b_pre, dq, dk, dkf, B, N, H, st);
}

cudaError_t launch_transpose_states(const float* in, float* out, int BH, int D, cudaStream_t st) {
    lsm_transpose_states<<<dim3((D * D + 255) / 256, BH), 256, 0, st>>>(in, out, D);
    return cudaGetLastError();
}

cudaError_t launch_apply_fmap(bool bf16, int fm, const void* x, void* y, size_t n, cudaStream_t st) {
    const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
#define AF(T, F) lsm_apply_fmap<T, F><<<grid, 256, 0, st>>>(static_cast<const T*>(x), static_cast<T*>(y), n)
    if (bf16) { if (fm == 1) AF(__nv_bfloat16, 1); else AF(__nv_bfloat16, 2); }
    else { if (fm == 1) AF(float, 1); else AF(float, 2); }
#undef AF
    return cudaGetLastError();
}

}  // namespace lmoe_dev

namespace lmoe_dev {
cudaError_t launch_norm_helpers(int op, bool bf16, void* a, const void* b, const void* c, const void* d, void* e,
                                void* f, size_t rows, int D, int* err, cudaStream_t st) {
    const unsigned grid = (unsigned)std::min<size_t>((rows * D + 255) / 256, 148 * 16);
    if (op == 0) {  // a <- e0 rows
        if (bf16) lsm_fill_e0<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(a), rows, D);
        else lsm_fill_e0<float><<<grid, 256, 0, st>>>(static_cast<float*>(a), rows, D);
    } else if (op == 1) {  // (num b, den c, dO d) -> dO1 e, dO2 f
        const unsigned g8 = (unsigned)((rows + 7) / 8);
        if (bf16)
            lsm_norm_prep<__nv_bfloat16, 128><<<g8, 256, 0, st>>>(
                static_cast<const __nv_bfloat16*>(b), static_cast<const __nv_bfloat16*>(c),
                static_cast<const __nv_bfloat16*>(d), static_cast<__nv_bfloat16*>(e), static_cast<__nv_bfloat16*>(f),
                rows, err);
        else
            lsm_norm_prep<float, 64><<<g8, 256, 0, st>>>(static_cast<const float*>(b), static_cast<const float*>(c),
                                                       static_cast<const float*>(d), static_cast<float*>(e),
                                                       static_cast<float*>(f), rows, err);
    } else {  // a += b over rows * D elements
        if (bf16) lsm_add_inplace<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(a),
                                                                        static_cast<const __nv_bfloat16*>(b), rows * D);
        else lsm_add_inplace<float><<<grid, 256, 0, st>>>(static_cast<float*>(a), static_cast<const float*>(b), rows * D);
    }
    return cudaGetLastError();
}
}  // namespace lmoe_dev
