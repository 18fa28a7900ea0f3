// lsm_combine.cu -- segment / rank prefix-combine kernels of the LSM forward.
// log-decays come per (b,h,segment) either as one scalar (None / ConstScalar / TokenScalar)
// or as a d_k vector (TokenVector: GLA / HGRN2 / RWKV6); `lw` is 1 or d_k, and the decay of
// element (i, j) of the state uses log-decay entry i (diag(D) M, parallel.hpp:340-361).
#include "lsm_fwd.cuh"
#include "lsm_launch.h"

namespace lmoe_dev {

// ------------------------------------------------------------------------------------
// Phase 2: decayed exclusive prefix over segments
//   Min[s] = acc ; acc = exp(logD[s][row]) * acc + S[s]        per element of [M | z]
// rev = 1 (backward dM): the same recurrence over segments last-to-first, seeded with
// dM_final; the value after segment 0 is dM0, the gradient of the initial state.
// ------------------------------------------------------------------------------------
__global__ void lsm_seg_combine(const float* __restrict__ S, const float* __restrict__ zS,
                                const float* __restrict__ logD, const float* __restrict__ M0,
                                const float* __restrict__ z0, float* __restrict__ Min,
                                float* __restrict__ zin, float* __restrict__ Mfin,
                                float* __restrict__ zfin, float* __restrict__ logDtot,
                                int fin_stride, int nseg, int dk, int dv, int norm, int lw, int rev,
                                int* err) {
    pdl_wait();
    pdl_trigger();
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int nm = dk * dv;
    const int total = nm + (norm ? dk : 0);
    if (logDtot && blockIdx.x == 0 && threadIdx.x < lw) {
        float t = 0.f;
        for (int s = 0; s < nseg; ++s) t += logD[((size_t)bh * nseg + s) * lw + threadIdx.x];
        logDtot[(size_t)bh * fin_stride + threadIdx.x] = t;
    }
    if (e >= total) return;
    const bool isz = e >= nm;
    const int ee = isz ? e - nm : e;
    const int row = isz ? ee : ee / dv;
    const int li = lw == 1 ? 0 : row;
    const int stride = isz ? dk : nm;
    const float* src = isz ? zS : S;
    float* dst = isz ? zin : Min;
    float acc = 0.f;
    if (isz) { if (z0) acc = z0[(size_t)bh * dk + ee]; }
    else if (M0) acc = M0[(size_t)bh * nm + ee];
    const size_t base = (size_t)bh * nseg * stride + ee;
    // the loads do not depend on the running prefix: fetch 8 segments ahead of the recurrence
    for (int i0 = 0; i0 < nseg; i0 += 8) {
        float sv[8], dv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u;
            const int s = rev ? nseg - 1 - i : i;
            sv[u] = i < nseg ? src[base + (size_t)s * stride] : 0.f;
            dv[u] = i < nseg ? __expf(logD[((size_t)bh * nseg + s) * lw + li]) : 1.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u;
            if (i < nseg) {
                const int s = rev ? nseg - 1 - i : i;
                if (dst) dst[base + (size_t)s * stride] = acc;
                acc = dv[u] * acc + sv[u];
            }
        }
    }
    if (!isfinite(acc)) atomicOr(&err[1], 1);
    float* fin = isz ? zfin : Mfin;
    const int fs = fin_stride ? fin_stride : (isz ? dk : nm);
    if (fin) fin[(size_t)bh * fs + ee] = acc;
}

// LSM sequence parallelism: rank `rank` folds the gathered per-rank payloads
// [world][BH][P] (P = dk*dv [+ dk] + lw: local state from zero, normaliser, total log decay)
// into its carried-in state -- the decayed exclusive prefix of sp_lsm_masked_rank
// (parallel.hpp:340-361): acc_{i+1} = D_i acc_i + M_i over ranks i < rank.
__global__ void sp_rank_combine(const float* __restrict__ gathered, int P, int BH, int rank,
                                int dk, int dv, int norm, int lw, float* __restrict__ M0,
                                float* __restrict__ z0) {
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int nm = dk * dv;
    const int total = nm + (norm ? dk : 0);
    if (e >= total) return;
    const int row = e < nm ? e / dv : e - nm;
    const int li = lw == 1 ? 0 : row;
    float acc = 0.f;
    for (int i = 0; i < rank; ++i) {
        const float* pl = gathered + ((size_t)i * BH + bh) * P;
        acc = __expf(pl[P - lw + li]) * acc + pl[e];
    }
    if (e < nm) M0[(size_t)bh * nm + e] = acc;
    else z0[(size_t)bh * dk + (e - nm)] = acc;
}

// SP phase B in one kernel: the decayed prefix over earlier ranks (sp_rank_combine) seeds the
// decayed exclusive prefix over this rank's segments (lsm_seg_combine): Min per segment and
// the rank's final state.
__global__ void sp_rank_seg_combine(const float* __restrict__ gathered, int P, int BH, int rank,
                                    const float* __restrict__ S, const float* __restrict__ zS,
                                    const float* __restrict__ logD, float* __restrict__ Min,
                                    float* __restrict__ zin, float* __restrict__ Mfin, float* __restrict__ zfin,
                                    int nseg, int dk, int dv, int norm, int lw) {
    pdl_wait();
    pdl_trigger();
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int nm = dk * dv;
    const int total = nm + (norm ? dk : 0);
    if (e >= total) return;
    const bool isz = e >= nm;
    const int ee = isz ? e - nm : e;
    const int row = isz ? ee : ee / dv;
    const int li = lw == 1 ? 0 : row;
    // decayed prefix over the earlier ranks; the payload loads do not depend on it, so they are
    // issued 8 ranks at a time ahead of the recurrence
    float acc = 0.f;
    for (int i0 = 0; i0 < rank; i0 += 8) {
        float mv[8], dv8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float* pl = gathered + ((size_t)(i0 + u) * BH + bh) * P;
            mv[u] = i0 + u < rank ? pl[e] : 0.f;
            dv8[u] = i0 + u < rank ? __expf(pl[P - lw + li]) : 1.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = dv8[u] * acc + mv[u];
    }
    const int stride = isz ? dk : nm;
    const float* src = isz ? zS : S;
    float* dst = isz ? zin : Min;
    const size_t base = (size_t)bh * nseg * stride + ee;
    for (int i0 = 0; i0 < nseg; i0 += 8) {
        float sv[8], dvv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u;
            sv[u] = i < nseg ? src[base + (size_t)i * stride] : 0.f;
            dvv[u] = i < nseg ? __expf(logD[((size_t)bh * nseg + i) * lw + li]) : 1.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (i0 + u < nseg) {
                dst[base + (size_t)(i0 + u) * stride] = acc;
                acc = dvv[u] * acc + sv[u];
            }
        }
    }
    float* fin = isz ? zfin : Mfin;
    if (fin) fin[(size_t)bh * (isz ? dk : nm) + ee] = acc;
}

cudaError_t launch_rank_seg_combine(const float* gathered, int P, int BH, int rank, const float* S, const float* zS,
                                    const float* logD, float* Min, float* zin, float* Mfin, float* zfin, int nseg,
                                    int dk, int dv, int norm, int lw, cudaStream_t st) {
    const int nel = dk * dv + (norm ? dk : 0);
    return launch_pdl(sp_rank_seg_combine, dim3((nel + 255) / 256, BH), dim3(256), 0, st, gathered, P, BH, rank, S,
                      zS, logD, Min, zin, Mfin, zfin, nseg, dk, dv, norm, lw);
}

// SP backward: the adjoint state entering the END of rank `rank`'s slice from the queries of
// later ranks, from the gathered reverse-time payloads [X_i | log D_i] (X_i = the adjoint at
// the start of slice i from its own queries): acc = D_i acc + X_i over i = world-1 .. rank+1.
__global__ void sp_rank_combine_rev(const float* __restrict__ gathered, int P, int BH, int rank, int world,
                                    int dk, int dv, int lw, float* __restrict__ X) {
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int nm = dk * dv;
    if (e >= nm) return;
    const int li = lw == 1 ? 0 : e / dv;
    float acc = 0.f;
    for (int i = world - 1; i > rank; --i) {
        const float* pl = gathered + ((size_t)i * BH + bh) * P;
        acc = __expf(pl[P - lw + li]) * acc + pl[e];
    }
    X[(size_t)bh * nm + e] = acc;
}

cudaError_t launch_rank_combine_rev(const float* gathered, int P, int BH, int rank, int world, int dk, int dv,
                                    int lw, float* X, cudaStream_t st) {
    sp_rank_combine_rev<<<dim3((dk * dv + 255) / 256, BH), 256, 0, st>>>(gathered, P, BH, rank, world, dk, dv, lw, X);
    return cudaGetLastError();
}

// Unmasked SP (parallel.hpp:293-296): M_global = sum over all ranks of the gathered
// local states [world][BH][nm].
__global__ void sp_sum_states(const float* __restrict__ gathered, int world, int BH, int nm,
                              float* __restrict__ M) {
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nm) return;
    float acc = 0.f;
    for (int i = 0; i < world; ++i) acc += gathered[((size_t)i * BH + bh) * nm + e];
    M[(size_t)bh * nm + e] = acc;
}

cudaError_t launch_sum_states(const float* gathered, int world, int BH, int nm, float* M, cudaStream_t st) {
    sp_sum_states<<<dim3((nm + 255) / 256, BH), 256, 0, st>>>(gathered, world, BH, nm, M);
    return cudaGetLastError();
}

cudaError_t launch_seg_combine(dim3 grid, cudaStream_t st, const float* S, const float* zS,
                               const float* logD, const float* M0, const float* z0, float* Min,
                               float* zin, float* Mfin, float* zfin, float* logDtot, int fin_stride,
                               int nseg, int dk, int dv, int norm, int lw, int rev, int* err) {
    return launch_pdl(lsm_seg_combine, grid, dim3(256), 0, st, S, zS, logD, M0, z0, Min, zin, Mfin, zfin, logDtot,
                      fin_stride, nseg, dk, dv, norm, lw, rev, err);
}
cudaError_t launch_rank_combine(dim3 grid, cudaStream_t st, const float* gathered, int P, int BH,
                                int rank, int dk, int dv, int norm, int lw, float* M0, float* z0) {
    sp_rank_combine<<<grid, 256, 0, st>>>(gathered, P, BH, rank, dk, dv, norm, lw, M0, z0);
    return cudaGetLastError();
}

}  // namespace lmoe_dev
