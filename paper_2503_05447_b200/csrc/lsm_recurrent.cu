// lsm_recurrent.cu -- the LSM kinds without a chunk-parallel form:
// DeltaNet, GatedDeltaNet (StateLinear), GFW, GateLoop (TokenOuter), TTT, Titans, RWKV7
// (Gradient), S4, Mamba (FullElementwise).  The reference evaluates them token by token
// (recurrent_step, lsm.hpp:335-441; lsm_forward_chunked runs them sequentially inside each
// chunk, lsm.hpp:604-637) and has no SP form for them (parallel.hpp:309-311); so does this
// kernel: one CTA per (b, h) walks the sequence with the d_k x d_v state in registers.
//
// 256 threads: thread = (state column j = tid % D, row group g = tid / D); RP = D*D/256 rows
// per thread (64 at D = 128, 16 at D = 64).  Per token, with the next token's inputs already
// prefetched into registers: k^ (feature map, L2 normalisation for the delta rules),
// c = k^ M (block reduction over the row groups), the elementwise update of M, and
// o = phi(q) M (block reduction) -- four barriers per token, fp32 throughout.
#include "common.h"
#include "internal.h"
#include "lsm_fwd.cuh"

namespace lmoe_dev {

struct RecParams {
    int B, N, H;
    const void* q;
    const void* k;
    const void* v;              // [B, N, H, D] in T
    const void* a_vec;          // RWKV7 / Mamba: a_pre [B, N, H, D] in T
    const float* a_scal;        // DeltaNet / GatedDeltaNet / Titans: a_pre [B, N, H] fp32
    const float* b_pre;         // [B, N, H] fp32 (DeltaNet, GatedDeltaNet, TTT, Titans, RWKV7)
    const void* alpha;          // GFW / GateLoop: alpha_pre [B, N, H, D] in T
    const void* beta;           //                 beta_pre  [B, N, H, D] in T
    const float* s4_delta_raw;  // [H, D]
    const float* s4_b;          // [H, D]
    const float* s4_A_raw;      // [H, D, D]
    const float* mamba_A_raw;   // [H, D, D]
    const float* M0;            // [B, H, D, D] or null
    void* o;                    // [B, N, H, D] in T
    float* M_out;               // [B, H, D, D] or null
    int* err;                   // [1]: non-finite state
};

enum RecKind { kRecDelta = 0, kRecGatedDelta, kRecOuter, kRecTTT, kRecTitans, kRecRWKV7, kRecS4, kRecMamba };

template <typename T>
__device__ __forceinline__ float rec_ld(const void* p, size_t i) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
    else return static_cast<const float*>(p)[i];
}
__device__ __forceinline__ float rec_sigm(float x) { return 1.f / (1.f + __expf(-x)); }

template <typename T, int D, int KIND, int FM>
__global__ void __launch_bounds__(256) lsm_recurrent_kernel(RecParams p) {
    constexpr int RG = 256 / D;   // row groups
    constexpr int RP = D / RG;    // rows per thread
    constexpr bool kVecA = KIND == kRecRWKV7 || KIND == kRecMamba;
    constexpr bool kDelta = KIND == kRecDelta || KIND == kRecGatedDelta;
    constexpr bool kNeedC = kDelta || KIND == kRecTTT || KIND == kRecTitans || KIND == kRecRWKV7;
    __shared__ float sIn[2][6 * D + 4];  // [q | k | v | a_vec | alpha | beta | a_s, b_s] per token
    __shared__ float sPart[RG][D];       // row-group partials of the column reductions
    __shared__ float sK[D];              // k^ of the current token
    __shared__ float sRow[D];            // per-row factor: S4 increment (static), Mamba delta (per token)
    __shared__ float sRed[8];
    const int h = blockIdx.x, b = blockIdx.y;
    const int tid = threadIdx.x, j = tid % D, g = tid / D;
    const size_t bh = (size_t)b * p.H + h;

    float M[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) M[r] = p.M0 ? p.M0[(bh * D + g * RP + r) * D + j] : 0.f;
    // static S4 / Mamba parameters of this thread's elements (S4: the static decay; Mamba:
    // softplus(A)); the S4 per-row increment softplus(delta) b goes to shared memory
    constexpr bool kElem = KIND == kRecS4 || KIND == kRecMamba;
    float sA[kElem ? RP : 1];
#pragma unroll
    for (int r = 0; r < (kElem ? RP : 1); ++r) {
        const int i = g * RP + r;
        sA[r] = 0.f;
        if constexpr (KIND == kRecS4) {
            const float dl = softplus_f(p.s4_delta_raw[h * D + i]);
            sA[r] = __expf(-softplus_f(p.s4_A_raw[((size_t)h * D + i) * D + j]) * dl);  // static decay
        }
        if constexpr (KIND == kRecMamba) sA[r] = softplus_f(p.mamba_A_raw[((size_t)h * D + i) * D + j]);
    }
    if constexpr (KIND == kRecS4) {
        if (tid < D) sRow[tid] = softplus_f(p.s4_delta_raw[h * D + tid]) * p.s4_b[h * D + tid];
    }
    // input loader: element e of [q | k | v | a_vec | alpha | beta | a_s | b_s] of token t
    auto load = [&](int t, int e) -> float {
        const size_t row = ((size_t)b * p.N + t) * p.H + h;
        const int seg = e / D, c = e % D;
        switch (seg) {
            case 0: return rec_ld<T>(p.q, row * D + c);
            case 1: return rec_ld<T>(p.k, row * D + c);
            case 2: return rec_ld<T>(p.v, row * D + c);
            case 3: return kVecA ? rec_ld<T>(p.a_vec, row * D + c) : 0.f;
            case 4: return KIND == kRecOuter ? rec_ld<T>(p.alpha, row * D + c) : 0.f;
            case 5: return KIND == kRecOuter ? rec_ld<T>(p.beta, row * D + c) : 0.f;
            default:
                if (c == 0) return p.a_scal ? p.a_scal[row] : 0.f;
                if (c == 1) return p.b_pre ? p.b_pre[row] : 0.f;
                return 0.f;
        }
    };
    constexpr int NE = 6 * D + 2;
    constexpr int PER = (NE + 255) / 256;
    float pre[PER];
    for (int u = 0; u < PER; ++u) {
        const int e = tid + u * 256;
        pre[u] = (e < NE && p.N > 0) ? load(0, e) : 0.f;
    }
    bool bad = false;
    for (int t = 0; t < p.N; ++t) {
        float* in = sIn[t & 1];
        for (int u = 0; u < PER; ++u) {
            const int e = tid + u * 256;
            if (e < NE) in[e] = pre[u];
        }
        __syncthreads();  // (1) token t inputs in smem
        if (t + 1 < p.N) {
            for (int u = 0; u < PER; ++u) {
                const int e = tid + u * 256;
                pre[u] = e < NE ? load(t + 1, e) : 0.f;  // latency overlaps this token's work
            }
        }
        const float* q = in;
        const float* k = in + D;
        const float* v = in + 2 * D;
        const float* av = in + 3 * D;
        const float* al = in + 4 * D;
        const float* be = in + 5 * D;
        const float a_s = in[6 * D], b_s = in[6 * D + 1];
        // k^ (feature map; L2-normalised for the delta rules, l2_normalize_rows eps 1e-12)
        float kj = 0.f;
        if (tid < D) {
            kj = k[tid];
            if constexpr (FM == 1) kj = kj > 0.f ? kj + 1.f : __expf(kj);
            if constexpr (FM == 2) kj = kj * kj;
        }
        if constexpr (kDelta) {
            float sq = kj * kj;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
            if (tid < D && (tid & 31) == 0) sRed[tid >> 5] = sq;
        }
        if (tid < D) sK[tid] = kj;
        if constexpr (KIND == kRecMamba) {
            if (tid < D) sRow[tid] = softplus_f(av[tid]);  // delta_i = softplus(a_pre row)
        }
        __syncthreads();  // (2) k^ (and its squared-norm partials)
        float knorm = 1.f;
        if constexpr (kDelta) {
            float s2 = 0.f;
#pragma unroll
            for (int w = 0; w < D / 32; ++w) s2 += sRed[w];
            knorm = rsqrtf(s2 + 1e-12f);
        }
        float c = 0.f;
        if constexpr (kNeedC) {
            float part = 0.f;
#pragma unroll
            for (int r = 0; r < RP; ++r) part += sK[g * RP + r] * knorm * M[r];
            sPart[g][j] = part;
            __syncthreads();  // (3) c = k^ M
#pragma unroll
            for (int gg = 0; gg < RG; ++gg) c += sPart[gg][j];
        }
        const float vj = v[j];
        float opart = 0.f;
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const int i = g * RP + r;
            const float ki = sK[i] * knorm;
            float m = M[r];
            if constexpr (KIND == kRecDelta) m = m - rec_sigm(a_s) * ki * c + rec_sigm(b_s) * ki * vj;
            if constexpr (KIND == kRecGatedDelta) m = rec_sigm(a_s) * (m - ki * c) + rec_sigm(b_s) * ki * vj;
            if constexpr (KIND == kRecOuter) m = rec_sigm(al[i]) * rec_sigm(be[j]) * m + ki * vj;
            if constexpr (KIND == kRecTTT) m = m - rec_sigm(b_s) * ki * (c - vj);
            if constexpr (KIND == kRecTitans) m = rec_sigm(a_s) * m - rec_sigm(b_s) * ki * (c - vj);
            if constexpr (KIND == kRecRWKV7) m = rec_sigm(av[i]) * m - rec_sigm(b_s) * ki * (c - vj);
            if constexpr (KIND == kRecS4) m = sA[r] * m + sRow[i] * vj;
            if constexpr (KIND == kRecMamba) m = __expf(-sA[r] * sRow[i]) * m + sRow[i] * ki * vj;
            bad |= !isfinite(m);
            M[r] = m;
            float qi = q[i];
            if constexpr (FM == 1) qi = qi > 0.f ? qi + 1.f : __expf(qi);
            if constexpr (FM == 2) qi = qi * qi;
            opart += qi * m;
        }
        if constexpr (kNeedC) __syncthreads();  // every c read precedes the partial overwrite
        sPart[g][j] = opart;
        __syncthreads();  // (4) o = phi(q) M
        if (g == 0) {
            float oj = 0.f;
#pragma unroll
            for (int gg = 0; gg < RG; ++gg) oj += sPart[gg][j];
            const size_t oi = (((size_t)b * p.N + t) * p.H + h) * D + j;
            if constexpr (sizeof(T) == 2) static_cast<__nv_bfloat16*>(p.o)[oi] = __float2bfloat16_rn(oj);
            else static_cast<float*>(p.o)[oi] = oj;
        }
    }
    if (bad) atomicOr(p.err, 1);
    if (p.M_out) {
#pragma unroll
        for (int r = 0; r < RP; ++r) p.M_out[(bh * D + g * RP + r) * D + j] = M[r];
    }
}

template <typename T, int D, int FM>
static cudaError_t rec_launch_kind(int kind, const RecParams& p, cudaStream_t st) {
    const dim3 grid(p.H, p.B);
    switch (kind) {
        case kRecDelta: lsm_recurrent_kernel<T, D, kRecDelta, FM><<<grid, 256, 0, st>>>(p); break;
        case kRecGatedDelta: lsm_recurrent_kernel<T, D, kRecGatedDelta, FM><<<grid, 256, 0, st>>>(p); break;
        case kRecOuter: lsm_recurrent_kernel<T, D, kRecOuter, FM><<<grid, 256, 0, st>>>(p); break;
        case kRecTTT: lsm_recurrent_kernel<T, D, kRecTTT, FM><<<grid, 256, 0, st>>>(p); break;
        case kRecTitans: lsm_recurrent_kernel<T, D, kRecTitans, FM><<<grid, 256, 0, st>>>(p); break;
        case kRecRWKV7: lsm_recurrent_kernel<T, D, kRecRWKV7, FM><<<grid, 256, 0, st>>>(p); break;
        case kRecS4: lsm_recurrent_kernel<T, D, kRecS4, FM><<<grid, 256, 0, st>>>(p); break;
        default: lsm_recurrent_kernel<T, D, kRecMamba, FM><<<grid, 256, 0, st>>>(p); break;
    }
    return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t rec_launch(int kind, int fm, const RecParams& p, cudaStream_t st) {
    if (fm == 1) return rec_launch_kind<T, D, 1>(kind, p, st);
    if (fm == 2) return rec_launch_kind<T, D, 2>(kind, p, st);
    return rec_launch_kind<T, D, 0>(kind, p, st);
}

// ====================================================================================
// Backward of the recurrent kinds: the tape VJP of recurrent_step (lsm.hpp:335-441) over
// the sequence, hand-written per kind (tensor.hpp:1178-1215 replays the same chain rule op
// by op).  One CTA per (b, h), the thread layout of the forward (column j, RP rows).
//   phase 1: forward recurrence from M0, the state at every L-token block start saved
//            (ckpt, [B*H][nblk][D][D] fp32);
//   phase 2: blocks last to first -- the block's states recomputed from its checkpoint into
//            scratch ([B*H][L][D][D]: the state entering each token), then tokens last to
//            first: dM += phi(q) dO^T, the per-kind VJP of the update, dM <- dM_prev.
// Reductions over the state's rows (sum over i, per column j) are thread partials plus a
// shared-memory combine; reductions over its columns (sum over j, per row i) go through a
// padded D x (D+1) shared tile (conflict-free row reads).  fp32 throughout.
// Per-kind VJPs (u = k^T dM_next column sums, R = row sums over j; A = sigma(a_s), B = sigma(b_s)):
//   DeltaNet:   dM = dMn - A k u^T;      dk^ = R[dMn (B v - A c)] - A R[M u]
//   GatedDelta: dM = A (dMn - k u^T);    dk^ as DeltaNet; dA = sum dMn (M - k c^T)
//   TTT-like:   dM = {1, A, sigma(a_vec)} dMn - B k u^T;   dk = -B (R[dMn e] + R[M u]), e = c - v
//   GFW:        dM = G dMn;  dk = R[dMn v];  dsa = R[dMn M sb];  dsb = C[dMn M sa]
//   S4 / Mamba: dM = E dMn;  static decay gradients accumulated per element across tokens
// ====================================================================================
struct RecBwdParams {
    RecParams f;             // forward inputs (f.o, f.M_out unused)
    const void* dO;          // [B, N, H, D] in T
    const float* dM_final;   // [B, H, D, D] or null
    void* dq;                // [B, N, H, D] in T
    void* dk;
    void* dv;
    void* da_vec;            // RWKV7 / Mamba [B, N, H, D] in T
    float* da_scal;          // DeltaNet / GatedDeltaNet / Titans [B, N, H]
    float* db_pre;           // [B, N, H]
    void* dalpha;            // GFW / GateLoop [B, N, H, D] in T
    void* dbeta;
    float* ds4_delta_raw;    // [H, D]       (accumulated over the batch: zeroed by the host)
    float* ds4_b;            // [H, D]
    float* ds4_A_raw;        // [H, D, D]
    float* dmamba_A_raw;     // [H, D, D]
    float* dM0;              // [B, H, D, D] or null
    float* ckpt;             // [B*H][nblk][D][D]
    float* scratch;          // [B*H][L][D][D]
    int L, nblk;
};

template <typename T>
__device__ __forceinline__ void rec_st(void* p, size_t i, float x) {
    if constexpr (sizeof(T) == 2) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(x);
    else static_cast<float*>(p)[i] = x;
}
template <int FM>
__device__ __forceinline__ float fmap_grad(float x) {  // d phi / dx
    if constexpr (FM == 1) return x > 0.f ? 1.f : __expf(x);
    else if constexpr (FM == 2) return 2.f * x;
    else return 1.f;
}

template <typename T, int D, int KIND, int FM>
__global__ void __launch_bounds__(256, 1) lsm_recurrent_bwd_kernel(RecBwdParams p) {
    constexpr int RG = 256 / D;
    constexpr int RP = D / RG;
    constexpr bool kVecA = KIND == kRecRWKV7 || KIND == kRecMamba;
    constexpr bool kDelta = KIND == kRecDelta || KIND == kRecGatedDelta;
    constexpr bool kNeedC = kDelta || KIND == kRecTTT || KIND == kRecTitans || KIND == kRecRWKV7;
    constexpr bool kElem = KIND == kRecS4 || KIND == kRecMamba;
    constexpr int NE = 7 * D + 2;  // [q | k | v | a_vec | alpha | beta | dO | a_s, b_s]
    extern __shared__ float sTile[];                  // [D][D + 1] row-reduction tile
    __shared__ float sIn[NE];
    __shared__ float sK[D], sQ[D], sRowA[D], sColB[D];  // k^, phi(q), per-row / per-column gates
    __shared__ float sPart[RG][D];
    __shared__ float sR[4][D];                         // row sums of this token
    __shared__ float sAcc[D];                          // S4: sum over tokens of d incr
    __shared__ float sRed[32];
    __shared__ float sScal[4];
    const RecParams& f = p.f;
    const int h = blockIdx.x, b = blockIdx.y;
    const int tid = threadIdx.x, j = tid % D, g = tid / D, lane = tid & 31, warp = tid >> 5;
    const size_t bh = (size_t)b * f.H + h;
    float* ckpt = p.ckpt + bh * p.nblk * D * D;
    float* scratch = p.scratch + bh * p.L * D * D;

    float sA[kElem ? RP : 1];   // S4: static decay; Mamba: softplus(A_raw)
    float acc[kElem ? RP : 1];  // static-gradient accumulators
#pragma unroll
    for (int r = 0; r < (kElem ? RP : 1); ++r) {
        const int i = g * RP + r;
        sA[r] = 0.f;
        acc[r] = 0.f;
        if constexpr (KIND == kRecS4) {
            const float dl = softplus_f(f.s4_delta_raw[h * D + i]);
            sA[r] = __expf(-softplus_f(f.s4_A_raw[((size_t)h * D + i) * D + j]) * dl);
        }
        if constexpr (KIND == kRecMamba) sA[r] = softplus_f(f.mamba_A_raw[((size_t)h * D + i) * D + j]);
    }
    if (tid < D) sAcc[tid] = 0.f;

    auto load = [&](int t, int e) -> float {
        const size_t row = ((size_t)b * f.N + t) * f.H + h;
        const int seg = e / D, c = e % D;
        switch (seg) {
            case 0: return rec_ld<T>(f.q, row * D + c);
            case 1: return rec_ld<T>(f.k, row * D + c);
            case 2: return rec_ld<T>(f.v, row * D + c);
            case 3: return kVecA ? rec_ld<T>(f.a_vec, row * D + c) : 0.f;
            case 4: return KIND == kRecOuter ? rec_ld<T>(f.alpha, row * D + c) : 0.f;
            case 5: return KIND == kRecOuter ? rec_ld<T>(f.beta, row * D + c) : 0.f;
            case 6: return p.dO ? rec_ld<T>(p.dO, row * D + c) : 0.f;
            default:
                if (c == 0) return f.a_scal ? f.a_scal[row] : 0.f;
                if (c == 1) return f.b_pre ? f.b_pre[row] : 0.f;
                return 0.f;
        }
    };
    // token t's inputs into shared memory, then k^ / phi(q) / per-row and per-column gates
    float knorm = 1.f;
    auto stage = [&](int t, bool with_do) {
        __syncthreads();  // previous token's readers of sIn / sK are done
        for (int e = tid; e < NE; e += 256)
            sIn[e] = (e / D == 6 && !with_do) ? 0.f : load(t, e);
        __syncthreads();
        float kj = 0.f;
        if (tid < D) {
            kj = fmap_t<FM>(sIn[D + tid]);
            sQ[tid] = fmap_t<FM>(sIn[tid]);
            if constexpr (KIND == kRecMamba) sRowA[tid] = softplus_f(sIn[3 * D + tid]);
            if constexpr (KIND == kRecRWKV7) sRowA[tid] = rec_sigm(sIn[3 * D + tid]);
            if constexpr (KIND == kRecOuter) {
                sRowA[tid] = rec_sigm(sIn[4 * D + tid]);
                sColB[tid] = rec_sigm(sIn[5 * D + tid]);
            }
            if constexpr (KIND == kRecS4) sRowA[tid] = softplus_f(f.s4_delta_raw[h * D + tid]) * f.s4_b[h * D + tid];
        }
        if constexpr (kDelta) {
            float sq = kj * kj;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
            if (tid < D && lane == 0) sRed[warp] = sq;
        }
        if (tid < D) sK[tid] = kj;
        __syncthreads();
        knorm = 1.f;
        if constexpr (kDelta) {
            float s2 = 0.f;
#pragma unroll
            for (int w = 0; w < D / 32; ++w) s2 += sRed[w];
            knorm = rsqrtf(s2 + 1e-12f);
        }
    };
    // column sums over the rows: out_j = sum_i X[i][j] (X given per thread for its RP rows)
    auto colsum = [&](const float (&x)[RP]) -> float {
        float part = 0.f;
#pragma unroll
        for (int r = 0; r < RP; ++r) part += x[r];
        __syncthreads();
        sPart[g][j] = part;
        __syncthreads();
        float c = 0.f;
#pragma unroll
        for (int gg = 0; gg < RG; ++gg) c += sPart[gg][j];
        return c;
    };
    // row sums over the columns into sR[slot][i]
    auto rowsum = [&](const float (&x)[RP], int slot) {
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RP; ++r) sTile[(g * RP + r) * (D + 1) + j] = x[r];
        __syncthreads();
        // RG threads per row, each summing D / RG columns; then combine through sPart
        const int i = tid % D, part = tid / D;
        float s = 0.f;
#pragma unroll 8
        for (int c = 0; c < D / RG; ++c) s += sTile[i * (D + 1) + part * (D / RG) + c];
        sPart[part][i] = s;
        __syncthreads();
        if (tid < D) {
            float tot = 0.f;
#pragma unroll
            for (int gg = 0; gg < RG; ++gg) tot += sPart[gg][tid];
            sR[slot][tid] = tot;
        }
    };
    // block-wide sum of one value per thread (result valid in every thread)
    auto blocksum = [&](float v) -> float {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        __syncthreads();
        if (lane == 0) sRed[warp] = v;
        __syncthreads();
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += sRed[w];
        return t;
    };
    // one forward update of M (the state entering the token) with the staged inputs
    auto fwd_update = [&](float (&M)[RP]) {
        float c = 0.f;
        if constexpr (kNeedC) {
            float x[RP];
#pragma unroll
            for (int r = 0; r < RP; ++r) x[r] = sK[g * RP + r] * knorm * M[r];
            c = colsum(x);
        }
        const float vj = sIn[2 * D + j];
        const float a_s = rec_sigm(sIn[7 * D]), b_s = rec_sigm(sIn[7 * D + 1]);
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const int i = g * RP + r;
            const float ki = sK[i] * knorm;
            float m = M[r];
            if constexpr (KIND == kRecDelta) m = m - a_s * ki * c + b_s * ki * vj;
            if constexpr (KIND == kRecGatedDelta) m = a_s * (m - ki * c) + b_s * ki * vj;
            if constexpr (KIND == kRecOuter) m = sRowA[i] * sColB[j] * m + ki * vj;
            if constexpr (KIND == kRecTTT) m = m - b_s * ki * (c - vj);
            if constexpr (KIND == kRecTitans) m = a_s * m - b_s * ki * (c - vj);
            if constexpr (KIND == kRecRWKV7) m = sRowA[i] * m - b_s * ki * (c - vj);
            if constexpr (KIND == kRecS4) m = sA[r] * m + sRowA[i] * vj;
            if constexpr (KIND == kRecMamba) m = __expf(-sA[r] * sRowA[i]) * m + sRowA[i] * ki * vj;
            M[r] = m;
        }
    };

    // ---- phase 1: checkpoints
    float M[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) M[r] = f.M0 ? f.M0[(bh * D + g * RP + r) * D + j] : 0.f;
    for (int t = 0; t < f.N; ++t) {
        if (t % p.L == 0) {
#pragma unroll
            for (int r = 0; r < RP; ++r) ckpt[((size_t)(t / p.L) * D + g * RP + r) * D + j] = M[r];
        }
        stage(t, false);
        fwd_update(M);
    }
    // ---- phase 2: reverse
    float dM[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) dM[r] = p.dM_final ? p.dM_final[(bh * D + g * RP + r) * D + j] : 0.f;
    for (int blk = p.nblk - 1; blk >= 0; --blk) {
        const int t0 = blk * p.L, t1 = min(f.N, t0 + p.L);
#pragma unroll
        for (int r = 0; r < RP; ++r) M[r] = ckpt[((size_t)blk * D + g * RP + r) * D + j];
        for (int t = t0; t < t1; ++t) {
#pragma unroll
            for (int r = 0; r < RP; ++r) scratch[((size_t)(t - t0) * D + g * RP + r) * D + j] = M[r];
            if (t + 1 < t1) {  // the last token's successor state is not needed
                stage(t, false);
                fwd_update(M);
            }
        }
        for (int t = t1 - 1; t >= t0; --t) {
            float Mp[RP];
#pragma unroll
            for (int r = 0; r < RP; ++r) Mp[r] = scratch[((size_t)(t - t0) * D + g * RP + r) * D + j];
            stage(t, true);
            const float vj = sIn[2 * D + j], doj = sIn[6 * D + j];
            const float a_s = rec_sigm(sIn[7 * D]), b_s = rec_sigm(sIn[7 * D + 1]);
            float x[RP];
            float c = 0.f;
            if constexpr (kNeedC) {
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = sK[g * RP + r] * knorm * Mp[r];
                c = colsum(x);
            }
            // the state after the token (recomputed elementwise, c known) times dO, and the
            // output adjoint dM += phi(q) dO^T
#pragma unroll
            for (int r = 0; r < RP; ++r) {
                const int i = g * RP + r;
                const float ki = sK[i] * knorm;
                float m = Mp[r];
                if constexpr (KIND == kRecDelta) m = m - a_s * ki * c + b_s * ki * vj;
                if constexpr (KIND == kRecGatedDelta) m = a_s * (m - ki * c) + b_s * ki * vj;
                if constexpr (KIND == kRecOuter) m = sRowA[i] * sColB[j] * m + ki * vj;
                if constexpr (KIND == kRecTTT) m = m - b_s * ki * (c - vj);
                if constexpr (KIND == kRecTitans) m = a_s * m - b_s * ki * (c - vj);
                if constexpr (KIND == kRecRWKV7) m = sRowA[i] * m - b_s * ki * (c - vj);
                if constexpr (KIND == kRecS4) m = sA[r] * m + sRowA[i] * vj;
                if constexpr (KIND == kRecMamba) m = __expf(-sA[r] * sRowA[i]) * m + sRowA[i] * ki * vj;
                x[r] = m * doj;
                dM[r] += sQ[i] * doj;
            }
            rowsum(x, 0);  // d phi(q)_i
            const size_t row = ((size_t)b * f.N + t) * f.H + h;
            // u_j = sum_i k^_i dMn_ij (k^: the key of the update, delta: normalised)
            float u = 0.f;
            if constexpr (KIND != kRecS4) {
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    const int i = g * RP + r;
                    const float kk = KIND == kRecMamba ? sRowA[i] * sK[i] : sK[i] * knorm;
                    x[r] = kk * dM[r];
                }
                u = colsum(x);
            } else {
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = sRowA[g * RP + r] * dM[r];
                u = colsum(x);  // dv_j
            }
            float dvj = 0.f, dscal_a = 0.f, dscal_b = 0.f;
            if constexpr (kDelta) {
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * (b_s * vj - a_s * c);
                rowsum(x, 1);
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = Mp[r] * u;
                rowsum(x, 2);
                dvj = b_s * u;
                const float uc = (g == 0) ? u * c : 0.f, uv = (g == 0) ? u * vj : 0.f;
                if constexpr (KIND == kRecDelta) {
                    dscal_a = -blocksum(uc);
                } else {
                    float part = 0.f;
#pragma unroll
                    for (int r = 0; r < RP; ++r) part += dM[r] * (Mp[r] - sK[g * RP + r] * knorm * c);
                    dscal_a = blocksum(part);
                }
                dscal_b = blocksum(uv);
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    const float ki = sK[g * RP + r] * knorm;
                    dM[r] = KIND == kRecDelta ? dM[r] - a_s * ki * u : a_s * (dM[r] - ki * u);
                }
            } else if constexpr (KIND == kRecTTT || KIND == kRecTitans || KIND == kRecRWKV7) {
                const float ej = c - vj;
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * ej;
                rowsum(x, 1);
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = Mp[r] * u;
                rowsum(x, 2);
                if constexpr (KIND == kRecRWKV7) {
#pragma unroll
                    for (int r = 0; r < RP; ++r) x[r] = dM[r] * Mp[r];
                    rowsum(x, 3);
                }
                dvj = b_s * u;
                dscal_b = -blocksum(g == 0 ? u * ej : 0.f);
                if constexpr (KIND == kRecTitans) {
                    float part = 0.f;
#pragma unroll
                    for (int r = 0; r < RP; ++r) part += dM[r] * Mp[r];
                    dscal_a = blocksum(part);
                }
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    const int i = g * RP + r;
                    const float fac = KIND == kRecTTT ? 1.f : (KIND == kRecTitans ? a_s : sRowA[i]);
                    dM[r] = fac * dM[r] - b_s * sK[i] * u;
                }
            } else if constexpr (KIND == kRecOuter) {
                dvj = u;
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * vj;
                rowsum(x, 1);
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * Mp[r] * sColB[j];
                rowsum(x, 2);
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * Mp[r] * sRowA[g * RP + r];
                const float dsb = colsum(x);
                if (g == 0) rec_st<T>(p.dbeta, row * D + j, dsb * sColB[j] * (1.f - sColB[j]));
#pragma unroll
                for (int r = 0; r < RP; ++r) dM[r] *= sRowA[g * RP + r] * sColB[j];
            } else if constexpr (KIND == kRecS4) {
                dvj = u;
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * vj;
                rowsum(x, 1);
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    acc[r] += dM[r] * Mp[r];
                    dM[r] *= sA[r];
                }
            } else {  // Mamba
                dvj = u;
#pragma unroll
                for (int r = 0; r < RP; ++r) x[r] = dM[r] * vj;
                rowsum(x, 1);
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    const float dl = sRowA[g * RP + r];
                    const float E = __expf(-sA[r] * dl);
                    x[r] = dM[r] * Mp[r] * E * sA[r];
                    acc[r] += dM[r] * Mp[r] * E * (-dl);
                    dM[r] *= E;
                }
                rowsum(x, 2);
            }
            __syncthreads();  // sR complete
            // per-row gradients (one thread per row i = tid < D)
            if (tid < D) {
                const int i = tid;
                const float qi = sIn[i], ki_raw = sIn[D + i];
                rec_st<T>(p.dq, row * D + i, sR[0][i] * fmap_grad<FM>(qi));
                float dphik = 0.f;
                if constexpr (kDelta) dphik = sR[1][i] - a_s * sR[2][i];  // d k^ (normalised key)
                if constexpr (KIND == kRecTTT || KIND == kRecTitans || KIND == kRecRWKV7)
                    dphik = -b_s * (sR[1][i] + sR[2][i]);
                if constexpr (KIND == kRecOuter) {
                    dphik = sR[1][i];
                    const float sa = sRowA[i];
                    rec_st<T>(p.dalpha, row * D + i, sR[2][i] * sa * (1.f - sa));
                }
                if constexpr (KIND == kRecRWKV7) {
                    const float sa = sRowA[i];
                    rec_st<T>(p.da_vec, row * D + i, sR[3][i] * sa * (1.f - sa));
                }
                if constexpr (KIND == kRecS4) sAcc[i] += sR[1][i];
                if constexpr (KIND == kRecMamba) {
                    const float dl = sRowA[i];
                    dphik = sR[1][i] * dl;
                    const float ddl = sR[1][i] * sK[i] - sR[2][i];
                    rec_st<T>(p.da_vec, row * D + i, ddl * rec_sigm(sIn[3 * D + i]));
                }
                sRowA[i] = dphik;  // reuse: d(k^) per row for the normalisation backward below
            }
            if constexpr (kDelta) {
                // k^ = phi(k) / |phi(k)|: d phi(k) = (d k^ - k^ (k^ . d k^)) / |phi(k)|
                __syncthreads();
                const float dot = blocksum(tid < D ? sRowA[tid] * sK[tid] * knorm : 0.f);
                if (tid < D) {
                    const float kh = sK[tid] * knorm;
                    sRowA[tid] = (sRowA[tid] - kh * dot) * knorm;
                }
            }
            __syncthreads();
            if (tid < D) {
                const float dk = KIND == kRecS4 ? 0.f : sRowA[tid] * fmap_grad<FM>(sIn[D + tid]);
                rec_st<T>(p.dk, row * D + tid, dk);
            }
            if (g == 0) rec_st<T>(p.dv, row * D + j, dvj);
            if (tid == 0) {
                if (p.da_scal) p.da_scal[row] = dscal_a * a_s * (1.f - a_s);
                if (p.db_pre) p.db_pre[row] = dscal_b * b_s * (1.f - b_s);
            }
        }
    }
    if (p.dM0) {
#pragma unroll
        for (int r = 0; r < RP; ++r) p.dM0[(bh * D + g * RP + r) * D + j] = dM[r];
    }
    // static parameters (summed over the batch)
    if constexpr (KIND == kRecS4) {
        // sA = exp(-softplus(A_raw) delta), delta = softplus(delta_raw), incr = delta * b
        float x[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const int i = g * RP + r;
            const float araw = f.s4_A_raw[((size_t)h * D + i) * D + j];
            const float dl = softplus_f(f.s4_delta_raw[h * D + i]);
            atomicAdd(&p.ds4_A_raw[((size_t)h * D + i) * D + j], acc[r] * sA[r] * (-dl) * rec_sigm(araw));
            x[r] = acc[r] * sA[r] * (-softplus_f(araw));
        }
        rowsum(x, 0);
        __syncthreads();
        if (tid < D) {
            const float draw = f.s4_delta_raw[h * D + tid], dl = softplus_f(draw), bb = f.s4_b[h * D + tid];
            const float ddl = sR[0][tid] + sAcc[tid] * bb;
            atomicAdd(&p.ds4_delta_raw[h * D + tid], ddl * rec_sigm(draw));
            atomicAdd(&p.ds4_b[h * D + tid], sAcc[tid] * dl);
        }
    }
    if constexpr (KIND == kRecMamba) {
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const int i = g * RP + r;
            const float araw = f.mamba_A_raw[((size_t)h * D + i) * D + j];
            atomicAdd(&p.dmamba_A_raw[((size_t)h * D + i) * D + j], acc[r] * rec_sigm(araw));
        }
    }
}

template <typename T, int D>
constexpr int rec_bwd_smem() { return D * (D + 1) * 4; }

template <typename T, int D, int FM>
static cudaError_t rec_bwd_launch_kind(int kind, const RecBwdParams& p, cudaStream_t st) {
    const dim3 grid(p.f.H, p.f.B);
    constexpr int smem = rec_bwd_smem<T, D>();
    auto go = [&](auto kern) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, 256, smem, st>>>(p);
        return cudaGetLastError();
    };
    switch (kind) {
        case kRecDelta: return go(lsm_recurrent_bwd_kernel<T, D, kRecDelta, FM>);
        case kRecGatedDelta: return go(lsm_recurrent_bwd_kernel<T, D, kRecGatedDelta, FM>);
        case kRecOuter: return go(lsm_recurrent_bwd_kernel<T, D, kRecOuter, FM>);
        case kRecTTT: return go(lsm_recurrent_bwd_kernel<T, D, kRecTTT, FM>);
        case kRecTitans: return go(lsm_recurrent_bwd_kernel<T, D, kRecTitans, FM>);
        case kRecRWKV7: return go(lsm_recurrent_bwd_kernel<T, D, kRecRWKV7, FM>);
        case kRecS4: return go(lsm_recurrent_bwd_kernel<T, D, kRecS4, FM>);
        default: return go(lsm_recurrent_bwd_kernel<T, D, kRecMamba, FM>);
    }
}

template <typename T, int D>
static cudaError_t rec_bwd_launch(int kind, int fm, const RecBwdParams& p, cudaStream_t st) {
    if (fm == 1) return rec_bwd_launch_kind<T, D, 1>(kind, p, st);
    if (fm == 2) return rec_bwd_launch_kind<T, D, 2>(kind, p, st);
    return rec_bwd_launch_kind<T, D, 0>(kind, p, st);
}

}  // namespace lmoe_dev

using namespace lmoe_host;

namespace {
// LsmInstance -> recurrence kind of this file, or -1
int rec_kind(int inst) {
    switch (inst) {
        case LMOE_DELTANET: return lmoe_dev::kRecDelta;
        case LMOE_GATED_DELTANET: return lmoe_dev::kRecGatedDelta;
        case LMOE_GFW: case LMOE_GATELOOP: return lmoe_dev::kRecOuter;
        case LMOE_TTT: return lmoe_dev::kRecTTT;
        case LMOE_TITANS: return lmoe_dev::kRecTitans;
        case LMOE_RWKV7: return lmoe_dev::kRecRWKV7;
        case LMOE_S4: return lmoe_dev::kRecS4;
        case LMOE_MAMBA: return lmoe_dev::kRecMamba;
        default: return -1;
    }
}
}  // namespace

extern "C" int lmoe_lsm_fwd_recurrent(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                                      const void* q, const void* k, const void* v,
                                      const lmoe_lsm_recurrent_inputs* in, const float* M0, void* o, float* M_out,
                                      void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        if (!desc) throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd_recurrent: null descriptor");
        if (N < 1 || B < 1 || H < 1) throw Error(LMOE_ERR_ARG, "lsm_forward_sequential: need N >= 1 rows");
        if (!q || !k || !v || !o || !in) throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd_recurrent: null tensor");
        const int kind = rec_kind(desc->instance);
        if (kind < 0)
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd_recurrent: instance has a chunk-parallel form (use lmoe_lsm_fwd)");
        if (desc->use_normalizer)
            throw Error(LMOE_ERR_ARG, "LsmSpec: normalizer unsupported for instance " +
                                          std::string(instance_name(desc->instance)));
        if (!((dtype == LMOE_BF16 && D == 128) || (dtype == LMOE_F32 && D == 64)))
            throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_lsm_fwd: supported (dtype, head_dim) pairs are (bf16, 128) and (f32, 64)");
        const char* need = nullptr;  // required gate inputs per kind (LsmGates, lsm.hpp:206-247)
        switch (kind) {
            case lmoe_dev::kRecDelta: case lmoe_dev::kRecGatedDelta: case lmoe_dev::kRecTitans:
                if (!in->a_scal || !in->b_pre) need = "a_pre (N) and b_pre (N)";
                break;
            case lmoe_dev::kRecTTT: if (!in->b_pre) need = "b_pre (N)"; break;
            case lmoe_dev::kRecRWKV7: if (!in->a_vec || !in->b_pre) need = "a_pre (N, d_k) and b_pre (N)"; break;
            case lmoe_dev::kRecOuter: if (!in->alpha_pre || !in->beta_pre) need = "alpha_pre and beta_pre"; break;
            case lmoe_dev::kRecS4:
                if (!in->s4_delta_raw || !in->s4_b || !in->s4_A_raw) need = "s4_delta_raw, s4_b and s4_A_raw";
                break;
            default: if (!in->a_vec || !in->mamba_A_raw) need = "a_pre (N, d_k) and mamba_A_raw"; break;
        }
        if (need)
            throw Error(LMOE_ERR_ARG, std::string("lmoe_lsm_fwd_recurrent: instance ") + instance_name(desc->instance) +
                                          " needs " + need);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (!workspace || workspace_bytes < 64)
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd_recurrent: workspace too small (need 64 bytes)");
        int* err = static_cast<int*>(workspace);
        LMOE_CUDA_CHECK(cudaMemsetAsync(err, 0, sizeof(int), st));
        lmoe_dev::RecParams p{B, N, H, q, k, v, in->a_vec, in->a_scal, in->b_pre, in->alpha_pre, in->beta_pre,
                              in->s4_delta_raw, in->s4_b, in->s4_A_raw, in->mamba_A_raw, M0, o, M_out, err};
        if (dtype == LMOE_BF16) LMOE_CUDA_CHECK((lmoe_dev::rec_launch<__nv_bfloat16, 128>(kind, desc->feature_map, p, st)));
        else LMOE_CUDA_CHECK((lmoe_dev::rec_launch<float, 64>(kind, desc->feature_map, p, st)));
        ++g_launch_count;
        if (desc->flags & LMOE_FLAG_CHECK) {
            int e = 0;
            LMOE_CUDA_CHECK(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
            LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
            if (e)
                throw Error(LMOE_ERR_NONFINITE, std::string("non-finite memory state in instance ") +
                                                    instance_name(desc->instance));
        }
    });
}

namespace {
constexpr int kRecBwdBlock = 32;  // tokens between checkpoints (scratch holds one block's states)
size_t rec_bwd_ws(int B, int N, int H, int D) {
    const size_t nblk = (size_t)(N + kRecBwdBlock - 1) / kRecBwdBlock;
    return 256 + (size_t)B * H * (nblk + kRecBwdBlock) * D * D * 4;
}
// shared argument checks of the recurrent entry points; returns the kernel kind
int rec_check(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype, const void* q, const void* k,
              const void* v, const lmoe_lsm_recurrent_inputs* in, const char* fn) {
    if (!desc) throw Error(LMOE_ERR_ARG, std::string(fn) + ": null descriptor");
    if (N < 1 || B < 1 || H < 1) throw Error(LMOE_ERR_ARG, "lsm_forward_sequential: need N >= 1 rows");
    if (!q || !k || !v || !in) throw Error(LMOE_ERR_ARG, std::string(fn) + ": null tensor");
    const int kind = rec_kind(desc->instance);
    if (kind < 0) throw Error(LMOE_ERR_ARG, std::string(fn) + ": instance has a chunk-parallel form (use lmoe_lsm_fwd)");
    if (desc->use_normalizer)
        throw Error(LMOE_ERR_ARG, "LsmSpec: normalizer unsupported for instance " + std::string(instance_name(desc->instance)));
    if (!((dtype == LMOE_BF16 && D == 128) || (dtype == LMOE_F32 && D == 64)))
        throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_lsm_fwd: supported (dtype, head_dim) pairs are (bf16, 128) and (f32, 64)");
    const char* need = nullptr;  // required gate inputs per kind (LsmGates, lsm.hpp:206-247)
    switch (kind) {
        case lmoe_dev::kRecDelta: case lmoe_dev::kRecGatedDelta: case lmoe_dev::kRecTitans:
            if (!in->a_scal || !in->b_pre) need = "a_pre (N) and b_pre (N)";
            break;
        case lmoe_dev::kRecTTT: if (!in->b_pre) need = "b_pre (N)"; break;
        case lmoe_dev::kRecRWKV7: if (!in->a_vec || !in->b_pre) need = "a_pre (N, d_k) and b_pre (N)"; break;
        case lmoe_dev::kRecOuter: if (!in->alpha_pre || !in->beta_pre) need = "alpha_pre and beta_pre"; break;
        case lmoe_dev::kRecS4:
            if (!in->s4_delta_raw || !in->s4_b || !in->s4_A_raw) need = "s4_delta_raw, s4_b and s4_A_raw";
            break;
        default: if (!in->a_vec || !in->mamba_A_raw) need = "a_pre (N, d_k) and mamba_A_raw"; break;
    }
    if (need)
        throw Error(LMOE_ERR_ARG, std::string(fn) + ": instance " + instance_name(desc->instance) + " needs " + need);
    return kind;
}
}  // namespace

extern "C" size_t lmoe_lsm_bwd_recurrent_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                                        lmoe_dtype dtype) {
    (void)desc;
    (void)dtype;
    if (B < 1 || N < 1 || H < 1 || D < 1) return 0;
    return rec_bwd_ws(B, N, H, D);
}

// The tape backward of lsm_forward_sequential / lsm_forward_chunked for the recurrent kinds
// (tensor.hpp:1178-1215 over recurrent_step, lsm.hpp:335-441).
extern "C" int lmoe_lsm_bwd_recurrent(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                                      const void* q, const void* k, const void* v,
                                      const lmoe_lsm_recurrent_inputs* in, const float* M0, const void* dO,
                                      const float* dM_final, void* dq, void* dk, void* dv,
                                      const lmoe_lsm_recurrent_grads* grads, float* dM0, void* workspace,
                                      size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        const int kind = rec_check(desc, B, N, H, D, dtype, q, k, v, in, "lmoe_lsm_bwd_recurrent");
        if (!dO || !dq || !dk || !dv || !grads) throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd_recurrent: null gradient buffer");
        const char* miss = nullptr;
        switch (kind) {
            case lmoe_dev::kRecDelta: case lmoe_dev::kRecGatedDelta: case lmoe_dev::kRecTitans:
                if (!grads->da_scal || !grads->db_pre) miss = "da_pre (N) and db_pre (N)";
                break;
            case lmoe_dev::kRecTTT: if (!grads->db_pre) miss = "db_pre (N)"; break;
            case lmoe_dev::kRecRWKV7: if (!grads->da_vec || !grads->db_pre) miss = "da_pre (N, d_k) and db_pre (N)"; break;
            case lmoe_dev::kRecOuter: if (!grads->dalpha_pre || !grads->dbeta_pre) miss = "dalpha_pre and dbeta_pre"; break;
            case lmoe_dev::kRecS4:
                if (!grads->ds4_delta_raw || !grads->ds4_b || !grads->ds4_A_raw) miss = "ds4_delta_raw, ds4_b, ds4_A_raw";
                break;
            default: if (!grads->da_vec || !grads->dmamba_A_raw) miss = "da_pre (N, d_k) and dmamba_A_raw"; break;
        }
        if (miss) throw Error(LMOE_ERR_ARG, std::string("lmoe_lsm_bwd_recurrent: instance ") +
                                                instance_name(desc->instance) + " needs gradient buffers " + miss);
        const size_t need = rec_bwd_ws(B, N, H, D);
        if (!workspace || workspace_bytes < need)
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd_recurrent: workspace too small (need " + std::to_string(need) + " bytes)");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        const int nblk = (N + kRecBwdBlock - 1) / kRecBwdBlock;
        // static-parameter gradients are summed over the batch by atomics
        if (kind == lmoe_dev::kRecS4) {
            LMOE_CUDA_CHECK(cudaMemsetAsync(grads->ds4_delta_raw, 0, (size_t)H * D * 4, st));
            LMOE_CUDA_CHECK(cudaMemsetAsync(grads->ds4_b, 0, (size_t)H * D * 4, st));
            LMOE_CUDA_CHECK(cudaMemsetAsync(grads->ds4_A_raw, 0, (size_t)H * D * D * 4, st));
        }
        if (kind == lmoe_dev::kRecMamba)
            LMOE_CUDA_CHECK(cudaMemsetAsync(grads->dmamba_A_raw, 0, (size_t)H * D * D * 4, st));
        lmoe_dev::RecBwdParams p{};
        p.f = lmoe_dev::RecParams{B, N, H, q, k, v, in->a_vec, in->a_scal, in->b_pre, in->alpha_pre, in->beta_pre,
                                  in->s4_delta_raw, in->s4_b, in->s4_A_raw, in->mamba_A_raw, M0, nullptr, nullptr,
                                  nullptr};
        p.dO = dO;
        p.dM_final = dM_final;
        p.dq = dq;
        p.dk = dk;
        p.dv = dv;
        p.da_vec = grads->da_vec;
        p.da_scal = grads->da_scal;
        p.db_pre = grads->db_pre;
        p.dalpha = grads->dalpha_pre;
        p.dbeta = grads->dbeta_pre;
        p.ds4_delta_raw = grads->ds4_delta_raw;
        p.ds4_b = grads->ds4_b;
        p.ds4_A_raw = grads->ds4_A_raw;
        p.dmamba_A_raw = grads->dmamba_A_raw;
        p.dM0 = dM0;
        p.ckpt = reinterpret_cast<float*>(ws + 256);
        p.scratch = p.ckpt + (size_t)B * H * nblk * D * D;
        p.L = kRecBwdBlock;
        p.nblk = nblk;
        if (dtype == LMOE_BF16) LMOE_CUDA_CHECK((lmoe_dev::rec_bwd_launch<__nv_bfloat16, 128>(kind, desc->feature_map, p, st)));
        else LMOE_CUDA_CHECK((lmoe_dev::rec_bwd_launch<float, 64>(kind, desc->feature_map, p, st)));
        ++g_launch_count;
    });
}
