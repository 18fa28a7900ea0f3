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
