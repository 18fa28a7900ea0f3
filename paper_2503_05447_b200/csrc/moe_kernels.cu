// moe_kernels.cu -- Linear-MoE expert layer on sm_100a.
//
// Restates MoeLayer::forward (/root/reference/proj/include/lmoe/moe.hpp:133-149):
//   route (moe.hpp:58-85)           warp-per-token top-k on fp32 logits, ties to the lower id,
//                                   ids ascending, renormalised gates, full softmax, counts
//   dispatch (moe.hpp:137-143)      stable counting sort by expert (token-ascending per
//                                   expert) -> permuted rows x_perm
//   Expert::forward (moe.hpp:45-47) grouped tcgen05 GEMMs: H = silu(X Wg) * (X Wu) fused in
//                                   one kernel (two TMEM accumulators), then Y = H Wd
//   combine (moe.hpp:144-146)       y[t] = sum over the token's experts, in ascending expert
//                                   order, of gate * Y[perm row]
//   load_balance_loss (:90-103)     E * sum_e f_e P_e
#include "moe_kernels.cuh"

namespace lmoe_dev {

// ====================================================================================
// Grouped GEMM  C[rows of group g] = A[rows] (K-major, bf16) x B_g (MN-major [K][N], bf16)
// Persistent: one CTA per SM walks the (128-row M tile, BN-column N tile) list, M-major so
// the CTAs running at once share A tiles in L2.  The smem ring runs continuously across
// tiles; the TMEM accumulator is double-buffered so the epilogue of tile i overlaps the
// MMAs of tile i+1.
// warps: 0 TMA producer, 1 MMA issuer, 2..5 epilogue (one thread per output row)
// ====================================================================================
template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    moe_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
             const __grid_constant__ CUtensorMap tmB1, GemmParams p) {
    constexpr int NB = (EPI == kEpiSwiGLU) ? 2 : 1;         // B operands per stage
    constexpr int A_BYTES = 128 * 128;                       // 128 rows x 64 K (bf16)
    constexpr int B_BYTES = 64 * 2 * BN;                     // 64 K rows x BN cols (bf16)
    constexpr int STAGE = A_BYTES + NB * B_BYTES;
    constexpr int NST = gemm_stages<BN, EPI>();
    constexpr uint32_t ACOLS = NB * BN;                      // accumulator columns per buffer
    constexpr uint32_t TCOLS = 2 * ACOLS;                    // two buffers (128 / 256 / 512)
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
    uint64_t* full = bars;             // [NST]
    uint64_t* empty = bars + NST;      // [NST]
    uint64_t* acc_full = bars + 2 * NST;   // [2]
    uint64_t* acc_empty = acc_full + 2;    // [2]
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int total = *p.num_tiles * p.ntn;
    const int kblocks = p.K / 64;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], kGemmEpiThreads); }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<TCOLS>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmA);
            tma_prefetch(&tmB0);
            if (NB == 2) tma_prefetch(&tmB1);
            int it = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int mt = t / p.ntn, n0 = (t % p.ntn) * BN;
                const int g = p.tile_group[mt], row0 = p.tile_row0[mt];
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const int s = it % NST;
                    if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
                    uint8_t* st = smem + s * STAGE;
                    mbar_expect_tx(&full[s], STAGE);
                    tma_load_2d(st, &tmA, &full[s], kb * 64, row0);
#pragma unroll
                    for (int nb = 0; nb < BN / 64; ++nb) {
                        tma_load_3d(st + A_BYTES + nb * 8192, &tmB0, &full[s], n0 + nb * 64, kb * 64, g);
                        if constexpr (NB == 2)
                            tma_load_3d(st + A_BYTES + B_BYTES + nb * 8192, &tmB1, &full[s], n0 + nb * 64, kb * 64, g);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // SwiGLU: the gate and up B tiles sit back to back in the stage (N atoms 8 KB apart),
            // so one N = 2 BN MMA covers both and reads the A tile once per K step
            constexpr uint32_t idesc = umma_idesc(1, 0, 1, 128, NB * BN);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
                const int buf = lt & 1;
                if (lt >= 2) mbar_wait(&acc_empty[buf], ((lt >> 1) - 1) & 1);  // epilogue drained it
                tc_fence_after();
                const uint32_t acc_t = tmem + buf * ACOLS;
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const int s = it % NST;
                    mbar_wait(&full[s], (it / NST) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + s * STAGE);
                    const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ad = umma_desc_sw128(a0 + kk * 32, 16, 1024);
                        const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                        mma_ss_f16(acc_t, ad, umma_desc_sw128(b0 + kk * 2048, 8192, 1024), idesc, acc);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&acc_full[buf]);
            }
        }
    } else {
        // epilogue: thread (quarter q, lane) owns output row q*32 + lane of the tile; the two
        // warps of a lane quarter take one column half each
        const int q = warp & 3;
        constexpr int EH = kGemmEpiThreads / 128;  // epilogue warps per lane quarter
        const int ch = (warp - 2) / 4;             // this warp's column part
        const int r = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        int lt = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
            const int buf = lt & 1;
            const int mt = t / p.ntn, n0 = (t % p.ntn) * BN;
            const int row0 = p.tile_row0[mt];
            const int rows_left = p.group_end[p.tile_group[mt]] - row0;  // valid rows (<= 128)
            mbar_wait(&acc_full[buf], (lt >> 1) & 1);
            tc_fence_after();
            const uint32_t acc_t = tmem + buf * ACOLS;
            const bool valid = r < rows_left;
            const size_t grow = (size_t)row0 + (valid ? r : 0);
#pragma unroll 1
            for (int cb = ch * (BN / EH); cb < (ch + 1) * (BN / EH); cb += 32) {
                uint32_t a[32];
                tmem_ld32(acc_t + lane_off + cb, a);
                if constexpr (EPI == kEpiSwiGLU) {
                    uint32_t u[32];
                    tmem_ld32(acc_t + lane_off + BN + cb, u);
                    tmem_wait_ld();
                    if (valid) {
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.C) + grow * p.ldc + n0 + cb;
#pragma unroll
                        for (int j = 0; j < 32; j += 8) {
                            uint4 v;
                            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float g0 = __uint_as_float(a[j + 2 * e]), g1 = __uint_as_float(a[j + 2 * e + 1]);
                                const float u0 = __uint_as_float(u[j + 2 * e]), u1 = __uint_as_float(u[j + 2 * e + 1]);
                                w[e] = pack_bf16(silu_f(g0) * u0, silu_f(g1) * u1);
                            }
                            *reinterpret_cast<uint4*>(dst + j) = v;
                        }
                    }
                } else if constexpr (EPI == kEpiBF16) {
                    tmem_wait_ld();
                    if (valid) {
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.C) + grow * p.ldc + n0 + cb;
#pragma unroll
                        for (int j = 0; j < 32; j += 8) {
                            uint4 v;
                            v.x = pack_bf16(__uint_as_float(a[j]), __uint_as_float(a[j + 1]));
                            v.y = pack_bf16(__uint_as_float(a[j + 2]), __uint_as_float(a[j + 3]));
                            v.z = pack_bf16(__uint_as_float(a[j + 4]), __uint_as_float(a[j + 5]));
                            v.w = pack_bf16(__uint_as_float(a[j + 6]), __uint_as_float(a[j + 7]));
                            *reinterpret_cast<uint4*>(dst + j) = v;
                        }
                    }
                } else {  // fp32
                    tmem_wait_ld();
                    if (valid) {
                        float* dst = reinterpret_cast<float*>(p.C) + grow * p.ldc + n0 + cb;
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<float4*>(dst + j) =
                                make_float4(__uint_as_float(a[j]), __uint_as_float(a[j + 1]),
                                            __uint_as_float(a[j + 2]), __uint_as_float(a[j + 3]));
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<TCOLS>(tmem);
}

template __global__ void moe_gemm<128, kEpiSwiGLU>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, GemmParams);
template __global__ void moe_gemm<256, kEpiBF16>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                 const __grid_constant__ CUtensorMap, GemmParams);
template __global__ void moe_gemm<128, kEpiBF16>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                 const __grid_constant__ CUtensorMap, GemmParams);
template __global__ void moe_gemm<64, kEpiF32>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                               const __grid_constant__ CUtensorMap, GemmParams);

// ====================================================================================
// Routing: each warp walks tokens; lane owns experts lane + 32 i (i < NE, E <= 32 NE);
// counts and probability column sums stay in registers until one shared-memory atomic per
// expert per warp, then one global atomic per block and expert.
// ====================================================================================
template <int NE>
__global__ void __launch_bounds__(256) moe_route(const float* __restrict__ logits, int T, int E, int K,
                                                 int* __restrict__ ids, float* __restrict__ gates,
                                                 float* __restrict__ probs, int* __restrict__ counts,
                                                 float* __restrict__ prob_colsum) {
    // per-block expert counts (integer atomics) and probability column sums: each warp keeps
    // its own row of partial sums, summed in warp order, and the block writes its partial to
    // prob_colsum[block][e] (no float atomics: the aux loss is bitwise repeatable)
    __shared__ int s_cnt[32 * NE];
    __shared__ float s_ps[8][32 * NE];
    for (int i = threadIdx.x; i < 32 * NE; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wglobal = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * (blockDim.x / 32);
    const float NEG = -INFINITY;
    bool has[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) has[i] = lane + 32 * i < E;
    int cnt[NE];
    float ps[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) { cnt[i] = 0; ps[i] = 0.f; }
    // logits map to order-preserving unsigned keys (0 = taken / absent)
    auto key = [](float f) -> unsigned {
        const unsigned u = __float_as_uint(f + 0.f);  // -0 -> +0: equal logits tie on id
        return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    };
    for (int t = wglobal; t < T; t += nwarps) {
        const float* l = logits + (size_t)t * E;
        float v[NE];
#pragma unroll
        for (int i = 0; i < NE; ++i) v[i] = has[i] ? l[lane + 32 * i] : NEG;
        // full softmax (tensor.hpp:767-789): max-subtracted over all logits
        float mx = v[0];
#pragma unroll
        for (int i = 1; i < NE; ++i) mx = fmaxf(mx, v[i]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        float e[NE];
        float zs = 0.f;
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            e[i] = has[i] ? __expf(v[i] - mx) : 0.f;
            zs += e[i];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) zs += __shfl_xor_sync(0xFFFFFFFFu, zs, o);
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const float pr = e[i] / zs;
            if (probs && has[i]) probs[(size_t)t * E + lane + 32 * i] = pr;
            ps[i] += pr;
        }
        // top-k by repeated warp argmax: larger logit first, ties -> lower id (moe.hpp:70-75).
        // Per round: the lane's best untaken candidate (first maximum in ascending id order),
        // one redux.sync max over the keys, one redux.sync min over the ids holding it.
        unsigned k[NE];
        bool sel[NE];
#pragma unroll
        for (int i = 0; i < NE; ++i) { k[i] = has[i] ? key(v[i]) : 0u; sel[i] = false; }
        unsigned topk = 0u;
        for (int r = 0; r < K; ++r) {
            unsigned cb = 0u, cid = 0xFFFFFFFFu;
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const unsigned c = sel[i] ? 0u : k[i];
                if (c > cb) { cb = c; cid = (unsigned)(lane + 32 * i); }
            }
            const unsigned best = __reduce_max_sync(0xFFFFFFFFu, cb);
            const unsigned bid = __reduce_min_sync(0xFFFFFFFFu, (cb == best && cb != 0u) ? cid : 0xFFFFFFFFu);
            if (r == 0) topk = best;
#pragma unroll
            for (int i = 0; i < NE; ++i)
                if ((unsigned)(lane + 32 * i) == bid) sel[i] = true;
        }
        const float top = __uint_as_float((topk & 0x80000000u) ? (topk & 0x7FFFFFFFu) : ~topk);
        // ascending ids of the selection (moe.hpp:77) + masked softmax (max = top-1 logit)
        float g[NE];
        float gz = 0.f;
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            g[i] = sel[i] ? __expf(v[i] - top) : 0.f;
            gz += g[i];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) gz += __shfl_xor_sync(0xFFFFFFFFu, gz, o);
        int base = 0;
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const unsigned m = __ballot_sync(0xFFFFFFFFu, sel[i]);
            if (sel[i]) {
                const int slot = base + __popc(m & ((1u << lane) - 1u));
                ids[(size_t)t * K + slot] = lane + 32 * i;
                gates[(size_t)t * K + slot] = g[i] / gz;
                ++cnt[i];
            }
            base += __popc(m);
        }
    }
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        s_ps[warp][lane + 32 * i] = ps[i];
        if (has[i] && cnt[i]) atomicAdd(&s_cnt[lane + 32 * i], cnt[i]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
        if (s_cnt[i]) atomicAdd(&counts[i], s_cnt[i]);
        if (prob_colsum) {
            float t = 0.f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_ps[w][i];
            prob_colsum[(size_t)blockIdx.x * E + i] = t;
        }
    }
}
template __global__ void moe_route<1>(const float*, int, int, int, int*, float*, float*, int*, float*);
template __global__ void moe_route<2>(const float*, int, int, int, int*, float*, float*, int*, float*);
template __global__ void moe_route<4>(const float*, int, int, int, int*, float*, float*, int*, float*);
template __global__ void moe_route<8>(const float*, int, int, int, int*, float*, float*, int*, float*);

// offsets / tile list / aux, one block of 256 threads (E <= kMoeMaxE).
// offsets[e] = sum_{e'<e} counts[e']; per group the 128-row GEMM tiles;
// aux = E * sum_e (counts_e / (T k)) (colsum_e / T)   (moe.hpp:90-103)
__global__ void __launch_bounds__(256) moe_plan(const int* __restrict__ counts, const float* __restrict__ prob_colsum,
                                                int nrb, int T, int E, int K, int* __restrict__ offsets,
                                                int* __restrict__ group_end, int* __restrict__ tile_group,
                                                int* __restrict__ tile_row0, int* __restrict__ num_tiles,
                                                float* __restrict__ aux) {
    __shared__ int s_off[kMoeMaxE + 1], s_toff[kMoeMaxE + 1];
    __shared__ double s_aux[kMoeMaxE];
    const int tid = threadIdx.x;
    if (tid == 0) {
        int off = 0, nt = 0;
        for (int e = 0; e < E; ++e) {
            s_off[e] = off;
            s_toff[e] = nt;
            off += counts[e];
            nt += (counts[e] + 127) / 128;
        }
        s_off[E] = off;
        s_toff[E] = nt;
    }
    if (tid < E) {
        const int c = counts[tid];
        double colsum = 0.0;  // the route blocks' partials, in block order
        if (prob_colsum)
            for (int bk = 0; bk < nrb; ++bk) colsum += prob_colsum[(size_t)bk * E + tid];
        s_aux[tid] = prob_colsum ? ((double)c / ((double)T * K)) * (colsum / T) : 0.0;
    }
    __syncthreads();
    for (int i = tid; i <= E; i += blockDim.x) offsets[i] = s_off[i];  // E + 1 entries (257 at E = 256)
    if (tid < E) group_end[tid] = s_off[tid + 1];
    const int nt = s_toff[E];
    for (int i = tid; i < nt; i += blockDim.x) {
        int lo = 0, hi = E - 1;  // last e with s_toff[e] <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_toff[mid] <= i) lo = mid; else hi = mid - 1;
        }
        tile_group[i] = lo;
        tile_row0[i] = s_off[lo] + (i - s_toff[lo]) * 128;
    }
    if (tid == 0) {
        *num_tiles = nt;
        double acc = 0.0;
        for (int e = 0; e < E; ++e) acc += s_aux[e];
        if (aux) *aux = (float)(acc * E);
    }
}

// Stable dispatch positions: block b owns tokens [b*256, b*256+256); blk_cnt[b][e] counted
// first, then each (token, slot) gets  offsets[e] + sum_{b'<b} blk_cnt[b'][e] + rank within
// the block among earlier tokens routed to e (token-ascending, moe.hpp:137-139).
__global__ void moe_block_counts(const int* __restrict__ ids, int T, int E, int K,
                                 int* __restrict__ blk_cnt) {
    __shared__ int c[kMoeMaxE];
    for (int i = threadIdx.x; i < kMoeMaxE; i += blockDim.x) c[i] = 0;
    __syncthreads();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < T)
        for (int s = 0; s < K; ++s) atomicAdd(&c[ids[(size_t)t * K + s]], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < E; i += blockDim.x) blk_cnt[(size_t)blockIdx.x * E + i] = c[i];
}

// blk_base[b][e] = offsets[e] + sum_{b'<b} blk_cnt[b'][e]: one block per expert, a
// block-wide exclusive scan over the token blocks (256 at a time with carry).
__global__ void __launch_bounds__(256) moe_block_scan(const int* __restrict__ blk_cnt, const int* __restrict__ offsets,
                                                      int nblk, int E, int* __restrict__ blk_base) {
    __shared__ int wsum[8];
    __shared__ int carry_s;
    const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) carry_s = offsets[e];
    __syncthreads();
    for (int b0 = 0; b0 < nblk; b0 += 256) {
        const int b = b0 + tid;
        const int v = b < nblk ? blk_cnt[(size_t)b * E + e] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        int before = 0;
        for (int i = 0; i < w; ++i) before += wsum[i];
        const int carry = carry_s;
        if (b < nblk) blk_base[(size_t)b * E + e] = carry + before + x - v;
        __syncthreads();
        if (tid == 255) carry_s = carry + before + x;
        __syncthreads();
    }
}

template <int KM>
__global__ void __launch_bounds__(256) moe_assign(const int* __restrict__ ids, int T, int E, int K,
                                                  const int* __restrict__ blk_base,
                                                  int* __restrict__ slot_pos,
                                                  int* __restrict__ perm_token) {
    __shared__ int warp_tot[8][kMoeMaxE];
    __shared__ int base[kMoeMaxE];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int t = blockIdx.x * 256 + tid;
    int my[KM];
#pragma unroll
    for (int s = 0; s < KM; ++s) my[s] = (s < K && t < T) ? ids[(size_t)t * K + s] : -1;
    for (int i = tid; i < E; i += 256) base[i] = blk_base[(size_t)blockIdx.x * E + i];
    // per expert: rank of this token among earlier tokens of the warp routed to e (a token
    // holds each expert at most once; its ids ascend, so slot search can stop early)
    int rank[KM];
#pragma unroll
    for (int s = 0; s < KM; ++s) rank[s] = 0;
    for (int e = 0; e < E; ++e) {
        bool hit = false;
        int hs = 0;
#pragma unroll
        for (int s = 0; s < KM; ++s)
            if (my[s] == e) { hit = true; hs = s; }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, hit);
        if (lane == 0) warp_tot[w][e] = __popc(m);
        if (hit) rank[hs] = __popc(m & ((1u << lane) - 1u));
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < KM; ++s) {
        if (my[s] < 0) continue;
        const int e = my[s];
        int before = 0;
        for (int ww = 0; ww < w; ++ww) before += warp_tot[ww][e];
        const int pos = base[e] + before + rank[s];
        slot_pos[(size_t)t * K + s] = pos;
        perm_token[pos] = t;
    }
}
template __global__ void moe_assign<8>(const int*, int, int, int, const int*, int*, int*);
template __global__ void moe_assign<32>(const int*, int, int, int, const int*, int*, int*);

// x_perm[slot_pos[t, s]] = x[t] for s < K: one warp per token reads its row once and writes
// it to its K dispatch rows.  (A gather in dispatch-row order read every token row K times in
// expert order and missed L2: 1.90 GB of DRAM per call at config 4 against 1.21 GB.)
__global__ void moe_scatter(const uint4* __restrict__ x, const int* __restrict__ slot_pos, int T, int K,
                            int row_vec, uint4* __restrict__ x_perm) {
    const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (t >= T) return;
    const int lane = threadIdx.x & 31;
    const int my_pos = lane < K ? slot_pos[(size_t)t * K + lane] : 0;  // K <= 32
    const uint4* src = x + (size_t)t * row_vec;
    for (int base = 0; base < row_vec; base += 128) {
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = base + j * 32 + lane;
            if (i < row_vec) v[j] = __ldg(src + i);
        }
        for (int s = 0; s < K; ++s) {
            uint4* dst = x_perm + (size_t)__shfl_sync(0xFFFFFFFFu, my_pos, s) * row_vec;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = base + j * 32 + lane;
                if (i < row_vec) dst[i] = v[j];
            }
        }
    }
}

// y[t] = sum_s gate[t,s] * y_perm[slot_pos[t,s]], slots in ascending expert order
// (moe.hpp:145-146 accumulates expert by expert).  One warp per token, 8 bf16 per lane-step;
// the row loads of up to 8 slots are in flight before their ordered accumulation.
template <int KM>
__global__ void moe_combine(const __nv_bfloat16* __restrict__ y_perm, const int* __restrict__ slot_pos,
                            const float* __restrict__ gates, int T, int K, int hidden,
                            void* __restrict__ y, int y_f32) {
    const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (t >= T) return;
    const int lane = threadIdx.x & 31;
    int pos[KM];
    float g[KM];
#pragma unroll
    for (int s = 0; s < KM; ++s) {
        pos[s] = s < K ? slot_pos[(size_t)t * K + s] : 0;
        g[s] = s < K ? gates[(size_t)t * K + s] : 0.f;
    }
    for (int c = lane * 8; c < hidden; c += 256) {
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
        for (int s0 = 0; s0 < KM; s0 += 8) {
            if (s0 >= K) break;
            uint4 vv[8];
#pragma unroll
            for (int s = 0; s < 8; ++s)
                vv[s] = s0 + s < K ? *reinterpret_cast<const uint4*>(y_perm + (size_t)pos[s0 + s] * hidden + c)
                                   : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                if (s0 + s >= K) break;
                const uint4 v = vv[s];
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f = unpack_bf16(w[i]);
                    acc[2 * i] += g[s0 + s] * f.x;
                    acc[2 * i + 1] += g[s0 + s] * f.y;
                }
            }
        }
        if (y_f32) {
            float* dst = reinterpret_cast<float*>(y) + (size_t)t * hidden + c;
            *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {
            uint4 o;
            o.x = pack_bf16(acc[0], acc[1]);
            o.y = pack_bf16(acc[2], acc[3]);
            o.z = pack_bf16(acc[4], acc[5]);
            o.w = pack_bf16(acc[6], acc[7]);
            *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(y) + (size_t)t * hidden + c) = o;
        }
    }
}
template __global__ void moe_combine<8>(const __nv_bfloat16*, const int*, const float*, int, int, int, void*, int);
template __global__ void moe_combine<32>(const __nv_bfloat16*, const int*, const float*, int, int, int, void*, int);

}  // namespace lmoe_dev
