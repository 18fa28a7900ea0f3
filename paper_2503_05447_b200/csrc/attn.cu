// attn.cu -- causal softmax attention with a row offset on sm_100a (tcgen05 + TMEM + TMA),
// and its sequence-parallel form with a K/V all-gather.
//
// Restates softmax_attention_parallel (/root/reference/proj/include/lmoe/attention.hpp:18-38):
//     O = softmax(Q K^T / sqrt(d), mask j <= i + row_offset) V
// and sp_attention_rank (parallel.hpp:380-387): all-gather K and V, local Q attends to the
// global sequence with its global row offset.
//
// One CTA per (128-row Q tile, h, b); tiles with more causal work are scheduled first.
//   warp 0       TMA: Q once, K/V tiles into a 2-stage ring
//   warp 1       MMA issuer: S_{j+1} = Q K_{j+1}^T (TMEM, 2 buffers) is issued before
//                O += P_j V_j, so the next scores overlap this tile's softmax; P_j is read
//                from TMEM (packed bf16 written over S_j)
//   warps 4..7   softmax, one query row per thread (TMEM lane = row), exp2 domain with a
//                lazily updated running max: O and l are rescaled only when the row max grows
//                by more than 2^8 (decided per warp), so exponents stay <= 2^8 and most tiles
//                need no O round trip
// TMEM: S0 [0,128) S1 [128,256) O [256,384).
#include <nccl.h>

#include <vector>

#include "common.h"
#include "internal.h"
#include "lsm_fwd.cuh"

namespace lmoe_dev {

constexpr int kAttnThreads = 256;
constexpr int kAttnKV = 3;  // K/V pipeline stages
constexpr float kRescaleLog2 = 8.f;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct AttnParams {
    int Nq, Nk, H;
    int row_offset;      // global row of local query 0
    float scale_log2;    // log2(e) / sqrt(d)
    __nv_bfloat16* o;    // [B, Nq, H, D]
};

__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, AttnParams p) {
    constexpr int D = 128, EPB = 64;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* qt = smem;                       // 32 KB
    // kAttnKV stages x [K | V] (64 KB each): the load of tile j + kAttnKV starts when PV_j
    // completes, so with three stages it has one more tile time to come from L2 than with two
    uint8_t* kv = smem + kTileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (1 + 2 * kAttnKV) * kTileBytes);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;             // [kAttnKV] K of the stage landed
    uint64_t* kv_empty = bars + 1 + kAttnKV;  // [kAttnKV]
    uint64_t* v_full = bars + 1 + 2 * kAttnKV;  // [kAttnKV] V of the stage landed (PV only)
    uint64_t* s_full = bars + 1 + 3 * kAttnKV;  // [2]
    uint64_t* p_full = s_full + 2;              // [2]
    uint64_t* o_done = p_full + 2;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(o_done + 1);

    const int ntq = (p.Nq + kC - 1) / kC;
    const int qtile = ntq - 1 - blockIdx.x;  // heavy (late) tiles first
    const int h = blockIdx.y, b = blockIdx.z;
    const int q0 = qtile * kC;
    const int last_row = p.row_offset + min(q0 + kC, p.Nq) - 1;  // global row of the last query
    const int nkv = min((last_row + kC) / kC, (p.Nk + kC - 1) / kC);
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < kAttnKV; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&v_full[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
        }
        mbar_init(o_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    const uint32_t tO = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
            mbar_expect_tx(q_full, kTileBytes);
            tma_load_4d(qt, &tmQ, q_full, 0, h, q0, b);
            tma_load_4d(qt + kBlockBytes, &tmQ, q_full, EPB, h, q0, b);
            for (int j = 0; j < nkv; ++j) {
                const int s = j % kAttnKV;
                if (j >= kAttnKV) mbar_wait(&kv_empty[s], ((j / kAttnKV) - 1) & 1);
                uint8_t* kt = kv + s * 2 * kTileBytes;
                uint8_t* vt = kt + kTileBytes;
                // K and V on separate barriers: S_j starts once K_j has landed
                mbar_expect_tx(&kv_full[s], kTileBytes);
                for (int blk = 0; blk < 2; ++blk)
                    tma_load_4d(kt + blk * kBlockBytes, &tmK, &kv_full[s], blk * EPB, h, j * kC, b);
                mbar_expect_tx(&v_full[s], kTileBytes);
                for (int blk = 0; blk < 2; ++blk)
                    tma_load_4d(vt + blk * kBlockBytes, &tmV, &v_full[s], blk * EPB, h, j * kC, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc(1, 0, 0, 128, 128);
            constexpr uint32_t idPV = umma_idesc(1, 0, 1, 128, D);
            const uint32_t qa = smem_u32(qt);
            auto issue_S = [&](int j) {
                const int s = j % kAttnKV, sb = j & 1;  // K/V stage, S buffer
                mbar_wait(&kv_full[s], (j / kAttnKV) & 1);
                tc_fence_after();
                const uint32_t kt = smem_u32(kv + s * 2 * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    mma_ss_f16(tmem + sb * 128, umma_desc_sw128(qa + off, 16, 1024),
                               umma_desc_sw128(kt + off, 16, 1024), idS, kk > 0);
                }
                mma_commit(&s_full[sb]);
            };
            mbar_wait(q_full, 0);
            issue_S(0);
            for (int j = 0; j < nkv; ++j) {
                const int s = j % kAttnKV, sb = j & 1;
                if (j + 1 < nkv) issue_S(j + 1);
                mbar_wait(&p_full[sb], (j >> 1) & 1);
                mbar_wait(&v_full[s], (j / kAttnKV) & 1);
                tc_fence_after();
                const uint32_t vt = smem_u32(kv + s * 2 * kTileBytes + kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts_f16(tO, tmem + sb * 128 + kk * 8,
                               umma_desc_sw128(vt + kk * 16 * 128, kBlockBytes, 1024), idPV, (j > 0 || kk > 0));
                mma_commit(&kv_empty[s]);
                mma_commit(o_done);
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        const int r = q * 32 + lane;             // query row of the tile == TMEM lane
        const int grow = p.row_offset + q0 + r;  // global query row
        const uint32_t lo = (uint32_t)(q * 32) << 16;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nkv; ++j) {
            const int s = j & 1;
            mbar_wait(&s_full[s], (j >> 1) & 1);
            tc_fence_after();
            // the row's 128 scores: all four TMEM loads in flight before one wait
            uint32_t u[128];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb)
                tmem_ld32(tmem + s * 128 + lo + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(u + cb * 32));
            tmem_wait_ld();
            // raw scores: the log2(e)/sqrt(d) scale is folded into the exponent's FFMA below (the
            // softmax warps are issue-bound; this drops one FMUL per score)
            float x[128];
#pragma unroll
            for (int i = 0; i < 128; ++i) x[i] = __uint_as_float(u[i]);
            const int k0 = j * kC;
            const bool full = k0 + kC - 1 <= p.row_offset + q0 && k0 + kC <= p.Nk;  // no masking
            if (!full) {
#pragma unroll
                for (int i = 0; i < 128; ++i)
                    if (k0 + i > grow || k0 + i >= p.Nk) x[i] = -INFINITY;
            }
            // row max over 8 independent accumulators (a single chain is 128 dependent FMNMX)
            float mx8[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) mx8[a] = x[a];
#pragma unroll
            for (int i = 8; i < 128; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], x[i]);
#pragma unroll
            for (int a = 4; a > 0; a >>= 1)
#pragma unroll
                for (int c = 0; c < a; ++c) mx8[c] = fmaxf(mx8[c], mx8[c + a]);
            const float mx = mx8[0] * p.scale_log2;  // scale > 0: the max commutes with it
            const float m_new = fmaxf(m, mx);
            const bool grow_max = m_new > m + kRescaleLog2;  // includes the first tile (m = -inf)
            if (__any_sync(0xFFFFFFFFu, grow_max && j > 0)) {
                // rescale O (and l) once PV_{j-1} has landed
                const float alpha = grow_max ? ex2(m - m_new) : 1.f;
                mbar_wait(o_done, (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int cb = 0; cb < 4; ++cb) {
                    uint32_t u[32];
                    tmem_ld32(tO + lo + cb * 32, u);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
                    tmem_st32(tO + lo + cb * 32, u);
                }
                l *= alpha;
            }
            if (grow_max) m = m_new;
            // P (bf16, packed in pairs) over the first 64 columns of S_j, 32 keys at a time
            float ls8[8];  // row sum over 8 independent accumulators
#pragma unroll
            for (int a = 0; a < 8; ++a) ls8[a] = 0.f;
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    // (a quarter of these on an FMA-pipe polynomial 2^x was measured: 1045 -> 915
                    // TFLOP/s; the softmax warps are issue-bound, one per scheduler, not MUFU-bound)
                    const float a = ex2(fmaf(x[cb * 32 + 2 * i], p.scale_log2, -m));
                    const float c2 = ex2(fmaf(x[cb * 32 + 2 * i + 1], p.scale_log2, -m));
                    ls8[(2 * i) & 7] += a;
                    ls8[(2 * i + 1) & 7] += c2;
                    pk[i] = pack_bf16(a, c2);
                }
                tmem_st16(tmem + s * 128 + lo + cb * 16, pk);
            }
#pragma unroll
            for (int a = 4; a > 0; a >>= 1)
#pragma unroll
                for (int c = 0; c < a; ++c) ls8[c] += ls8[c + a];
            l += ls8[0];
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[s]);
        }
        // epilogue: O / l -> global bf16
        mbar_wait(o_done, (nkv - 1) & 1);
        tc_fence_after();
        const float inv = 1.f / l;
        const bool vrow = q0 + r < p.Nq;
        __nv_bfloat16* dst = p.o + (((size_t)b * p.Nq + q0 + (vrow ? r : 0)) * p.H + h) * D;
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
            uint32_t u[32];
            tmem_ld32(tO + lo + cb * 32, u);
            tmem_wait_ld();
            if (vrow) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint4 w;
                    w.x = pack_bf16(__uint_as_float(u[c * 8 + 0]) * inv, __uint_as_float(u[c * 8 + 1]) * inv);
                    w.y = pack_bf16(__uint_as_float(u[c * 8 + 2]) * inv, __uint_as_float(u[c * 8 + 3]) * inv);
                    w.z = pack_bf16(__uint_as_float(u[c * 8 + 4]) * inv, __uint_as_float(u[c * 8 + 5]) * inv);
                    w.w = pack_bf16(__uint_as_float(u[c * 8 + 6]) * inv, __uint_as_float(u[c * 8 + 7]) * inv);
                    *reinterpret_cast<uint4*>(dst + cb * 32 + c * 8) = w;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------------------------
// Two query tiles per CTA (A = rows q0..q0+127, B = the next 128), softmax ping-pong: two
// softmax warpgroups, one per tile, so each scheduler runs two softmax warps, and the tensor
// core computes one tile's PV and next scores while the other tile's softmax runs.
//   warps 0 TMA, 1 MMA, 2-5 softmax tile A, 6-9 softmax tile B (TMEM lane quarter = warp % 4)
//   TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512); P packed into its S buffer
//   MMA order for key tile j: S_A(j), PV_B(j-1), S_B(j), PV_A(j)
// K/V tile j is released after PV_B(j) (the later tile reaches at least as far as A).
// ------------------------------------------------------------------------------------
constexpr int kPPThreads = 320;  // 204 registers per thread (384 threads would cap at 168 and spill)
constexpr int kPPKV = 2;

__global__ void __launch_bounds__(kPPThreads, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, AttnParams p) {
    constexpr int D = 128, EPB = 64;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* qt = smem;                   // [A | B], 32 KB each
    uint8_t* kv = smem + 2 * kTileBytes;  // kPPKV stages x [K | V]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (2 + 2 * kPPKV) * kTileBytes);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;             // [kPPKV]
    uint64_t* v_full = k_full + kPPKV;       // [kPPKV]
    uint64_t* kv_empty = v_full + kPPKV;     // [kPPKV]
    uint64_t* s_full = kv_empty + kPPKV;     // [2] per tile
    uint64_t* p_full = s_full + 2;           // [2]
    uint64_t* o_done = p_full + 2;           // [2]
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(o_done + 2);

    const int ntq = (p.Nq + kC - 1) / kC;
    const int npair = (ntq + 1) / 2;
    const int pair = npair - 1 - blockIdx.x;  // heavy (late) pairs first
    const int h = blockIdx.y, b = blockIdx.z;
    const bool hasB = 2 * pair + 1 < ntq;
    const int nkt = (p.Nk + kC - 1) / kC;
    auto nkv_of = [&](int t) {
        const int q0 = (2 * pair + t) * kC;
        const int last_row = p.row_offset + min(q0 + kC, p.Nq) - 1;
        return min((last_row + kC) / kC, nkt);
    };
    const int nkvA = nkv_of(0), nkvB = hasB ? nkv_of(1) : 0;
    const int nkv = max(nkvA, nkvB);
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < kPPKV; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 128);
            mbar_init(&o_done[t], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
            mbar_expect_tx(q_full, (hasB ? 2 : 1) * kTileBytes);
            for (int t = 0; t < (hasB ? 2 : 1); ++t)
                for (int blk = 0; blk < 2; ++blk)
                    tma_load_4d(qt + t * kTileBytes + blk * kBlockBytes, &tmQ, q_full, blk * EPB, h,
                                (2 * pair + t) * kC, b);
            for (int j = 0; j < nkv; ++j) {
                const int s = j % kPPKV;
                if (j >= kPPKV) mbar_wait(&kv_empty[s], ((j / kPPKV) - 1) & 1);
                uint8_t* kt = kv + s * 2 * kTileBytes;
                uint8_t* vt = kt + kTileBytes;
                mbar_expect_tx(&k_full[s], kTileBytes);
                for (int blk = 0; blk < 2; ++blk)
                    tma_load_4d(kt + blk * kBlockBytes, &tmK, &k_full[s], blk * EPB, h, j * kC, b);
                mbar_expect_tx(&v_full[s], kTileBytes);
                for (int blk = 0; blk < 2; ++blk)
                    tma_load_4d(vt + blk * kBlockBytes, &tmV, &v_full[s], blk * EPB, h, j * kC, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc(1, 0, 0, 128, 128);
            constexpr uint32_t idPV = umma_idesc(1, 0, 1, 128, D);
            auto issue_S = [&](int t, int j) {
                const uint32_t qa = smem_u32(qt + t * kTileBytes);
                const uint32_t kt = smem_u32(kv + (j % kPPKV) * 2 * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    mma_ss_f16(tmem + t * 128, umma_desc_sw128(qa + off, 16, 1024),
                               umma_desc_sw128(kt + off, 16, 1024), idS, kk > 0);
                }
                mma_commit(&s_full[t]);
            };
            auto issue_PV = [&](int t, int j) {
                mbar_wait(&p_full[t], j & 1);
                mbar_wait(&v_full[j % kPPKV], (j / kPPKV) & 1);
                tc_fence_after();
                const uint32_t vt = smem_u32(kv + (j % kPPKV) * 2 * kTileBytes + kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts_f16(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                               umma_desc_sw128(vt + kk * 16 * 128, kBlockBytes, 1024), idPV, (j > 0 || kk > 0));
                mma_commit(&o_done[t]);
            };
            mbar_wait(q_full, 0);
            for (int j = 0; j < nkv; ++j) {
                mbar_wait(&k_full[j % kPPKV], (j / kPPKV) & 1);
                tc_fence_after();
                if (j < nkvA) issue_S(0, j);
                if (j >= 1 && j - 1 < nkvB) {
                    issue_PV(1, j - 1);
                    mma_commit(&kv_empty[(j - 1) % kPPKV]);
                }
                if (j < nkvB) issue_S(1, j);
                if (j < nkvA) {
                    issue_PV(0, j);
                    if (j >= nkvB) mma_commit(&kv_empty[j % kPPKV]);  // B does not use this tile
                }
            }
            if (nkvB >= 1) {
                issue_PV(1, nkvB - 1);
                mma_commit(&kv_empty[(nkvB - 1) % kPPKV]);
            }
        }
    } else if (warp >= 2) {
        const int t = (warp - 2) >> 2;  // tile of this softmax warpgroup
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const int q0 = (2 * pair + t) * kC;
        const int nkv_t = t ? nkvB : nkvA;
        const int grow = p.row_offset + q0 + r;
        const uint32_t lo = (uint32_t)(q * 32) << 16;
        const uint32_t tS = tmem + t * 128, tO = tmem + 256 + t * 128;
        if (t == 0 || hasB) {
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < nkv_t; ++j) {
                mbar_wait(&s_full[t], j & 1);
                tc_fence_after();
                // two passes over the row's 128 scores in TMEM, 64 at a time (the whole row in
                // registers would exceed the 168 registers of 3 warps per scheduler): row max,
                // then exponentials and the packed P.  Raw scores; the scale is folded into the
                // exponent's FFMA.
                const int k0 = j * kC;
                const bool full = k0 + kC - 1 <= p.row_offset + q0 && k0 + kC <= p.Nk;
                auto load_half = [&](int hf, uint32_t (&u)[64]) {
                    tmem_ld32(tS + lo + hf * 64, *reinterpret_cast<uint32_t(*)[32]>(u));
                    tmem_ld32(tS + lo + hf * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
                    tmem_wait_ld();
                    if (!full) {
#pragma unroll
                        for (int i = 0; i < 64; ++i) {
                            const int key = k0 + hf * 64 + i;
                            if (key > grow || key >= p.Nk) u[i] = __float_as_uint(-INFINITY);
                        }
                    }
                };
                float mx8[8];
#pragma unroll
                for (int a = 0; a < 8; ++a) mx8[a] = -INFINITY;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t u[64];
                    load_half(hf, u);
#pragma unroll
                    for (int i = 0; i < 64; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(u[i]));
                }
#pragma unroll
                for (int a = 4; a > 0; a >>= 1)
#pragma unroll
                    for (int c = 0; c < a; ++c) mx8[c] = fmaxf(mx8[c], mx8[c + a]);
                const float m_new = fmaxf(m, mx8[0] * p.scale_log2);
                const bool grow_max = m_new > m + kRescaleLog2;
                if (__any_sync(0xFFFFFFFFu, grow_max && j > 0)) {
                    const float alpha = grow_max ? ex2(m - m_new) : 1.f;
                    mbar_wait(&o_done[t], (j - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int cb = 0; cb < 4; ++cb) {
                        uint32_t w[32];
                        tmem_ld32(tO + lo + cb * 32, w);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
                        tmem_st32(tO + lo + cb * 32, w);
                    }
                    l *= alpha;
                }
                if (grow_max) m = m_new;
                float ls8[8];
#pragma unroll
                for (int a = 0; a < 8; ++a) ls8[a] = 0.f;
                uint32_t pk[2][32];
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t u[64];
                    load_half(hf, u);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float a = ex2(fmaf(__uint_as_float(u[2 * i]), p.scale_log2, -m));
                        const float c2 = ex2(fmaf(__uint_as_float(u[2 * i + 1]), p.scale_log2, -m));
                        ls8[(2 * i) & 7] += a;
                        ls8[(2 * i + 1) & 7] += c2;
                        pk[hf][i] = pack_bf16(a, c2);
                    }
                }
                // P overwrites the scores only after both passes read them
                tmem_st32(tS + lo, pk[0]);
                tmem_st32(tS + lo + 32, pk[1]);
#pragma unroll
                for (int a = 4; a > 0; a >>= 1)
#pragma unroll
                    for (int c = 0; c < a; ++c) ls8[c] += ls8[c + a];
                l += ls8[0];
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&p_full[t]);
            }
            // epilogue: O / l -> global bf16
            mbar_wait(&o_done[t], (nkv_t - 1) & 1);
            tc_fence_after();
            const float inv = 1.f / l;
            const bool vrow = q0 + r < p.Nq;
            __nv_bfloat16* dst = p.o + (((size_t)b * p.Nq + q0 + (vrow ? r : 0)) * p.H + h) * D;
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                uint32_t w[32];
                tmem_ld32(tO + lo + cb * 32, w);
                tmem_wait_ld();
                if (vrow) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint4 o4;
                        o4.x = pack_bf16(__uint_as_float(w[c * 8 + 0]) * inv, __uint_as_float(w[c * 8 + 1]) * inv);
                        o4.y = pack_bf16(__uint_as_float(w[c * 8 + 2]) * inv, __uint_as_float(w[c * 8 + 3]) * inv);
                        o4.z = pack_bf16(__uint_as_float(w[c * 8 + 4]) * inv, __uint_as_float(w[c * 8 + 5]) * inv);
                        o4.w = pack_bf16(__uint_as_float(w[c * 8 + 6]) * inv, __uint_as_float(w[c * 8 + 7]) * inv);
                        *reinterpret_cast<uint4*>(dst + cb * 32 + c * 8) = o4;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// Gathered padded slices [T][B][maxlen][H][D] -> contiguous [B][N][H][D] (chunk_range order).
__global__ void attn_compact_kv(const uint4* __restrict__ src, uint4* __restrict__ dst, int T, int B, int N,
                                int maxlen, int rowvec) {
    const size_t total = (size_t)B * N * rowvec;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t row = i / rowvec;
        const int e = (int)(i % rowvec);
        const int b = (int)(row / N), n = (int)(row % N);
        const int base = N / T, rem = N % T;
        // rank of global row n under chunk_range (parallel.hpp:192-197)
        const int big = rem * (base + 1);
        const int r = n < big ? n / (base + 1) : rem + (n - big) / base;
        const int r0 = r * base + min(r, rem);
        dst[i] = src[(((size_t)r * B + b) * maxlen + (n - r0)) * rowvec + e];
    }
}

}  // namespace lmoe_dev

namespace lmoe_host {
using namespace lmoe_dev;

static void attn_validate(int B, int Nq, int Nk, int H, int D, lmoe_dtype dt, const void* q, const void* k,
                          const void* v, const void* o) {
    if (Nq < 1) throw Error(LMOE_ERR_ARG, "softmax_attention_parallel: need N >= 1 rows");
    if (B < 1 || H < 1 || Nk < 1) throw Error(LMOE_ERR_ARG, "softmax_attention_parallel: bad shape");
    if (dt != LMOE_BF16 || D != 128)
        throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_attn_fwd: supported (dtype, head_dim) is (bf16, 128)");
    if (!q || !k || !v || !o) throw Error(LMOE_ERR_ARG, "lmoe_attn_fwd: null tensor");
}

// ldq / ldkv: elements per token row of q and of k, v (0: H * D)
static void attn_launch(int B, int Nq, int Nk, int H, int D, int row_offset, const void* q, const void* k,
                        const void* v, void* o, cudaStream_t st, int ldq = 0, int ldkv = 0) {
    const CUtensorMap tq = make_tmap_4d(q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, H, Nq, B, 64, kC, 0, ldq);
    const CUtensorMap tk = make_tmap_4d(k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, H, Nk, B, 64, kC, 0, ldkv);
    const CUtensorMap tv = make_tmap_4d(v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, H, Nk, B, 64, kC, 0, ldkv);
    AttnParams p{Nq, Nk, H, row_offset, 1.4426950408889634f / sqrtf((float)D), static_cast<__nv_bfloat16*>(o)};
    // one query tile per CTA with three K/V stages; LMOE_ATTN_PP=1 (developer A/B) runs the
    // two-tile softmax ping-pong, measured 0-10% slower at the cfg5 rank shapes (its two Q tiles
    // leave room for only two K/V stages, and the three stages are what made the difference)
    static const bool pp = getenv("LMOE_ATTN_PP") != nullptr && atoi(getenv("LMOE_ATTN_PP")) != 0;
    if (pp) {
        constexpr int smem = (2 + 2 * kPPKV) * kTileBytes + 256;
        LMOE_CUDA_CHECK(lmoe_dev::ensure_smem((const void*)attn_fwd_pp_kernel, smem));
        const int ntq = (Nq + kC - 1) / kC;
        attn_fwd_pp_kernel<<<dim3((ntq + 1) / 2, H, B), kPPThreads, smem, st>>>(tq, tk, tv, p);
    } else {
        constexpr int smem = (1 + 2 * kAttnKV) * kTileBytes + 256;
        LMOE_CUDA_CHECK(lmoe_dev::ensure_smem((const void*)attn_fwd_kernel, smem));
        attn_fwd_kernel<<<dim3((Nq + kC - 1) / kC, H, B), kAttnThreads, smem, st>>>(tq, tk, tv, p);
    }
    LMOE_CUDA_CHECK(cudaGetLastError());
    ++g_launch_count;
}

static thread_local long long g_attn_gather_elements = 0;

void attn_core(int B, int Nq, int Nk, int H, int D, const void* q, const void* k, const void* v, int ld,
               void* o, int row_offset, cudaStream_t st) {
    attn_validate(B, Nq, Nk, H, D, LMOE_BF16, q, k, v, o);
    attn_launch(B, Nq, Nk, H, D, row_offset, q, k, v, o, st, ld, ld);
}

size_t sp_attn_ws(int B, int N_total, int H, int D, int world) {
    if (B < 1 || N_total < world || world < 1) return 0;
    const size_t maxlen = (N_total + world - 1) / world;
    const size_t row = (size_t)H * D * 2;
    // gathered K, V (padded) + compact K, V
    return 2 * align_up((size_t)world * B * maxlen * row, 256) + 2 * align_up((size_t)B * N_total * row, 256);
}

// sp_attention_rank (parallel.hpp:380-387) over strided local rows (ld elements; 0: H * D).
void sp_attn_core(int B, int N_total, int H, int D, const void* q_loc, const void* k_loc, const void* v_loc,
                  int ld, void* o_loc, void* nccl_comm, int rank, int world, void* workspace,
                  size_t workspace_bytes, cudaStream_t st) {
    if (world < 1 || rank < 0 || rank >= world) throw Error(LMOE_ERR_ARG, "lmoe_sp_attn_fwd: bad rank");
    if (N_total < world) throw Error(LMOE_ERR_ARG, "chunk_range: need at least one row per rank");
    const int base = N_total / world, rem = N_total % world;
    const int r0 = rank * base + std::min(rank, rem);
    const int len = base + (rank < rem ? 1 : 0);
    attn_validate(B, len, N_total, H, D, LMOE_BF16, q_loc, k_loc, v_loc, o_loc);
    if (world > 1 && !nccl_comm) throw Error(LMOE_ERR_ARG, "lmoe_sp_attn_fwd: null communicator");
    const size_t need = sp_attn_ws(B, N_total, H, D, world);
    if (!workspace || workspace_bytes < need)
        throw Error(LMOE_ERR_ARG, "lmoe_sp_attn_fwd: workspace too small (need " + std::to_string(need) + " bytes)");
    const int maxlen = (N_total + world - 1) / world;
    const size_t row = (size_t)H * D * 2;
    const size_t src_pitch = (ld ? (size_t)ld : (size_t)H * D) * 2;
    const size_t gbytes = align_up((size_t)world * B * maxlen * row, 256);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    uint8_t* gk = ws;
    uint8_t* gv = ws + gbytes;
    uint8_t* ck = ws + 2 * gbytes;
    uint8_t* cv = ck + align_up((size_t)B * N_total * row, 256);
    const size_t send = (size_t)B * maxlen * row;  // bytes per rank (padded)
    // this rank's slice at the front of a maxlen-row slot per batch row (strided -> dense rows)
    const bool direct = B == 1 && rem == 0;  // gathered layout == global layout
    uint8_t* dk = direct ? ck : gk;
    uint8_t* dv = direct ? cv : gv;
    for (int b = 0; b < B; ++b) {
        LMOE_CUDA_CHECK(cudaMemcpy2DAsync(dk + ((size_t)rank * B + b) * maxlen * row, row,
                                          static_cast<const uint8_t*>(k_loc) + (size_t)b * len * src_pitch,
                                          src_pitch, row, len, cudaMemcpyDeviceToDevice, st));
        LMOE_CUDA_CHECK(cudaMemcpy2DAsync(dv + ((size_t)rank * B + b) * maxlen * row, row,
                                          static_cast<const uint8_t*>(v_loc) + (size_t)b * len * src_pitch,
                                          src_pitch, row, len, cudaMemcpyDeviceToDevice, st));
    }
    if (nccl_comm) {  // world 1 with a 1-rank communicator runs the gather too
        ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
        ncclResult_t r = ncclGroupStart();
        if (r == ncclSuccess) r = ncclAllGather(dk + rank * send, dk, send, ncclUint8, comm, st);
        if (r == ncclSuccess) r = ncclAllGather(dv + rank * send, dv, send, ncclUint8, comm, st);
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            throw Error(LMOE_ERR_NCCL, std::string("NCCL error: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
    }
    g_attn_gather_elements = 2LL * world * (long long)B * maxlen * H * D;
    if (!direct) {
        const int rowvec = (int)(row / 16);
        const size_t total = (size_t)B * N_total * rowvec;
        const int grid = (int)std::min<size_t>((total + 255) / 256, 148 * 8);
        attn_compact_kv<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(gk), reinterpret_cast<uint4*>(ck),
                                              world, B, N_total, maxlen, rowvec);
        attn_compact_kv<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(gv), reinterpret_cast<uint4*>(cv),
                                              world, B, N_total, maxlen, rowvec);
        LMOE_CUDA_CHECK(cudaGetLastError());
        g_launch_count += 2;
    }
    attn_launch(B, len, N_total, H, D, r0, q_loc, ck, cv, o_loc, st, ld, 0);
}

}  // namespace lmoe_host

using namespace lmoe_host;

// softmax_attention_parallel(q, k, v, causal=true, row_offset) (attention.hpp:18-38):
// q [B, Nq, H, D], k / v [B, Nk, H, D] bf16, o [B, Nq, H, D] bf16.
extern "C" int lmoe_attn_fwd(int B, int Nq, int Nk, int H, int D, lmoe_dtype dtype, const void* q,
                             const void* k, const void* v, void* o, int row_offset, lmoe_stream_t stream) {
    return guarded([&]() {
        attn_validate(B, Nq, Nk, H, D, dtype, q, k, v, o);
        if (row_offset < 0) throw Error(LMOE_ERR_ARG, "lmoe_attn_fwd: negative row_offset");
        attn_launch(B, Nq, Nk, H, D, row_offset, q, k, v, o, reinterpret_cast<cudaStream_t>(stream));
    });
}

extern "C" size_t lmoe_sp_attn_workspace_size(int B, int N_total, int H, int D, lmoe_dtype dtype, int world) {
    (void)dtype;
    return sp_attn_ws(B, N_total, H, D, world);
}

extern "C" long long lmoe_sp_attn_last_gather_elements(void) { return g_attn_gather_elements; }

// sp_attention_rank (parallel.hpp:380-387): this rank's contiguous slice (chunk_range of
// N_total) of q, k, v [B, N_local, H, D]; K and V are all-gathered (one NCCL group of two
// all-gathers, the reference's two collectives) into the global sequence and the local
// queries attend with row_offset = r0.
extern "C" int lmoe_sp_attn_fwd(int B, int N_total, int H, int D, lmoe_dtype dtype, const void* q_loc,
                                const void* k_loc, const void* v_loc, void* o_loc, void* nccl_comm, int rank,
                                int world, void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        if (dtype != LMOE_BF16 || D != 128)
            throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_attn_fwd: supported (dtype, head_dim) is (bf16, 128)");
        sp_attn_core(B, N_total, H, D, q_loc, k_loc, v_loc, 0, o_loc, nccl_comm, rank, world, workspace,
                     workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
    });
}
