// lsm_dgate.cu -- Mamba2 (TokenScalar) decay-gate gradients of the LSM backward.
//
// The gradient of the per-token log decay g_j (G = inclusive cumsum of g) is the sum over
// all (query t, key s) pairs that straddle j:
//     dg_j = sum_{s < j <= t} A_ts,   A_ts = (phi(q_t).keff_s) (dO_t.v_s) e^{G_t - G_s}
// (with the initial / final states as extra keys / queries).  The telescoped form
// sum_{t >= j} (phi(q_t).dphi(q_t) - keff_t.dkeff_t) cancels nearly equal totals, which
// bf16 operand rounding cannot survive.  Here every term is a product of fp32 tensor-core
// accumulators, evaluated per 128-token chunk c (persistent CTAs, chunks independent):
//     dg_j = C(j) + sum_{t in [j, end]} X_t + sum_{s in [start, j)} Y_s + e^{g_c} <M_c, dM_c>
//   C(j)  within-chunk straddle: C(j) = sum_{i < j} (colsum_i - rowsum_i) of strictly
//         lower A (S = phiQ phiK^T and dP = dO V^T on tcgen05, A in fp32 registers)
//   X_t   = e^{G_t} phi(q_t) M_c dO_t^T       (Z = phiQ M_c on tcgen05)
//   Y_s   = e^{g_c - G_s} keff_s dM_c v_s^T   (W = phiK dM_c on tcgen05)
//   M_c   = state before chunk c (dq pass side output, M^T rows), dM_c = state gradient after
//           chunk c (dk pass side output, dM^T rows): both [BH][nchunk][D][D] in T.
// Then db_j = sigma(b_j) (dkf_j - softplus(a) dg_j) and da_raw += sigma(a) dg_j (-softplus(b_j))
// (decay_vector_rows / effective_keys chain, lsm.hpp:483-518; oracle lmo_lsm_backward).
#include "lsm_fwd.cuh"
#include "lsm_launch.h"

namespace lmoe_dev {

namespace {

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + __expf(-x)); }

// 32 consecutive elements [col0, col0 + 32) of `row` from an SW128 tile of two column
// blocks (block stride blk_bytes).
template <typename T>
__device__ __forceinline__ void tile_row32(const uint8_t* tile, int blk_bytes, int row, int col0,
                                           float (&out)[32]) {
    using TT = TileTraits<T>;
    const uint8_t* blk = tile + (col0 / TT::EPB) * blk_bytes;
    const int ch0 = (col0 % TT::EPB) / TT::EPC;
#pragma unroll
    for (int c = 0; c < 32 / TT::EPC; ++c) {
        const uint4 v = *reinterpret_cast<const uint4*>(blk + sw128_off(row, ch0 + c));
        if constexpr (sizeof(T) == 2) {
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = unpack_bf16(w[i]);
                out[c * 8 + 2 * i] = f.x;
                out[c * 8 + 2 * i + 1] = f.y;
            }
        } else {
            out[c * 4] = __uint_as_float(v.x); out[c * 4 + 1] = __uint_as_float(v.y);
            out[c * 4 + 2] = __uint_as_float(v.z); out[c * 4 + 3] = __uint_as_float(v.w);
        }
    }
}

// 128-thread inclusive prefix sum (4 warps); `ws` holds 4 floats of shared scratch.
__device__ __forceinline__ float block_incl_scan128(float x, float* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    for (int i = 0; i < warp; ++i) x += ws[i];
    return x;
}
__device__ __forceinline__ float block_sum128(float x, float* ws) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    return ws[0] + ws[1] + ws[2] + ws[3];
}

template <typename T>
struct DgateSmem {
    static constexpr int D = TileTraits<T>::D;
    static constexpr int kMT = D * D * (int)sizeof(T);  // state tile bytes
    static constexpr int kQ = 0, kK = kTileBytes, kV = 2 * kTileBytes, kO = 3 * kTileBytes;
    static constexpr int kM = 4 * kTileBytes, kDM = kM + kMT;
    static constexpr int kMisc = kDM + kMT;  // sG, sKf, 5 x [2][128] partials, scratch, barriers
    static constexpr int kTotal = kMisc + (2 + 5 * 4) * 128 * 4 + 64 * 4 + 64;
};

}  // namespace

// kDgNH x 128 threads: warp w owns TMEM lane quadrant w % 4 (query rows) and column part
// w / 4 of every row-wise phase; the 128-entry scans run on warps 0-3 (named barrier 1).
constexpr int kDgNH = 4;
constexpr int kDgThreads = 128 * kDgNH;
// MMA-issuing thread.  Issuing the next chunk's MMAs from warp 4 during this chunk's final
// scans was measured slower (2.34 vs 2.24 ms at config 3) than issuing at the chunk start.
constexpr int kDgMma = 0;

// 128-thread inclusive prefix sum over warps 0-3 (named barrier 1); `ws` holds 4 floats
__device__ __forceinline__ float scan128_w03(float x, float* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    named_bar_sync(1, 128);
    if (lane == 31) ws[warp] = x;
    named_bar_sync(1, 128);
    for (int i = 0; i < warp; ++i) x += ws[i];
    return x;
}
// three inclusive prefix sums at once over warps 0-3 (named barrier 1); `ws` holds 12 floats;
// tb receives the total of b
__device__ __forceinline__ void scan3_w03(float& a, float& b, float& c, float& tb, float* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float ya = __shfl_up_sync(0xFFFFFFFFu, a, o);
        const float yb = __shfl_up_sync(0xFFFFFFFFu, b, o);
        const float yc = __shfl_up_sync(0xFFFFFFFFu, c, o);
        if (lane >= o) { a += ya; b += yb; c += yc; }
    }
    if (lane == 31) { ws[warp] = a; ws[4 + warp] = b; ws[8 + warp] = c; }
    named_bar_sync(1, 128);
    float pa = 0.f, pb = 0.f, pc = 0.f;
    for (int i = 0; i < warp; ++i) { pa += ws[i]; pb += ws[4 + i]; pc += ws[8 + i]; }
    tb = ws[4] + ws[5] + ws[6] + ws[7];
    named_bar_sync(1, 128);  // ws reusable
    a += pa; b += pb; c += pc;
}
__device__ __forceinline__ float sum128_w03(float x, float* ws) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    named_bar_sync(1, 128);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = x;
    named_bar_sync(1, 128);
    return ws[0] + ws[1] + ws[2] + ws[3];
}

// Column sums of a warp's 32 x 32 block (row = lane, column = register): a butterfly
// transpose-reduce, 31 shuffles; returns the sum of column `lane`.
__device__ __forceinline__ float warp_colsum32(float (&a)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const bool up = (lane & w) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const float send = up ? a[i] : a[i + w];
            const float keep = up ? a[i + w] : a[i];
            a[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, w);
        }
    }
    return a[0];
}

// Persistent: CTA i takes chunks lin = i, i + grid, ... (lin = c + nchunk * bh).  One set of
// tiles per CTA; every tile is consumed (MMAs committed, row reads of K / O / V and the M, dM
// dot done) before the A-matrix phase, so the next chunk's loads are issued at that point and
// land while this chunk's straddle sums, scans and gate outputs run.
template <typename T>
__global__ void __launch_bounds__(kDgThreads, 1)
    lsm_mamba_dgate(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmDM,
                    const float* __restrict__ b_pre, const float* __restrict__ a_raw,
                    const float* __restrict__ dkf, const T* __restrict__ dk, float* __restrict__ db_pre,
                    float* __restrict__ da_raw, int N, int H, int nchunk, int total, int p_pf_ahead) {
    using TT = TileTraits<T>;
    using L = DgateSmem<T>;
    constexpr int D = TT::D;
    constexpr int MBLK = D * 128;  // column-block stride of a state tile
    extern __shared__ __align__(1024) uint8_t smem[];
    float* sG = reinterpret_cast<float*>(smem + L::kMisc);
    float* sKf = sG + 128;
    constexpr int NH = kDgNH;
    float* sX = sKf + 128;   // [NH][128] partials: X, Y, row sums (per column part), column sums
    float* sY = sX + NH * 128;  // (per row quadrant), dkf
    float* sR = sY + NH * 128;
    float* sC = sR + NH * 128;
    float* sF = sC + NH * 128;
    float* ws = sF + NH * 128;  // 64 floats scratch: [0, 4) scans, [8, 24) <M, dM> parts, [32, 44) scan3
    uint64_t* bar = reinterpret_cast<uint64_t*>(ws + 64);
    uint64_t* mma_done = bar + 1;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bar + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t = (warp & 3) * 32 + lane;  // TMEM lane == query row t
    const int hc = warp >> 2;              // column part of the row-wise phases
    constexpr int PW = D / NH;             // state columns per thread (bf16 32, tf32 16)
    constexpr int SW = 128 / NH;           // S / dP columns per thread
    static_assert(SW == 32, "one 32-column block of S / dP per thread");

    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(mma_done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;

    // all six tiles of chunk `lin` on `bar` (thread 0), and an L2 prefetch p_pf_ahead chunks on
    auto issue = [&](int lin) {
        const int c = lin % nchunk, bh = lin / nchunk, b = bh / H, h = bh % H, t0 = c * kC;
        const int mrow = (bh * nchunk + c) * D;
        mbar_expect_tx(bar, 4 * kTileBytes + 2 * L::kMT);
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
            tma_load_4d(smem + L::kQ + blk * kBlockBytes, &tmQ, bar, blk * TT::EPB, h, t0, b);
            tma_load_4d(smem + L::kK + blk * kBlockBytes, &tmK, bar, blk * TT::EPB, h, t0, b);
            tma_load_4d(smem + L::kV + blk * kBlockBytes, &tmV, bar, blk * TT::EPB, h, t0, b);
            tma_load_4d(smem + L::kO + blk * kBlockBytes, &tmO, bar, blk * TT::EPB, h, t0, b);
            tma_load_2d(smem + L::kM + blk * MBLK, &tmM, bar, blk * TT::EPB, mrow);
            tma_load_2d(smem + L::kDM + blk * MBLK, &tmDM, bar, blk * TT::EPB, mrow);
        }
        const long long l2 = (long long)lin + p_pf_ahead;
        if (p_pf_ahead > 0 && l2 < total) {
            const int c2 = (int)(l2 % nchunk), bh2 = (int)(l2 / nchunk);
            const int b2 = bh2 / H, h2 = bh2 % H, t2 = c2 * kC, mrow2 = (bh2 * nchunk + c2) * D;
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                tma_prefetch_l2_4d(&tmQ, blk * TT::EPB, h2, t2, b2);
                tma_prefetch_l2_4d(&tmK, blk * TT::EPB, h2, t2, b2);
                tma_prefetch_l2_4d(&tmV, blk * TT::EPB, h2, t2, b2);
                tma_prefetch_l2_4d(&tmO, blk * TT::EPB, h2, t2, b2);
                tma_prefetch_l2_2d(&tmM, blk * TT::EPB, mrow2);
                tma_prefetch_l2_2d(&tmDM, blk * TT::EPB, mrow2);
            }
        }
    };
    if (tid == 0 && (int)blockIdx.x < total) issue(blockIdx.x);

    // S = phiQ phiK^T (cols 0..127), dP = dO V^T (128..255), Z = phiQ M_c (256..),
    // W = phiK dM_c (384..): all operands K-major.  Issued by thread kDgMma once the chunk's
    // tiles have landed (phase `phase` of `bar`); the previous chunk's TMEM reads are done.
    auto issue_mma = [&](uint32_t phase) {
        mbar_wait(bar, phase);
        tc_fence_after();
        constexpr uint32_t idSq = umma_idesc(TT::FMT, 0, 0, 128, 128);
        constexpr uint32_t idSt = umma_idesc(TT::FMT, 0, 0, 128, D);
        const uint32_t q = smem_u32(smem + L::kQ), k = smem_u32(smem + L::kK);
        const uint32_t v = smem_u32(smem + L::kV), o = smem_u32(smem + L::kO);
        const uint32_t m = smem_u32(smem + L::kM), dm = smem_u32(smem + L::kDM);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
            const uint32_t moff = (kk >> 2) * MBLK + (kk & 3) * 32;
            const uint32_t acc = kk > 0;
            if constexpr (sizeof(T) == 2) {
                mma_ss_f16(tmem, umma_desc_sw128(q + off, 16, 1024), umma_desc_sw128(k + off, 16, 1024), idSq, acc);
                mma_ss_f16(tmem + 128, umma_desc_sw128(o + off, 16, 1024), umma_desc_sw128(v + off, 16, 1024), idSq, acc);
                mma_ss_f16(tmem + 256, umma_desc_sw128(q + off, 16, 1024), umma_desc_sw128(m + moff, 16, 1024), idSt, acc);
                mma_ss_f16(tmem + 384, umma_desc_sw128(k + off, 16, 1024), umma_desc_sw128(dm + moff, 16, 1024), idSt, acc);
            } else {
                mma_ss_tf32(tmem, umma_desc_sw128(q + off, 16, 1024), umma_desc_sw128(k + off, 16, 1024), idSq, acc);
                mma_ss_tf32(tmem + 128, umma_desc_sw128(o + off, 16, 1024), umma_desc_sw128(v + off, 16, 1024), idSq, acc);
                mma_ss_tf32(tmem + 256, umma_desc_sw128(q + off, 16, 1024), umma_desc_sw128(m + moff, 16, 1024), idSt, acc);
                mma_ss_tf32(tmem + 384, umma_desc_sw128(k + off, 16, 1024), umma_desc_sw128(dm + moff, 16, 1024), idSt, acc);
            }
        }
        mma_commit(mma_done);
    };
    auto load_b = [&](int lin) -> float {
        if (lin >= total) return 0.f;
        const int c = lin % nchunk, bh = lin / nchunk, t0 = c * kC;
        return t < min(kC, N - t0) ? b_pre[((size_t)(bh / H) * N + t0 + t) * H + bh % H] : 0.f;
    };
    float bv_next = load_b(blockIdx.x);
    uint32_t ph = 0;
    for (int lin = blockIdx.x; lin < total; lin += gridDim.x, ph ^= 1u) {
        const int c = lin % nchunk, bh = lin / nchunk;
        const int b = bh / H, h = bh % H;
        const int t0 = c * kC;
        const int nvalid = min(kC, N - t0);
        // gates: g_t = -softplus(b_t) softplus(a_h), kf_t = softplus(b_t); b_t was loaded one
        // chunk ahead, the next chunk's is requested now
        const float spa = softplus_f(a_raw[h]);
        const float bv = t < nvalid ? bv_next : 0.f;
        const float kf = t < nvalid ? softplus_f(bv) : 0.f;
        bv_next = load_b(lin + gridDim.x);
        // dkf_t = phi(k_t) . dkeff_t: given, or from dk = kf dkeff (identity feature map); the
        // global dk row is read before the tiles are needed (latency overlaps the TMA loads)
        // raw words: unpacked where they are used, so the load latency stays hidden
        constexpr int NRAW = sizeof(T) == 2 ? PW / 8 : PW / 4;
        uint4 dkraw[NRAW];
        const bool dk_direct = dkf == nullptr;
        if (dk_direct && t < nvalid) {
            const uint4* dkr = reinterpret_cast<const uint4*>(dk + (((size_t)b * N + t0 + t) * H + h) * D + hc * PW);
#pragma unroll
            for (int j = 0; j < NRAW; ++j) dkraw[j] = __ldg(dkr + j);
        }
        if (tid == kDgMma) issue_mma(ph);  // first: the MMAs do not need the gates
        if (warp < 4) {
            const float G = scan128_w03(t < nvalid ? -kf * spa : 0.f, ws);
            sG[t] = G;
            sKf[t] = kf;
        }
        __syncthreads();  // sG / sKf visible
        const float gend = sG[127];
        // B_c partial: <M_c, dM_c> over this thread's 16-byte slices of the (identically laid out) tiles
        float bpart = 0.f;
        {
            const uint8_t* pm = smem + L::kM + tid * 16;
            const uint8_t* pd = smem + L::kDM + tid * 16;
            mbar_wait(bar, ph);
#pragma unroll 4
            for (int i = 0; i < L::kMT; i += kDgThreads * 16) {
                const uint4 a = *reinterpret_cast<const uint4*>(pm + i);
                const uint4 d = *reinterpret_cast<const uint4*>(pd + i);
                const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, dw[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if constexpr (sizeof(T) == 2) {
                        const float2 fa = unpack_bf16(aw[e]), fd = unpack_bf16(dw[e]);
                        bpart += fa.x * fd.x + fa.y * fd.y;
                    } else {
                        bpart += __uint_as_float(aw[e]) * __uint_as_float(dw[e]);
                    }
                }
            }
        }
        // dkf_t partial from this part of the K row
        float dkf_part = 0.f;
        if (dk_direct && t < nvalid) {
            float dkrow[PW];
#pragma unroll
            for (int j = 0; j < NRAW; ++j) {
                const uint32_t w[4] = {dkraw[j].x, dkraw[j].y, dkraw[j].z, dkraw[j].w};
                if constexpr (sizeof(T) == 2) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = unpack_bf16(w[e]);
                        dkrow[j * 8 + 2 * e] = f.x;
                        dkrow[j * 8 + 2 * e + 1] = f.y;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) dkrow[j * 4 + e] = __uint_as_float(w[e]);
                }
            }
            float vk[32];
            tile_row32<T>(smem + L::kK, kBlockBytes, t, (hc * PW) & ~31, vk);
#pragma unroll
            for (int j = 0; j < PW; ++j) dkf_part += vk[j] * dkrow[j];
            if (PW == 16 && (hc & 1)) {  // odd parts: the upper 16 of the 32 loaded columns
                dkf_part = 0.f;
#pragma unroll
                for (int j = 0; j < PW; ++j) dkf_part += vk[(16 + j) & 31] * dkrow[j];
            }
        }
        mbar_wait(mma_done, ph);
        tc_fence_after();
        const uint32_t lo = (uint32_t)((warp & 3) * 32) << 16;
        // X_t, Y_t partials from this part of the Z, W rows against dO / V rows (smem)
        float xs = 0.f, ys = 0.f;
        {
            static_assert(PW == 32 || PW == 16, "state columns per thread");
            const int col = hc * PW;
            uint32_t rz[32], rw[32];
            if constexpr (PW == 32) {
                tmem_ld32(tmem + 256 + lo + col, rz);
                tmem_ld32(tmem + 384 + lo + col, rw);
            } else {
                uint32_t z16[16], w16[16];
                tmem_ld16(tmem + 256 + lo + col, z16);
                tmem_ld16(tmem + 384 + lo + col, w16);
#pragma unroll
                for (int j = 0; j < 16; ++j) { rz[j] = z16[j]; rw[j] = w16[j]; }
            }
            tmem_wait_ld();
            float vo[32], vv[32];
            tile_row32<T>(smem + L::kO, kBlockBytes, t, col & ~31, vo);
            tile_row32<T>(smem + L::kV, kBlockBytes, t, col & ~31, vv);
            // static register indices (PW == 16: odd parts read the upper half of the 32 loaded)
            if (PW == 32 || (hc & 1) == 0) {
#pragma unroll
                for (int j = 0; j < PW; ++j) {
                    xs += __uint_as_float(rz[j]) * vo[j];
                    ys += __uint_as_float(rw[j]) * vv[j];
                }
            } else {
#pragma unroll
                for (int j = 0; j < PW; ++j) {
                    xs += __uint_as_float(rz[j]) * vo[(16 + j) & 31];
                    ys += __uint_as_float(rw[j]) * vv[(16 + j) & 31];
                }
            }
        }
        sX[hc * 128 + t] = xs;
        sY[hc * 128 + t] = ys;
        sF[hc * 128 + t] = dkf_part;
        const float Gt = sG[t];
        __syncthreads();  // MMAs committed, every tile read done: the tiles are free
        if (tid == 0 && lin + (int)gridDim.x < total) issue(lin + gridDim.x);
        // strictly lower A_ts = S_ts kf_s dP_ts e^{G_t - G_s} (s < t) over this thread's 32
        // columns: row sums in the thread, column sums by the warp transpose-reduce
        float rsum = 0.f, csum;
        {
            const int s0 = hc * SW;
            uint32_t rs[32], rp[32];
            tmem_ld32(tmem + lo + s0, rs);
            tmem_ld32(tmem + 128 + lo + s0, rp);
            tmem_wait_ld();
            float a[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int s = s0 + j;
                a[j] = 0.f;
                if (s < t) a[j] = __uint_as_float(rs[j]) * __uint_as_float(rp[j]) * sKf[s] * __expf(Gt - sG[s]);
                rsum += a[j];
            }
            csum = warp_colsum32(a);
        }
        sR[hc * 128 + t] = rsum;
        sC[(warp & 3) * 128 + hc * SW + lane] = csum;  // column hc*32+lane over row quadrant warp&3
        __syncthreads();
        if (warp < 4) {
            float xsum = 0.f, ysum = 0.f, rs = 0.f, cs = 0.f;
#pragma unroll
            for (int i = 0; i < NH; ++i) {
                xsum += sX[i * 128 + t]; ysum += sY[i * 128 + t];
                rs += sR[i * 128 + t]; cs += sC[i * 128 + t];
            }
            const float X = t < nvalid ? __expf(Gt) * xsum : 0.f;
            const float Y = t < nvalid ? __expf(gend - Gt) * sKf[t] * ysum : 0.f;
            // dg_t = C(t) + sum_{u >= t} X_u + sum_{s < t} Y_s + e^{g_c} <M_c, dM_c>
            const float dlt = cs - rs;
            float Cin = dlt, Xin = X, Yin = Y, Xtot;
            scan3_w03(Cin, Xin, Yin, Xtot, ws + 32);  // inclusive prefixes, one barrier pair
            Cin -= dlt;                               // exclusive
            const float Xsuf = Xtot - Xin + X;
            const float Ypre = Yin - Y;
            sX[t] = Cin + Xsuf + Ypre;  // dg without the boundary term
        }
        // boundary term over all threads
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bpart += __shfl_xor_sync(0xFFFFFFFFu, bpart, o);
        if (lane == 0) ws[8 + warp] = bpart;
        __syncthreads();
        if (warp < 4) {
            float Bc = 0.f;
#pragma unroll
            for (int i = 0; i < 4 * NH; ++i) Bc += ws[8 + i];
            Bc *= __expf(gend);
            const float dg = sX[t] + Bc;
            float dkf_t = 0.f;
            if (t < nvalid) {
                float f = 0.f;
#pragma unroll
                for (int i = 0; i < NH; ++i) f += sF[i * 128 + t];
                dkf_t = dk_direct ? f / kf : dkf[(size_t)bh * N + t0 + t];
            }
            float dr = 0.f;
            if (t < nvalid) {
                const size_t row = ((size_t)b * N + t0 + t) * H + h;
                db_pre[row] = sigm(bv) * (dkf_t - spa * dg);
                dr = dg * -kf;
            }
            dr = sum128_w03(dr, ws);
            if (tid == 0) atomicAdd(da_raw + h, dr * sigm(a_raw[h]));
        }
        tc_fence_before();
        __syncthreads();  // TMEM, sG / sKf and the partials are reused by the next chunk
        tc_fence_after();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <typename T>
static cudaError_t dgate_t(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                           const CUtensorMap& dO, const CUtensorMap& m, const CUtensorMap& dm,
                           const float* b_pre, const float* a_raw, const float* dkf, const void* dk,
                           float* db_pre, float* da_raw, int B, int N, int H, cudaStream_t st) {
    constexpr int smem = DgateSmem<T>::kTotal;
    if (cudaError_t e = ensure_smem((const void*)lsm_mamba_dgate<T>, smem); e != cudaSuccess) return e;
    const int nchunk = (N + kC - 1) / kC;
    const int total = nchunk * B * H;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // L2 prefetch distance in chunks beyond the directly loaded next one (LMOE_DG_PF waves)
    const char* e = getenv("LMOE_DG_PF");
    const int pf = (e ? atoi(e) : 0) * sms;  // off: the next chunk's direct loads overlap already
    int grid = std::min(total, sms);
    if (const char* g = getenv("LMOE_DG_GRID"))  // test knob: fewer CTAs, many chunks each
        grid = std::max(1, std::min(grid, atoi(g)));
    cudaError_t r = cudaMemsetAsync(da_raw, 0, sizeof(float) * H, st);
    if (r != cudaSuccess) return r;
    lsm_mamba_dgate<T><<<grid, kDgThreads, smem, st>>>(q, k, v, dO, m, dm, b_pre, a_raw, dkf,
                                                       static_cast<const T*>(dk), db_pre, da_raw, N, H,
                                                       nchunk, total, pf > 0 ? pf + grid : 0);
    return cudaGetLastError();
}

cudaError_t launch_mamba_dgate(bool bf16, const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                               const CUtensorMap& dO, const CUtensorMap& m, const CUtensorMap& dm,
                               const float* b_pre, const float* a_raw, const float* dkf, const void* dk,
                               float* db_pre, float* da_raw, int B, int N, int H, cudaStream_t st) {
    return bf16 ? dgate_t<__nv_bfloat16>(q, k, v, dO, m, dm, b_pre, a_raw, dkf, dk, db_pre, da_raw, B, N, H, st)
                : dgate_t<float>(q, k, v, dO, m, dm, b_pre, a_raw, dkf, dk, db_pre, da_raw, B, N, H, st);
}

}  // namespace lmoe_dev
