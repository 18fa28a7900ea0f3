// lsm_vec_bwd.cu -- backward of the TokenVector-decay LSM (GLA / HGRN2 / RWKV6, lsm.hpp:64-85,
// 483-518) on sm_100a, bf16 operands, head dim 128.
//
// The reference differentiates chunk_forward_separable (lsm.hpp:554-598) on its tape
// (tensor.hpp:1178-1215).  Per key column c, with la_t = log sigmoid(a_t), G the inclusive
// cumulative log decay and A_ts = q_t[c] keff_s[c] e^{G_t[c]-G_s[c]} (dO_t . v_s):
//   dq_t   = dO_t M_t^T                       (M_t the state after token t)
//   dkeff_s= v_s dM_s^T                        (dM_s = dL/dM_s, the adjoint state)
//   dv_s   = sum_{t>=s} (q_t . e^{G_t-G_s} . keff_s) dO_t + keff_s-weighted dM_final
//   dla_j  = sum_{t>=j} sum_{s<j} A_ts
// Here the sequence is cut into 128-token chunks and every chunk is differentiated
// independently, given the state before it (M_c) and the adjoint after it (X_{c+1}):
//   1. lsm_state_pass_vec (forward) + segment combine      -> M at every segment start
//   2. lsm_vec_carry<FWD>   per segment, chunk by chunk   -> snapM[c] = M before chunk c (bf16)
//   3. lsm_state_pass_vec<REV> + reverse combine           -> X at every segment end, dM0
//   4. lsm_vec_carry<REV>                                  -> snapX[c+1] = X after chunk c,
//                                                             bd[c][k] = <M_c[k,:], X_c[k,:]>
//   5. lsm_vec_bwd_chunk    one CTA per chunk: dq, dk, dv, da_pre.
// The gate gradient avoids the sequence-long cancellation of the telescoped identity
// dla_j = sum_{t>=j} (q.dq - keff.dkeff)_t: inside a chunk [a, b) the same identity holds
// with the sum stopped at the chunk end plus the exact boundary term
//   dla_j = sum_{t in [j,b)} (q.dq - keff.dkeff)_t + <M_{b-1}[c,:], X_b[c,:]>,
// so the cancellation spans at most 128 tokens.  Inside the chunk the pairwise decay is
// folded into the operands around the midpoint r = G_63 (as in the forward,
// lsm_vec_kernels.cuh): q~ = q e^{G-r}, k~ = keff e^{r-G}, and
//   dq    = e^{G-r} . (dP_m k~ + dO (diag(e^r) M_c)^T)
//   dkeff = e^{r-G} . (dP_m^T q~ + V (diag(e^{G_end-r}) X)^T)
//   dv    = (S_m^T dO) + k~ (diag(e^{G_end-r}) X)
// with dP_m = (dO V^T) . [s<=t], S_m = (q~ k~^T) . [s<=t]; and q.dq - keff.dkeff =
// q~.dq' - k~.dk' needs no per-element factor.
#include "lsm_launch.h"
#include "lsm_vec_kernels.cuh"
#include "lsm_vec_scan.cuh"

namespace lmoe_dev {


// ====================================================================================
// Carry pass: per (b,h,segment) the state is carried chunk by chunk in TMEM and written
// out (bf16) at every chunk boundary.
//   FWD: snap[c]   = M;  M <- diag(e^{G_end}) M + (keff . e^{G_end - G})^T V
//   REV: snap[c+1] = X;  X <- diag(e^{G_end}) X + (q . e^{G})^T dO      (chunks last-to-first)
// Every weight is <= 1, so no range restriction applies here.  Warps: 0 TMA, 1 MMA,
// 4-11 transforms (2-D scan layout); warps 4-7 also own the TMEM state rows (row = key c).
// ====================================================================================
constexpr int kCarryThreads = 128 + kVecNT;
constexpr int kCarryStages = 2;
constexpr int carry_smem() { return kCarryStages * 3 * kTileBytes + (16 + 3) * 128 * 4 + 128; }

template <bool HG, bool REV>
__global__ void __launch_bounds__(kCarryThreads, 1)
    lsm_vec_carry(const __grid_constant__ CUtensorMap tmX1, const __grid_constant__ CUtensorMap tmX2,
                  const __grid_constant__ CUtensorMap tmA, VecBwdParams p) {
    using T = __nv_bfloat16;
    using TT = TileTraits<T>;
    constexpr int D = TT::D;
    constexpr int NST = kCarryStages;
    constexpr int STAGE = 3 * kTileBytes;  // X1 | X2 | A
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    float* sTot = reinterpret_cast<float*>(smem + NST * STAGE);  // [16][D]
    float* sR = sTot + 16 * D;
    float* sGe = sR + D;
    float* sG0 = sGe + D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sG0 + D);
    uint64_t* full = bars;         // [NST]
    uint64_t* empty = bars + NST;  // [NST]
    uint64_t* xf = bars + 2 * NST;
    uint64_t* acc = xf + 1;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(acc + 1);

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int c_first = t_begin / kC;
    const int warp = warp_id(), lane = lane_id();
    auto chunk_idx = [&](int it) { return c_first + (REV ? nchunks - 1 - it : it); };

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(xf, kVecNT);
        mbar_init(acc, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<128>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmX1); tma_prefetch(&tmX2); tma_prefetch(&tmA);
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % NST;
                if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
                const int t0 = chunk_idx(it) * kC;
                // REV: the forward snapshot this chunk's boundary dot reads (owner rows, below)
                if constexpr (REV)
                    bulk_prefetch_l2(p.snap_fwd + ((size_t)bh * (p.nchunk + 1) + chunk_idx(it) + 1) * D * D,
                                     D * D * sizeof(T));
                uint8_t* st = smem + s * STAGE;
                mbar_expect_tx(&full[s], STAGE);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    tma_load_4d(st + blk * kBlockBytes, &tmX1, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + kTileBytes + blk * kBlockBytes, &tmX2, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + 2 * kTileBytes + blk * kBlockBytes, &tmA, &full[s], blk * TT::EPB, h, t0, b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc(TT::FMT, 1, 1, 128, D);
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % NST;
                mbar_wait(&full[s], (it / NST) & 1);
                mbar_wait(xf, it & 1);
                tc_fence_after();
                const uint32_t xa = smem_u32(smem + s * STAGE), xb = xa + kTileBytes;
#pragma unroll
                for (int kk = 0; kk < kC / TT::KSTEP; ++kk)
                    mma_ss_f16(tmem, umma_desc_sw128(xa + kk * TT::KSTEP * 128, kBlockBytes, 1024),
                               umma_desc_sw128(xb + kk * TT::KSTEP * 128, kBlockBytes, 1024), idesc, 1u);
                mma_commit(&empty[s]);
                mma_commit(acc);
            }
        }
    } else if (warp >= 4) {
        using L = VecLayout<T>;
        const int tid = threadIdx.x - 128;
        const int cg = tid & 15, rg = tid >> 4;
        const bool owner = warp < 8;  // TMEM state row c = tid
        const int c = tid;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        // state entering this segment
        if (owner) {
            const float* src = p.Min + (((size_t)bh * p.nseg + seg) * D + c) * D;
#pragma unroll
            for (int cb = 0; cb < D / 32; ++cb) {
                uint32_t r[32];
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    const float4 f = *reinterpret_cast<const float4*>(src + cb * 32 + j);
                    r[j] = __float_as_uint(f.x); r[j + 1] = __float_as_uint(f.y);
                    r[j + 2] = __float_as_uint(f.z); r[j + 3] = __float_as_uint(f.w);
                }
                tmem_st32(tmem + lane_off + cb * 32, r);
            }
            tmem_wait_st();
        }
        // REV: row c of the forward snapshot idx, loaded before the wait for the MMA so its
        // latency hides behind it (the TMA warp has prefetched the snapshot into L2)
        uint4 mrow[REV ? D / 8 : 1];
        auto load_mrow = [&](int idx) {
            if constexpr (REV) {
                const uint4* src = reinterpret_cast<const uint4*>(p.snap_fwd + (((size_t)bh * (p.nchunk + 1) + idx) * D + c) * D);
#pragma unroll
                for (int u = 0; u < D / 8; ++u) mrow[u] = src[u];
            }
        };
        auto snapshot = [&](int idx, float scale) {
            // write row c of the TMEM state to snap[idx] (bf16) and rescale it in place; REV also
            // forms the gate gradient's boundary term bd[idx][c] = <M_idx[c, :], X_idx[c, :]>
            // against the forward snapshot (written by the FWD carry before this pass)
            const size_t srow = ((size_t)bh * (p.nchunk + 1) + idx) * D + c;
            __nv_bfloat16* dst = p.snap + srow * D;
            float bdot = 0.f;
#pragma unroll
            for (int cb = 0; cb < D / 32; ++cb) {
                uint32_t r[32];
                tmem_ld32(tmem + lane_off + cb * 32, r);
                tmem_wait_ld();
                if constexpr (REV) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint4 mu = mrow[cb * 4 + u];
                        const uint32_t mw[4] = {mu.x, mu.y, mu.z, mu.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 f = unpack_bf16(mw[e]);
                            bdot += f.x * __uint_as_float(r[u * 8 + 2 * e]) + f.y * __uint_as_float(r[u * 8 + 2 * e + 1]);
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    uint4 u;
                    u.x = pack_bf16(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
                    u.y = pack_bf16(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                    u.z = pack_bf16(__uint_as_float(r[j + 4]), __uint_as_float(r[j + 5]));
                    u.w = pack_bf16(__uint_as_float(r[j + 6]), __uint_as_float(r[j + 7]));
                    *reinterpret_cast<uint4*>(dst + cb * 32 + j) = u;
                }
                if (scale != 1.f) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * scale);
                    tmem_st32(tmem + lane_off + cb * 32, r);
                }
            }
            tmem_wait_st();
            if constexpr (REV) p.bd_out[srow] = bdot;
        };
        for (int it = 0; it < nchunks; ++it) {
            const int s = it % NST;
            const int ci = chunk_idx(it);
            const int nvalid = min(kC, p.N - ci * kC);
            uint8_t* x1 = smem + s * STAGE;
            uint8_t* at = x1 + 2 * kTileBytes;
            mbar_wait(&full[s], (it / NST) & 1);
            float G[L::R][L::EPC];
            float nocarry = 0.f;
            vec_log_scan<T>(at, nvalid, tid, G, sTot, sR, sGe, sG0, nullptr, nocarry);
            // operand weights in place in the X1 tile: FWD e^{G_end - G} keff, REV e^{G} q
#pragma unroll
            float gev[L::EPC];
#pragma unroll
            for (int j = 0; j < L::EPC; ++j) gev[j] = REV ? 0.f : sGe[cg * L::EPC + j];
            for (int ii = 0; ii < L::R; ++ii) {
                const int row = rg * L::R + ii;
                const float vm = row < nvalid ? 1.f : 0.f;
                float x[L::EPC], av[L::EPC];
                ld_chunk<T>(x1, row, cg, x);
                if constexpr (HG && !REV) ld_chunk<T>(at, row, cg, av);
#pragma unroll
                for (int j = 0; j < L::EPC; ++j) {
                    const float w = vm * fast_exp(REV ? G[ii][j] : gev[j] - G[ii][j]);
                    float xv;
                    if constexpr (HG && !REV) xv = sigmoid_fast(-av[j]);
                    else xv = x[j];
                    x[j] = xv * w;
                }
                st_chunk<T>(x1, row, cg, x);
            }
            // state: wait for the previous chunk's MMA, snapshot, decay by the chunk total
            if (owner) {
                load_mrow(ci + 1);
                if (it > 0) mbar_wait(acc, (it - 1) & 1);
                tc_fence_after();
                snapshot(REV ? ci + 1 : ci, __expf(sGe[c]));
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(xf);
        }
        if (owner) {
            mbar_wait(acc, (nchunks - 1) & 1);
            tc_fence_after();
            if (REV ? seg == 0 : seg == p.nseg - 1) {
                load_mrow(0);
                snapshot(REV ? 0 : p.nchunk, 1.f);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<128>(tmem);
}

// ====================================================================================
// Fused chunk backward: one CTA per (chunk, h, b).  Warps 0 TMA, 1 MMA, 4-11 math.
// smem: Q | K | V | dO | A | M | X tiles (7 x 32 KB).  The 2-D scan scratch of the gate
// scan lives in the M tile region, so M and X are loaded once that scan is done (their
// latency hides behind the operand transforms) and the region is reused by the final
// gate-gradient scan once M' has been consumed.
// TMEM (512 cols): [0,128) dP -> packed dP_m | [128,256) dP^T -> packed | [256,384) S^T ->
// packed S_m^T | [384,512) dq' then dv;  dk' halves in [64,128) and [192,256) once the
// packed operands have been written.
// ====================================================================================
constexpr int kVbThreads = 384;

// developer trace (LMOE_TRACE): clock64 at phase `slot` of the CTA of chunk nchunk / 2, head 0;
// row = warp role (0 TMA, 1 MMA, 2 math warp 4)
__device__ __forceinline__ void vb_mark(const VecBwdParams& p, int role, int slot) {
    if (p.trace != nullptr && blockIdx.x == p.nchunk / 2 && blockIdx.y == 0 && blockIdx.z == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[role * 16 + slot] = t;
    }
}
constexpr int vb_smem() { return 7 * kTileBytes + 3 * 128 * 4 + 256; }

// 8 consecutive bf16 of row `row`, columns [col8*8, col8*8+8) of a two-block SW128 tile
__device__ __forceinline__ uint4* tile_chunk(uint8_t* tile, int row, int col8) {
    return reinterpret_cast<uint4*>(tile + (col8 >> 3) * kBlockBytes + sw128_off(row, col8 & 7));
}

template <bool HG>
__global__ void __launch_bounds__(kVbThreads, 1)
    lsm_vec_bwd_chunk(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                      const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                      const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDQ,
                      const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV,
                      const __grid_constant__ CUtensorMap tmDA, VecBwdParams p) {
    using T = __nv_bfloat16;
    constexpr int D = 128;
    constexpr int NM = 256;  // math threads
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* Qt = smem;
    uint8_t* Kt = Qt + kTileBytes;
    uint8_t* Vt = Qt + 2 * kTileBytes;
    uint8_t* Ot = Qt + 3 * kTileBytes;  // dO
    uint8_t* At = Qt + 4 * kTileBytes;  // a_pre -> e^{G-r} -> q~dq' - k~dk'
    uint8_t* Mt = Qt + 5 * kTileBytes;
    uint8_t* Xt = Qt + 6 * kTileBytes;
    float* sTot = reinterpret_cast<float*>(Mt);  // [16][128] scan scratch (M region, see above)
    float* sR = reinterpret_cast<float*>(Qt + 7 * kTileBytes);
    float* sGe = sR + D;
    float* sG0 = sGe + D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sG0 + D);
    uint64_t* full = bars;
    uint64_t* xf = bars + 1;
    uint64_t* s_full = bars + 2;
    uint64_t* p_full = bars + 3;
    uint64_t* dq_full = bars + 4;
    uint64_t* dk_full = bars + 5;
    uint64_t* dq_free = bars + 6;
    uint64_t* dv_full = bars + 7;
    uint64_t* q_free = bars + 8;
    uint64_t* a_full = bars + 9;
    uint64_t* scan_done = bars + 10;
    uint64_t* mx_full = bars + 11;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 12);

    const int ci = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t0 = ci * kC;
    const int nvalid = min(kC, p.N - t0);
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(xf, NM);
        mbar_init(s_full, 1);
        mbar_init(p_full, NM);
        mbar_init(dq_full, 1);
        mbar_init(dk_full, 1);
        mbar_init(dq_free, NM);
        mbar_init(dv_full, 1);
        mbar_init(q_free, NM);
        mbar_init(a_full, 1);
        mbar_init(scan_done, NM);
        mbar_init(mx_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    const uint32_t T0 = tmem, T1 = tmem + 128, T2 = tmem + 256, T3 = tmem + 384;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmDO);
            tma_prefetch(&tmA); tma_prefetch(&tmM); tma_prefetch(&tmX);
            const int mrow = (bh * (p.nchunk + 1) + ci) * D;
            const int xrow = (bh * (p.nchunk + 1) + ci + 1) * D;
            vb_mark(p, 0, 0);
            mbar_expect_tx(full, 5 * kTileBytes);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                const int c0 = blk * 64;
                tma_load_4d(At + blk * kBlockBytes, &tmA, full, c0, h, t0, b);
                tma_load_4d(Qt + blk * kBlockBytes, &tmQ, full, c0, h, t0, b);
                tma_load_4d(Kt + blk * kBlockBytes, &tmK, full, c0, h, t0, b);
                tma_load_4d(Vt + blk * kBlockBytes, &tmV, full, c0, h, t0, b);
                tma_load_4d(Ot + blk * kBlockBytes, &tmDO, full, c0, h, t0, b);
            }
            mbar_expect_tx(mx_full, 2 * kTileBytes);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) tma_load_2d(Xt + blk * kBlockBytes, &tmX, mx_full, blk * 64, xrow);
            // warm L2 with the tiles of the CTA one wave ahead (one CTA per SM, linear launch
            // order): its loads then come from L2 while this SM computes (as lsm_mamba_dgate)
            if (p.pf_ahead > 0) {
                const long long lin = ci + (long long)gridDim.x * (h + (long long)gridDim.y * b) + p.pf_ahead;
                if (lin < (long long)gridDim.x * gridDim.y * gridDim.z) {
                    const int c2 = (int)(lin % gridDim.x), bh2 = (int)(lin / gridDim.x);
                    const int h2 = bh2 % p.H, b2 = bh2 / p.H, t2 = c2 * kC;
                    const int mrow2 = (bh2 * (p.nchunk + 1) + c2) * D, xrow2 = mrow2 + D;
#pragma unroll
                    for (int blk = 0; blk < 2; ++blk) {
                        const int c0 = blk * 64;
                        tma_prefetch_l2_4d(&tmA, c0, h2, t2, b2);
                        tma_prefetch_l2_4d(&tmQ, c0, h2, t2, b2);
                        tma_prefetch_l2_4d(&tmK, c0, h2, t2, b2);
                        tma_prefetch_l2_4d(&tmV, c0, h2, t2, b2);
                        tma_prefetch_l2_4d(&tmDO, c0, h2, t2, b2);
                        tma_prefetch_l2_2d(&tmM, c0, mrow2);
                        tma_prefetch_l2_2d(&tmX, c0, xrow2);
                    }
                }
            }
            mbar_wait(scan_done, 0);  // the scan scratch in the M region is dead
            vb_mark(p, 0, 1);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) tma_load_2d(Mt + blk * kBlockBytes, &tmM, mx_full, blk * 64, mrow);
            // raw gates again for the gate-gradient scan, into the M region once dO M'^T is done
            mbar_wait(s_full, 0);
            vb_mark(p, 0, 2);
            mbar_expect_tx(a_full, kTileBytes);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) tma_load_4d(Mt + blk * kBlockBytes, &tmA, a_full, blk * 64, h, t0, b);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idSS = umma_idesc(1, 0, 0, 128, 128);   // A K-major, B K-major
            constexpr uint32_t idTS = umma_idesc(1, 0, 1, 128, 128);   // B MN-major
            constexpr uint32_t idTSh = umma_idesc(1, 0, 1, 128, 64);
            constexpr uint32_t idSSh = umma_idesc(1, 0, 0, 128, 64);
            constexpr uint32_t idSM = umma_idesc(1, 0, 1, 128, 128);   // A K-major, B MN-major
            const uint32_t q = smem_u32(Qt), k = smem_u32(Kt), v = smem_u32(Vt), o = smem_u32(Ot);
            const uint32_t m = smem_u32(Mt), x = smem_u32(Xt);
            auto kdesc = [](uint32_t base, int kk) {  // K-major operand, K slice kk of 16
                return umma_desc_sw128(base + (kk >> 2) * kBlockBytes + (kk & 3) * 32, 16, 1024);
            };
            auto mdesc = [](uint32_t base, int kk) {  // MN-major operand, K rows [16kk, 16kk+16)
                return umma_desc_sw128(base + kk * 16 * 128, kBlockBytes, 1024);
            };
            mbar_wait(full, 0);
            vb_mark(p, 1, 0);
            mbar_wait(mx_full, 0);
            vb_mark(p, 1, 1);
            mbar_wait(xf, 0);
            vb_mark(p, 1, 2);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ss_f16(T0, kdesc(o, kk), kdesc(v, kk), idSS, kk > 0);  // dP
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ss_f16(T1, kdesc(v, kk), kdesc(o, kk), idSS, kk > 0);  // dP^T
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ss_f16(T2, kdesc(k, kk), kdesc(q, kk), idSS, kk > 0);  // S^T
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ss_f16(T3, kdesc(o, kk), kdesc(m, kk), idSS, kk > 0);  // dO M'^T
            mma_commit(s_full);
            mbar_wait(p_full, 0);
            vb_mark(p, 1, 3);
            tc_fence_after();
            // dq' += dP_m k~
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ts_f16(T3, T0 + kk * 8, mdesc(k, kk), idTS, 1u);
            mma_commit(dq_full);
            // dk' = dP_m^T q~ + V X'^T, two N = 64 halves
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const uint32_t dst = hf ? tmem + 192 : tmem + 64;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts_f16(dst, T1 + kk * 8, mdesc(q + hf * kBlockBytes, kk), idTSh, kk > 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ss_f16(dst, kdesc(v, kk), kdesc(x + hf * 8192, kk), idSSh, 1u);
            }
            mma_commit(dk_full);
            // dv = S_m^T dO + k~ X'   (into [384,512) once dq' has been read)
            mbar_wait(dq_free, 0);
            vb_mark(p, 1, 4);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ts_f16(T3, T2 + kk * 8, mdesc(o, kk), idTS, kk > 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_ss_f16(T3, kdesc(k, kk), mdesc(x, kk), idSM, 1u);
            mma_commit(dv_full);
        }
    } else if (warp >= 4) {
        const int tid = threadIdx.x - 128;  // 0..255
        // ---------------- (T) 2-D column scan, operand transforms, M' / X' row scales
        using L = VecLayout<T>;
        const int cg = tid & 15, rg = tid >> 4;
        mbar_wait(full, 0);
        if (threadIdx.x == 128) vb_mark(p, 2, 0);
        {
            float G[L::R][L::EPC];
            float nocarry = 0.f;
            vec_log_scan<T>(At, nvalid, tid, G, sTot, sR, sGe, sG0, nullptr, nocarry);
            mbar_arrive(scan_done);
            if (threadIdx.x == 128) vb_mark(p, 2, 1);
            if (tid < D && !vec_split_ok(sG0[tid], sR[tid], sGe[tid])) atomicOr(&p.err[2], 1);
            float rr[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) rr[j] = sR[cg * 8 + j];
#pragma unroll
            for (int ii = 0; ii < L::R; ++ii) {
                const int i = rg * L::R + ii;
                const float vm = i < nvalid ? 1.f : 0.f;
                float xq[8], xk[8], xa[8];
                ld_chunk<T>(Qt, i, cg, xq);
                ld_chunk<T>(At, i, cg, xa);
                if constexpr (!HG) ld_chunk<T>(Kt, i, cg, xk);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float gr = G[ii][j] - rr[j];
                    const float e = fast_exp(gr);
                    const float keff = HG ? sigmoid_fast(-xa[j]) : xk[j];
                    xq[j] = xq[j] * (vm * e);
                    xk[j] = keff * (vm * fast_exp(-gr));
                    xa[j] = e;
                }
                st_chunk<T>(Qt, i, cg, xq);
                st_chunk<T>(Kt, i, cg, xk);
                st_chunk<T>(At, i, cg, xa);
            }
        }
        if (threadIdx.x == 128) vb_mark(p, 2, 2);
        mbar_wait(mx_full, 0);
        if (threadIdx.x == 128) vb_mark(p, 2, 3);
        {
            // M' = diag(e^r) M_c, X' = diag(e^{G_end - r}) X_{c+1}: thread = (row, column block)
            const int row = tid & 127, blk = tid >> 7;
            xform_half_row<T, 0, false>(Mt + blk * kBlockBytes, row, __expf(sR[row]));
            xform_half_row<T, 0, false>(Xt + blk * kBlockBytes, row, __expf(sGe[row] - sR[row]));
        }
        fence_proxy_async_smem();
        mbar_arrive(xf);

        // ---------------- (E1) masks, packed bf16 operands in TMEM (row layout)
        const int mw = warp - 4;
        const int qd = warp & 3, hh = mw >> 2;
        const int row = qd * 32 + lane;
        const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
        mbar_wait(s_full, 0);
        if (threadIdx.x == 128) vb_mark(p, 2, 4);
        tc_fence_after();
        auto pack_masked = [&](uint32_t base, bool lower, uint32_t (&pk)[32]) {
            uint32_t r0[32], r1[32];
            tmem_ld32(base + lane_off + hh * 64, r0);
            tmem_ld32(base + lane_off + hh * 64 + 32, r1);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c0 = hh * 64 + 2 * j, c1 = c0 + 32;
                // lower: keep col <= row (dP, rows t / cols s); else keep col >= row (transposed)
                const bool k00 = lower ? c0 <= row : c0 >= row, k01 = lower ? c0 + 1 <= row : c0 + 1 >= row;
                const bool k10 = lower ? c1 <= row : c1 >= row, k11 = lower ? c1 + 1 <= row : c1 + 1 >= row;
                pk[j] = pack_bf16(k00 ? __uint_as_float(r0[2 * j]) : 0.f, k01 ? __uint_as_float(r0[2 * j + 1]) : 0.f);
                pk[16 + j] = pack_bf16(k10 ? __uint_as_float(r1[2 * j]) : 0.f, k11 ? __uint_as_float(r1[2 * j + 1]) : 0.f);
            }
        };
        {
            uint32_t pa[32], pb[32];
            pack_masked(T0, true, pa);
            pack_masked(T1, false, pb);
            named_bar_sync(1, NM);  // every fp32 read of these regions precedes the packed writes
            tmem_st32(T0 + lane_off + hh * 32, pa);
            tmem_st32(T1 + lane_off + hh * 32, pb);
            pack_masked(T2, false, pa);
            named_bar_sync(1, NM);
            tmem_st32(T2 + lane_off + hh * 32, pa);
            tmem_wait_st();
        }
        tc_fence_before();
        mbar_arrive(p_full);

        // ---------------- (E2) dq, dk and the gate integrand q~dq' - k~dk'.  bf16 dq / dk are
        // staged in the dead q~ / V tiles (own elements only) and written with TMA bulk stores.
        if (threadIdx.x == 128) vb_mark(p, 2, 5);
        mbar_wait(dq_full, 0);
        mbar_wait(dk_full, 0);
        if (threadIdx.x == 128) vb_mark(p, 2, 6);
        tc_fence_after();
        const bool f32out = p.out_f32 != 0;
        {
            const bool vrow = row < nvalid;
            const size_t grow = (((size_t)b * p.N + t0 + (vrow ? row : 0)) * p.H + h) * D;
#pragma unroll 1
            for (int cb = 0; cb < 2; ++cb) {
                const int cbase = hh * 64 + cb * 32;
                uint32_t rq[32], rk[32];
                tmem_ld32(T3 + lane_off + cbase, rq);
                tmem_ld32(tmem + 64 + hh * 128 + cb * 32 + lane_off, rk);
                tmem_wait_ld();
                float dqv[32], dkv[32];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const int c8 = cbase / 8 + ch;
                    const uint4 eu = *tile_chunk(At, row, c8);
                    const uint4 qu = *tile_chunk(Qt, row, c8);
                    const uint4 ku = *tile_chunk(Kt, row, c8);
                    const uint32_t* ew = reinterpret_cast<const uint32_t*>(&eu);
                    const uint32_t* qw = reinterpret_cast<const uint32_t*>(&qu);
                    const uint32_t* kw = reinterpret_cast<const uint32_t*>(&ku);
                    uint4 du, hu, qo, ko;
                    uint32_t* dw = reinterpret_cast<uint32_t*>(&du);
                    uint32_t* hw = reinterpret_cast<uint32_t*>(&hu);
                    uint32_t* qow = reinterpret_cast<uint32_t*>(&qo);
                    uint32_t* kow = reinterpret_cast<uint32_t*>(&ko);
#pragma unroll
                    for (int w2 = 0; w2 < 4; ++w2) {
                        const float2 e = unpack_bf16(ew[w2]), qq = unpack_bf16(qw[w2]), kq = unpack_bf16(kw[w2]);
                        const int j = ch * 8 + w2 * 2;
                        const float q0 = __uint_as_float(rq[j]), q1 = __uint_as_float(rq[j + 1]);
                        const float k0 = __uint_as_float(rk[j]), k1 = __uint_as_float(rk[j + 1]);
                        dqv[j] = e.x * q0; dqv[j + 1] = e.y * q1;
                        dkv[j] = HG ? 0.f : k0 * rcp_ftz(e.x); dkv[j + 1] = HG ? 0.f : k1 * rcp_ftz(e.y);
                        dw[w2] = pack_bf16(qq.x * q0 - kq.x * k0, qq.y * q1 - kq.y * k1);
                        if constexpr (HG) hw[w2] = pack_bf16(kq.x * k0, kq.y * k1);
                        qow[w2] = pack_bf16(dqv[j], dqv[j + 1]);
                        kow[w2] = pack_bf16(dkv[j], dkv[j + 1]);
                    }
                    *tile_chunk(At, row, c8) = du;  // own elements: no cross-thread hazard
                    if constexpr (HG) {
                        *tile_chunk(Vt, row, c8) = hu;  // V is dead once dk' is done
                    } else if (!f32out) {
                        *tile_chunk(Vt, row, c8) = ko;
                    }
                    if (!f32out) *tile_chunk(Qt, row, c8) = qo;
                }
                if (f32out && vrow) {
                    float* gq = static_cast<float*>(p.dq) + grow + cbase;
                    float* gk = static_cast<float*>(p.dk) + grow + cbase;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        *reinterpret_cast<float4*>(gq + j) = make_float4(dqv[j], dqv[j + 1], dqv[j + 2], dqv[j + 3]);
                        *reinterpret_cast<float4*>(gk + j) = make_float4(dkv[j], dkv[j + 1], dkv[j + 2], dkv[j + 3]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(dq_free);
            fence_proxy_async_smem();
            named_bar_sync(1, NM);
            if (tid == 0 && !f32out) {
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    tma_store_4d(&tmDQ, Qt + blk * kBlockBytes, blk * 64, h, t0, b);
                    if constexpr (!HG) tma_store_4d(&tmDK, Vt + blk * kBlockBytes, blk * 64, h, t0, b);
                }
                bulk_commit();
            }
            if (threadIdx.x == 128) vb_mark(p, 2, 7);
            // ---------------- (E3) dv, staged in the dead k~ tile (own elements)
            mbar_wait(dv_full, 0);
            if (threadIdx.x == 128) vb_mark(p, 2, 8);
            tc_fence_after();
#pragma unroll 1
            for (int cb = 0; cb < 2; ++cb) {
                const int cbase = hh * 64 + cb * 32;
                uint32_t rv[32];
                tmem_ld32(T3 + lane_off + cbase, rv);
                tmem_wait_ld();
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint4 a;
                    const int j = ch * 8;
                    a.x = pack_bf16(__uint_as_float(rv[j]), __uint_as_float(rv[j + 1]));
                    a.y = pack_bf16(__uint_as_float(rv[j + 2]), __uint_as_float(rv[j + 3]));
                    a.z = pack_bf16(__uint_as_float(rv[j + 4]), __uint_as_float(rv[j + 5]));
                    a.w = pack_bf16(__uint_as_float(rv[j + 6]), __uint_as_float(rv[j + 7]));
                    *tile_chunk(Kt, row, cbase / 8 + ch) = a;
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();
        }
        named_bar_sync(1, NM);  // the integrand tile and the staged dv are complete
        if (tid == 0) {
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) tma_store_4d(&tmDV, Kt + blk * kBlockBytes, blk * 64, h, t0, b);
            bulk_commit();
        }

        // ---------------- (S) gate gradient: reverse in-chunk scan + boundary term (2-D layout;
        // scratch in the dead X region, raw gates reloaded into the M region, da staged in dO)
        if (threadIdx.x == 128) vb_mark(p, 2, 9);
        mbar_wait(a_full, 0);
        if (threadIdx.x == 128) vb_mark(p, 2, 10);
        {
            float* sSc = reinterpret_cast<float*>(Xt);
            float Dv[L::R][8];
            float tot[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) tot[j] = 0.f;
#pragma unroll
            for (int ii = 0; ii < L::R; ++ii) {
                ld_chunk<T>(At, rg * L::R + ii, cg, Dv[ii]);
#pragma unroll
                for (int j = 0; j < 8; ++j) tot[j] += Dv[ii][j];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) sSc[rg * D + cg * 8 + j] = tot[j];
            named_bar_sync(1, NM);
            if (tid < D) {  // exclusive suffix over later row groups, seeded with the boundary term
                float acc = p.bd[((size_t)bh * (p.nchunk + 1) + ci + 1) * D + tid];
#pragma unroll
                for (int g = L::RG - 1; g >= 0; --g) {
                    const float v = sSc[g * D + tid];
                    sSc[g * D + tid] = acc;
                    acc += v;
                }
            }
            named_bar_sync(1, NM);
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = sSc[rg * D + cg * 8 + j];
#pragma unroll
            for (int ii = L::R - 1; ii >= 0; --ii) {
                const int i = rg * L::R + ii;
                float av[8], kd[8], g[8];
                ld_chunk<T>(Mt, i, cg, av);  // raw a_pre (reloaded)
                if constexpr (HG) ld_chunk<T>(Vt, i, cg, kd);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    acc[j] += Dv[ii][j];
                    const float sg = sigmoid_fast(av[j]);
                    g[j] = acc[j] * (1.f - sg);
                    if constexpr (HG) g[j] -= kd[j] * sg;
                }
                st_chunk<T>(Ot, i, cg, g);
            }
            fence_proxy_async_smem();
            named_bar_sync(1, NM);
            if (tid == 0) {
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) tma_store_4d(&tmDA, Ot + blk * kBlockBytes, blk * 64, h, t0, b);
                bulk_commit();
                bulk_wait_read0();  // smem must outlive the bulk stores' reads of it
            }
        }
        if (threadIdx.x == 128) vb_mark(p, 2, 11);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------------------- launchers
template <bool HG, bool REV>
static cudaError_t carry_t(dim3 grid, cudaStream_t st, const CUtensorMap& x1, const CUtensorMap& x2,
                           const CUtensorMap& a, const VecBwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_vec_carry<HG, REV>, carry_smem()); e != cudaSuccess) return e;
    lsm_vec_carry<HG, REV><<<grid, kCarryThreads, carry_smem(), st>>>(x1, x2, a, p);
    return cudaGetLastError();
}

cudaError_t launch_vec_carry(bool hgrn2, bool rev, dim3 grid, cudaStream_t st, const CUtensorMap& x1,
                             const CUtensorMap& x2, const CUtensorMap& a, const VecBwdParams& p) {
    if (rev) return carry_t<false, true>(grid, st, x1, x2, a, p);
    return hgrn2 ? carry_t<true, false>(grid, st, x1, x2, a, p) : carry_t<false, false>(grid, st, x1, x2, a, p);
}

template <bool HG>
static cudaError_t chunk_t(dim3 grid, cudaStream_t st, const CUtensorMap* tm, const VecBwdParams& p) {
    if (cudaError_t e = ensure_smem((const void*)lsm_vec_bwd_chunk<HG>, vb_smem()); e != cudaSuccess) return e;
    lsm_vec_bwd_chunk<HG><<<grid, kVbThreads, vb_smem(), st>>>(tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], tm[6], tm[7],
                                                                tm[8], tm[9], tm[10], p);
    return cudaGetLastError();
}

// tm = {q, k, v, dO, a_pre, snapM, snapX, dq, dk, dv, da}
cudaError_t launch_vec_bwd_chunk(bool hgrn2, dim3 grid, cudaStream_t st, const CUtensorMap* tm,
                                 const VecBwdParams& p) {
    return hgrn2 ? chunk_t<true>(grid, st, tm, p) : chunk_t<false>(grid, st, tm, p);
}

}  // namespace lmoe_dev
