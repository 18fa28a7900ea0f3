// lsm_vec_kernels.cuh -- TokenVector decays (GLA, HGRN2, RWKV6; lsm.hpp:64-85) on sm_100a.
//
// Decay per (token t, key column k): a_tk = sigmoid(a_pre[t, k]) (decay_vector_rows,
// lsm.hpp:504-518); effective key phi(k) for GLA/RWKV6, 1 - a for HGRN2 (lsm.hpp:483-501).
// Per chunk, G[t][k] = inclusive log-space cumsum of log a down each column (column-slab
// scans by the math warps), and the pairwise factor e^{G_ik - G_jk} is folded into the
// operands around a per-column midpoint reference r_k = G[63][k]:
//     q~ = phi(q) e^{G - r},  k~ = keff e^{r - G}          (both finite while each
//                                                           half-chunk column span < 80)
//     S  = (q~ k~^T) . [j <= i]                             (no per-element factors)
//     O  = P V + q~ (diag(e^r) M)                           (operand M' = diag(e^r) M)
//     M' += k~^T V ;  M_next = diag(e^{G_end - r}) M'       (state resident in TMEM)
// The state pass visits chunks last-to-first with one backward pass per column:
//     w_jk = e^{L_jk} keff_jk,  L_jk = sum of log a over tokens after j up to the segment end.
// A chunk whose half-chunk span exceeds the bound raises "non-finite output in div" -- the
// reference's own message for its K/p form (lsm.hpp:576-577) in the same regime.
// REV (backward adjoint states, lsm_vec_bwd.cu): the state pass visits chunks first-to-last
// with w_jk = e^{P_jk}, P_jk = log decay from the segment start through token j (inclusive),
// so S_seg = sum_j (phi(q_j) . w_j)^T dO_j is the segment's contribution to dM at its start.
#pragma once
#include "lsm_vec_scan.cuh"

namespace lmoe_dev {

__device__ __forceinline__ float log_sigmoid(float x) { return -softplus_f(-x); }
__device__ __forceinline__ float sigmoid_f(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }  // exact-ish (outside hot loops)

// element (row, col) of a [128 x 256 B] SW128 tile (two 128-B column blocks)
template <typename T>
__device__ __forceinline__ T* tile_elem(uint8_t* tile, int row, int col) {
    using TT = TileTraits<T>;
    const int blk = col / TT::EPB, cin = col % TT::EPB;
    return reinterpret_cast<T*>(tile + blk * kBlockBytes + sw128_off(row, cin / TT::EPC) +
                                (cin % TT::EPC) * sizeof(T));
}
template <typename T>
__device__ __forceinline__ float ld_elem(uint8_t* tile, int row, int col) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(*tile_elem<T>(tile, row, col));
    else return *tile_elem<T>(tile, row, col);
}
template <typename T>
__device__ __forceinline__ void st_elem(uint8_t* tile, int row, int col, float v) {
    if constexpr (sizeof(T) == 2) *tile_elem<T>(tile, row, col) = __float2bfloat16_rn(v);
    else *tile_elem<T>(tile, row, col) = tf32r(v);
}
// fp32 transposed K-major tile [64 d rows x 128 tok]
__device__ __forceinline__ float* tr_elem(uint8_t* tileT, int d, int tok) {
    return reinterpret_cast<float*>(tileT + (tok >> 5) * 8192 + sw128_off(d, (tok & 31) >> 2) + ((tok & 3) << 2));
}

// ====================================================================================
// Phase 1 (vector decay): warps 0 TMA, 1 MMA, 2-3 idle, 4-11 transform (2-D layout,
// lsm_vec_scan.cuh); warps 4-7 also drain the TMEM accumulator.
// ====================================================================================
constexpr int kStatePassVecThreads = 128 + kVecNT;

template <typename T, int FM, bool NORM, bool HG, bool REV = false>
__global__ void __launch_bounds__(kStatePassVecThreads, 1)
    lsm_state_pass_vec(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ CUtensorMap tmA, LsmFwdParams p) {
    using TT = TileTraits<T>;
    using L = VecLayout<T>;
    constexpr int D = TT::D;
    constexpr int EPC = L::EPC;
    constexpr bool TR = TT::kTransposed;
    constexpr int NST = TR ? 1 : 2;
    constexpr int STAGE = 3 * kTileBytes;  // K | V | A
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* tiles = smem;
    uint8_t* kT = tiles + NST * STAGE;
    uint8_t* vT = kT + (TR ? kTileBytes : 0);
    float* sTot = reinterpret_cast<float*>(vT + (TR ? kTileBytes : 0));  // [RG][D]
    float* sR = sTot + L::RG * D;
    float* sGe = sR + D;
    float* sG0 = sGe + D;
    float* sCar = sG0 + D;
    float* sZ = sCar + D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sZ + D);
    uint64_t* full = bars;          // [NST]
    uint64_t* empty = bars + 2;     // [NST]
    uint64_t* xf = bars + 4;
    uint64_t* acc_full = bars + 5;
    uint64_t* kt_free = bars + 6;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 7);

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id();
    auto chunk_t0 = [&](int it) { return t_begin + (REV ? it : nchunks - 1 - it) * kC; };

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(xf, kVecNT);
        mbar_init(acc_full, 1);
        mbar_init(kt_free, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<128>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    pdl_wait();  // predecessor's outputs (segment states / prefixes) are visible from here
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmA);
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % NST;
                if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
                const int t0 = chunk_t0(it);
                uint8_t* st = tiles + s * STAGE;
                mbar_expect_tx(&full[s], STAGE);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    tma_load_4d(st + blk * kBlockBytes, &tmK, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + kTileBytes + blk * kBlockBytes, &tmV, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + 2 * kTileBytes + blk * kBlockBytes, &tmA, &full[s], blk * TT::EPB, h, t0, b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % NST;
                mbar_wait(&full[s], (it / NST) & 1);
                mbar_wait(xf, it & 1);
                tc_fence_after();
                const uint32_t kt = smem_u32(tiles + s * STAGE);
                const uint32_t vt = kt + kTileBytes;
                if constexpr (!TR) {
                    constexpr uint32_t idesc = umma_idesc(TT::FMT, 1, 1, 128, D);
#pragma unroll
                    for (int kk = 0; kk < kC / TT::KSTEP; ++kk)
                        mma_ss_f16(tmem, umma_desc_sw128(kt + kk * TT::KSTEP * 128, kBlockBytes, 1024),
                                   umma_desc_sw128(vt + kk * TT::KSTEP * 128, kBlockBytes, 1024), idesc,
                                   (it > 0 || kk > 0) ? 1u : 0u);
                } else {
                    constexpr uint32_t idesc = umma_idesc(TT::FMT, 0, 0, 64, D);
                    const uint32_t ka = smem_u32(kT), va = smem_u32(vT);
#pragma unroll
                    for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                        const uint32_t off = (kk >> 2) * 8192 + (kk & 3) * 32;
                        mma_ss_tf32(tmem, umma_desc_sw128(ka + off, 16, 1024), umma_desc_sw128(va + off, 16, 1024),
                                    idesc, (it > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(kt_free);
                }
                mma_commit(&empty[s]);
            }
            mma_commit(acc_full);
        }
    } else if (warp >= 4) {
        const int tid = threadIdx.x - 128;
        const int cg = tid & 15, rg = tid >> 4;
        // carry: FWD the log decay of the later chunks of the segment (suffix), REV of the
        // earlier ones (prefix); per column, held by threads tid < D
        float carry = 0.f;
        if constexpr (NORM) {
            if (tid < D) sZ[tid] = 0.f;
        }
        for (int it = 0; it < nchunks; ++it) {
            const int s = it % NST;
            uint8_t* kt = tiles + s * STAGE;
            uint8_t* vt = kt + kTileBytes;
            uint8_t* at = kt + 2 * kTileBytes;
            const int nvalid = min(kC, t_end - chunk_t0(it));
            mbar_wait(&full[s], (it / NST) & 1);
            if (TR && it >= 1) mbar_wait(kt_free, (it - 1) & 1);
            float G[L::R][EPC];
            vec_log_scan<T>(at, nvalid, tid, G, sTot, sR, sGe, sG0, sCar, carry);
            float zc[EPC];
#pragma unroll
            for (int j = 0; j < EPC; ++j) zc[j] = 0.f;
#pragma unroll
            float base[EPC];  // REV: prefix; FWD: G_end + suffix
#pragma unroll
            for (int j = 0; j < EPC; ++j) base[j] = sCar[cg * EPC + j] + (REV ? 0.f : sGe[cg * EPC + j]);
            for (int ii = 0; ii < L::R; ++ii) {
                const int row = rg * L::R + ii;
                const float vm = row < nvalid ? 1.f : 0.f;
                float x[EPC], av[EPC];
                ld_chunk<T>(kt, row, cg, x);
                if constexpr (HG && !REV) ld_chunk<T>(at, row, cg, av);
#pragma unroll
                for (int j = 0; j < EPC; ++j) {
                    // REV: w = e^{prefix + G}; FWD: w = e^{(G_end - G) + suffix} (both <= 1)
                    const float w = vm * fast_exp(REV ? base[j] + G[ii][j] : base[j] - G[ii][j]);
                    float keff;
                    if constexpr (HG && !REV) keff = sigmoid_fast(-av[j]);
                    else keff = fmap_t<FM>(x[j]);
                    x[j] = keff * w;
                    if constexpr (NORM) zc[j] += x[j];
                }
                if constexpr (!TR) {
                    st_chunk<T>(kt, row, cg, x);
                } else {
                    float vv[EPC];
                    ld_chunk<T>(vt, row, cg, vv);
#pragma unroll
                    for (int j = 0; j < EPC; ++j) {
                        *tr_elem(kT, cg * EPC + j, row) = tf32r(x[j]);
                        *tr_elem(vT, cg * EPC + j, row) = tf32r(vv[j]);
                    }
                }
            }
            if constexpr (NORM) {
#pragma unroll
                for (int j = 0; j < EPC; ++j) atomicAdd(&sZ[cg * EPC + j], zc[j]);
            }
            fence_proxy_async_smem();
            mbar_arrive(xf);
        }
        mbar_wait(acc_full, 0);
        tc_fence_after();
        if (warp < 8) {
            const int q = warp & 3;
            const uint32_t lane_off = (uint32_t)(q * 32) << 16;
            const int row = TR ? q * 16 + lane : q * 32 + lane;
            const bool own = TR ? lane < 16 : true;
            float* dst = p.Sseg + (((size_t)bh * p.nseg + seg) * D + (own ? row : 0)) * D;
#pragma unroll
            for (int cb = 0; cb < D / 32; ++cb) {
                uint32_t r[32];
                tmem_ld32(tmem + lane_off + cb * 32, r);
                tmem_wait_ld();
                if (own) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(dst + cb * 32 + j) =
                            make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                        __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                }
            }
        }
        named_bar_sync(1, kVecNT);  // sZ complete
        if (tid < D) {
            p.logDseg[((size_t)bh * p.nseg + seg) * D + tid] = carry;
            if constexpr (NORM) p.zseg[((size_t)bh * p.nseg + seg) * D + tid] = sZ[tid];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<128>(tmem);
}

// ====================================================================================
// Phase 3 (vector decay): warps 0 TMA, 1 MMA, 2-3 idle, 4-11 math (256 threads)
// TMEM: S [0,128), O [128,256), M [256,384) (tf32: O [128,192), M [192,256) M=64 layout);
// row partials (normaliser) in S columns 64.. (bf16) / [384,388) (tf32).
// ====================================================================================
// bf16: 16 math warps (four 32-column groups per row, as the scalar pass); tf32: 8
template <typename T>
constexpr int vec_math_threads() { return sizeof(T) == 2 ? 512 : 256; }
template <typename T>
constexpr int output_pass_vec_threads() { return 128 + vec_math_threads<T>(); }

template <typename T, int FM, bool NORM, bool HG>
__global__ void __launch_bounds__(output_pass_vec_threads<T>(), 1)
    lsm_output_pass_vec(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmO, LsmFwdParams p) {
    using TT = TileTraits<T>;
    constexpr int D = TT::D;
    constexpr bool kBF16 = sizeof(T) == 2;
    constexpr bool TR = TT::kTransposed;
    constexpr int NM = vec_math_threads<T>();
    constexpr int NQ = NM / 128;  // column groups per row in the row-layout phases
    constexpr int DH = D / NQ;    // state / O columns per thread (32)
    static_assert(DH == 32, "row-layout phases assume 32 columns per thread");
    using L = VecLayout<T, NM>;
    // Gate tiles are double-buffered for bf16 (the next one loads while this chunk runs, so
    // its scan overlaps the Q / K / V loads); each gate buffer then holds its chunk's state
    // operand M' (dead gate tile), freed by the QM GEMM.
    constexpr int NAB = kBF16 ? 2 : 1;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* qt = smem;
    uint8_t* kt = qt + kTileBytes;
    uint8_t* vt = qt + 2 * kTileBytes;
    uint8_t* abase = qt + 3 * kTileBytes;
    uint8_t* kT = abase + NAB * kTileBytes;
    uint8_t* vT = kT + (TR ? kTileBytes : 0);
    uint8_t* ostg = vT + (TR ? kTileBytes : 0);  // bf16: O staging for the bulk tensor store
    float* sOffI = reinterpret_cast<float*>(ostg + (kBF16 ? kTileBytes : 0));  // [RG][D] group factors
    float* sER = sOffI + L::RG * D;                                 // [D] e^{r} = prod sigma rows < 64
    float* sEG = sER + D;                                           // [D] e^{G_end - r} = prod rows >= 64
    float* sZ = sEG + D;                                            // [D]
    float* sZP = sZ + D;                                            // [D]  e^r z
    float* sZC = sZP + D;                                           // [D]  this chunk's colsum of k~
    uint64_t* bars = reinterpret_cast<uint64_t*>(sZC + D);
    uint64_t* full = bars;
    uint64_t* empty = bars + 1;
    uint64_t* xf = bars + 2;
    uint64_t* s_full = bars + 3;
    uint64_t* p_full = bars + 4;
    uint64_t* mo_full = bars + 5;
    uint64_t* a_full = bars + 6;  // [NAB]
    uint64_t* a_free = bars + 8;  // [NAB]
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 10);
    auto abuf = [&](int c) { return abase + (c % NAB) * kTileBytes; };

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(empty, 1);
        mbar_init(xf, NM);
        mbar_init(s_full, 1);
        mbar_init(p_full, NM);
        mbar_init(mo_full, 1);
        for (int i = 0; i < NAB; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_free[i], 1); }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    pdl_wait();  // predecessor's outputs (segment states / prefixes) are visible from here
    pdl_trigger();
    const uint32_t tS = tmem, tO = tmem + 128, tM = tmem + (kBF16 ? 256 : 192);

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmA);
            for (int c = 0; c < nchunks; ++c) {
                const int t0 = t_begin + c * kC;
                const int ab = c % NAB;
                if (c >= NAB) mbar_wait(&a_free[ab], ((c / NAB) - 1) & 1);  // M'(c - NAB) consumed
                mbar_expect_tx(&a_full[ab], kTileBytes);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk)
                    tma_load_4d(abuf(c) + blk * kBlockBytes, &tmA, &a_full[ab], blk * TT::EPB, h, t0, b);
                if (c >= 1) mbar_wait(empty, (c - 1) & 1);
                trace_mark(p, c, 10);
                mbar_expect_tx(full, 3 * kTileBytes);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    tma_load_4d(qt + blk * kBlockBytes, &tmQ, full, blk * TT::EPB, h, t0, b);
                    tma_load_4d(kt + blk * kBlockBytes, &tmK, full, blk * TT::EPB, h, t0, b);
                    tma_load_4d(vt + blk * kBlockBytes, &tmV, full, blk * TT::EPB, h, t0, b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc(TT::FMT, 0, 0, 128, 128);
            constexpr uint32_t idPV = umma_idesc(TT::FMT, 0, TR ? 0 : 1, 128, D);
            constexpr uint32_t idQM = umma_idesc(TT::FMT, 0, TR ? 0 : 1, 128, D);
            constexpr uint32_t idDM = TR ? umma_idesc(TT::FMT, 0, 0, 64, D) : umma_idesc(TT::FMT, 1, 1, 128, D);
            const uint32_t qa = smem_u32(qt), ka = smem_u32(kt), va = smem_u32(vt);
            const uint32_t kTa = smem_u32(kT), vTa = smem_u32(vT);
            for (int c = 0; c < nchunks; ++c) {
                const uint32_t mb = smem_u32(abuf(c));  // M' lives in this chunk's gate buffer
                mbar_wait(full, c & 1);
                mbar_wait(xf, c & 1);
                tc_fence_after();
                // S = q~ k~^T ; O = q~ M' ; M' += k~^T V
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    const uint64_t a = umma_desc_sw128(qa + off, 16, 1024);
                    if constexpr (kBF16) mma_ss_f16(tS, a, umma_desc_sw128(ka + off, 16, 1024), idS, kk > 0);
                    else mma_ss_tf32(tS, a, umma_desc_sw128(ka + off, 16, 1024), idS, kk > 0);
                }
                mma_commit(s_full);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    const uint64_t a = umma_desc_sw128(qa + off, 16, 1024);
                    if constexpr (!TR) mma_ss_f16(tO, a, umma_desc_sw128(mb + kk * TT::KSTEP * 128, D * 128, 1024), idQM, kk > 0);
                    else mma_ss_tf32(tO, a, umma_desc_sw128(mb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idQM, kk > 0);
                }
#pragma unroll
                for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                    if constexpr (!TR) {
                        mma_ss_f16(tM, umma_desc_sw128(ka + kk * TT::KSTEP * 128, kBlockBytes, 1024),
                                   umma_desc_sw128(va + kk * TT::KSTEP * 128, kBlockBytes, 1024), idDM, 1u);
                    } else {
                        const uint32_t off = (kk >> 2) * 8192 + (kk & 3) * 32;
                        mma_ss_tf32(tM, umma_desc_sw128(kTa + off, 16, 1024), umma_desc_sw128(vTa + off, 16, 1024), idDM, 1u);
                    }
                }
                mma_commit(&a_free[c % NAB]);
                mbar_wait(p_full, c & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                    if constexpr (!TR)
                        mma_ts_f16(tO, tS + kk * 8, umma_desc_sw128(va + kk * TT::KSTEP * 128, kBlockBytes, 1024), idPV, 1u);
                    else
                        mma_ts_tf32(tO, tS + kk * 8, umma_desc_sw128(vTa + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idPV, 1u);
                }
                mma_commit(mo_full);
                mma_commit(empty);
            }
        }
    } else if (warp >= 4) {
        const int tid = threadIdx.x - 128;  // 0..NM-1
        const int mw = warp - 4;
        const int q = warp & 3, hh = mw >> 2;
        const int row = q * 32 + lane;     // row mapping (S / O / P epilogues)
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int srow = TR ? q * 16 + lane : row;  // state row (d_k index)
        const bool sown = TR ? lane < 16 : true;

        // initial state: M_T <- M_in (fp32), z <- z_in; zero in local mode (lsm_local_fix_vec)
        const bool local = kBF16 && p.local;
        float gtot = 0.f;  // local mode, tid < D: the segment's log decay of column tid
        {
            const float* src = p.Min + (((size_t)bh * p.nseg + seg) * D + (sown ? srow : 0)) * D + hh * DH;
#pragma unroll
            for (int cb = 0; cb < DH / 32; ++cb) {
                uint32_t r[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(sown && !local ? src[cb * 32 + j] : 0.f);
                tmem_st32(tM + lane_off + hh * DH + cb * 32, r);
            }
            tmem_wait_st();
            if constexpr (NORM) {
                if (tid < D) {
                    sZ[tid] = p.zin[((size_t)bh * p.nseg + seg) * D + tid];
                    sZC[tid] = 0.f;
                }
            }
        }
        for (int c = 0; c < nchunks; ++c) {
            const int t0 = t_begin + c * kC;
            const int nvalid = min(kC, t_end - t0);
            uint8_t* at = abuf(c);
            uint8_t* mop = at;
            mbar_wait(&a_full[c % NAB], (c / NAB) & 1);
            if constexpr (HG) mbar_wait(full, c & 1);  // keff = 1 - sigma(a) is written into K
            if (tid == 0) trace_mark(p, c, 0);
            // (1)+(2) 2-D column scan (lsm_vec_scan.cuh), then in place q~ = phi(q) e^{G - r},
            // k~ = keff e^{r - G} (tf32: also the K-major K~^T, V^T tiles)
            // The pairwise factor e^{G_i - G_j} = E_i / E_j with E_t = e^{G_t - r} is a product of
            // per-token sigmas relative to the midpoint (row 63): E_t = prod_{t<u<=63} 1/sigma_u
            // for t < 64, prod_{64<=u<=t} sigma_u for t >= 64 -- two MUFU ops per element (ex2,
            // rcp) and FMA-pipe products, instead of log-space sums and two exponentials.
            {
                const int cg = tid & 15, rg = tid >> 4;
                constexpr int HALF = L::RG / 2;  // row groups below the midpoint
                const bool lower = rg < HALF;
                float sg[L::R][L::EPC], isg[L::R][L::EPC];
                float tot[L::EPC];
#pragma unroll
                for (int j = 0; j < L::EPC; ++j) tot[j] = 1.f;
#pragma unroll
                for (int ii = 0; ii < L::R; ++ii) {
                    const int i = rg * L::R + ii;
                    const bool valid = i < nvalid;
                    float xa[L::EPC], keff[L::EPC];
                    ld_chunk<T>(at, i, cg, xa);
#pragma unroll
                    for (int j = 0; j < L::EPC; ++j) {
                        const float ex = ex2_ftz(-xa[j] * 1.4426950408889634f);  // e^{-a}
                        const float sgm = rcp_ftz(1.f + ex);                       // sigma(a)
                        sg[ii][j] = valid ? sgm : 1.f;
                        isg[ii][j] = valid ? 1.f + ex : 1.f;
                        tot[j] *= sg[ii][j];
                        keff[j] = ex * sgm;                                        // HGRN2: 1 - sigma(a)
                    }
                    if constexpr (HG) st_chunk_raw<T>(kt, i, cg, keff);  // k is unused by HGRN2
                }
#pragma unroll
                for (int j = 0; j < L::EPC; ++j) sOffI[rg * D + cg * L::EPC + j] = tot[j];
                named_bar_sync(1, NM);
                if (tid < D) {
                    // per group, the factor 1/E of the row just past it (Einv offsets):
                    // first half, exclusive suffix of sigma over the later groups below the midpoint
                    float sfx = 1.f;
                    for (int g = HALF - 1; g >= 0; --g) {
                        const float pg = sOffI[g * D + tid];
                        sOffI[g * D + tid] = sfx;
                        sfx *= pg;
                    }
                    sER[tid] = sfx;
                    // second half, 1 / (exclusive prefix of sigma from the midpoint)
                    float pfx = 1.f;
                    for (int g = HALF; g < L::RG; ++g) {
                        const float pg = sOffI[g * D + tid];
                        sOffI[g * D + tid] = rcp_ftz(pfx);
                        pfx *= pg;
                    }
                    sEG[tid] = pfx;
                    // both half products are >= e^{-80} unless the chunk raises the range error
                    if (local) gtot += __logf(sfx) + __logf(pfx);
                }
                named_bar_sync(1, NM);
                if (tid == 0) trace_mark(p, c, 1);
                if constexpr (!HG) mbar_wait(full, c & 1);
                float E[L::EPC], Ei[L::EPC];
#pragma unroll
                for (int j = 0; j < L::EPC; ++j) {
                    Ei[j] = sOffI[rg * D + cg * L::EPC + j];
                    E[j] = rcp_ftz(Ei[j]);
                }
                float zc[L::EPC];
#pragma unroll
                for (int j = 0; j < L::EPC; ++j) zc[j] = 0.f;
                bool bad = false;
                // one row of q~ / k~ with the current factors.  The next row's chunks are loaded
                // before this row's stores (rows walk in order): with load / transform / store per
                // row, every load waited for the previous row's stores (possible aliasing)
                auto ld_row = [&](int ii, uint4& uq, uint4& uk) {
                    const int i = rg * L::R + ii;
                    uq = ld_chunk_raw(qt, i, cg);
                    uk = ld_chunk_raw(kt, i, cg);
                };
                auto xform_row = [&](int ii, const uint4& uq, const uint4& uk, const float (&Ef)[L::EPC],
                                     const float (&Eif)[L::EPC]) {
                    const int i = rg * L::R + ii;
                    const float vm = i < nvalid ? 1.f : 0.f;
                    float xq[L::EPC], xk[L::EPC];
                    unpack_chunk<T>(uq, xq);
                    unpack_chunk<T>(uk, xk);
#pragma unroll
                    for (int j = 0; j < L::EPC; ++j) {
                        const float keff = HG ? xk[j] : fmap_t<FM>(xk[j]);
                        xq[j] = fmap_t<FM>(xq[j]) * (vm * Ef[j]);
                        xk[j] = keff * (vm * Eif[j]);
                        if constexpr (NORM) zc[j] += xk[j];
                    }
                    st_chunk<T>(qt, i, cg, xq);
                    st_chunk<T>(kt, i, cg, xk);
                    if constexpr (TR) {
                        float xv[L::EPC];
                        ld_chunk<T>(vt, i, cg, xv);
#pragma unroll
                        for (int j = 0; j < L::EPC; ++j) {
                            *tr_elem(kT, cg * L::EPC + j, i) = tf32r(xk[j]);
                            *tr_elem(vT, cg * L::EPC + j, i) = tf32r(xv[j]);
                        }
                    }
                };
                // range of the midpoint split (|G - r| < 80, as the log-space check): the extreme
                // factors are the first row (lower half) and the last row (upper half)
                uint4 cq, ck;
                if (lower) {  // warp-uniform: half-warps share a row group pair
                    ld_row(L::R - 1, cq, ck);
#pragma unroll
                    for (int kk = 0; kk < L::R; ++kk) {
                        const int ii = L::R - 1 - kk;  // exclusive suffix: walk upwards
                        uint4 nq = cq, nk = ck;
                        if (kk + 1 < L::R) ld_row(ii - 1, nq, nk);
                        xform_row(ii, cq, ck, E, Ei);
                        cq = nq;
                        ck = nk;
#pragma unroll
                        for (int j = 0; j < L::EPC; ++j) { E[j] *= isg[ii][j]; Ei[j] *= sg[ii][j]; }
                    }
#pragma unroll
                    for (int j = 0; j < L::EPC; ++j) bad |= !(E[j] * sg[0][j] < 5.54e34f);
                } else {
                    ld_row(0, cq, ck);
#pragma unroll
                    for (int ii = 0; ii < L::R; ++ii) {  // inclusive prefix: walk downwards
                        uint4 nq = cq, nk = ck;
                        if (ii + 1 < L::R) ld_row(ii + 1, nq, nk);
#pragma unroll
                        for (int j = 0; j < L::EPC; ++j) { E[j] *= sg[ii][j]; Ei[j] *= isg[ii][j]; }
                        xform_row(ii, cq, ck, E, Ei);
                        cq = nq;
                        ck = nk;
                    }
#pragma unroll
                    for (int j = 0; j < L::EPC; ++j) bad |= !(E[j] > 1.81e-35f);
                }
                if constexpr (NORM) {
#pragma unroll
                    for (int j = 0; j < L::EPC; ++j) atomicAdd(&sZC[cg * L::EPC + j], zc[j]);
                }
                if (bad) atomicOr(&p.err[2], 1);
            }
            if (tid == 0) bulk_wait_read0();  // the previous chunk's O store has left the staging tile
            named_bar_sync(1, NM);
            if (tid == 0) trace_mark(p, c, 2);
            // (3) state operand M' = diag(e^r) M  (and the TMEM copy), z' = e^r z
            {
                const float er = sER[srow < D ? srow : 0];
                float vals[DH];
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    uint32_t rr[32];
                    tmem_ld32(tM + lane_off + hh * DH + cb * 32, rr);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        vals[cb * 32 + j] = __uint_as_float(rr[j]) * er;
                        rr[j] = __float_as_uint(vals[cb * 32 + j]);
                    }
                    tmem_st32(tM + lane_off + hh * DH + cb * 32, rr);
                }
                if (sown) {
                    if constexpr (!TR) {
                        // columns [32 hh, 32 hh + 32): block hh / 2, 16-byte chunks 4 (hh % 2) ..
                        uint8_t* dst = mop + (hh >> 1) * (D * 128);
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            uint4 v;
                            v.x = pack_bf16(vals[ch * 8 + 0], vals[ch * 8 + 1]);
                            v.y = pack_bf16(vals[ch * 8 + 2], vals[ch * 8 + 3]);
                            v.z = pack_bf16(vals[ch * 8 + 4], vals[ch * 8 + 5]);
                            v.w = pack_bf16(vals[ch * 8 + 6], vals[ch * 8 + 7]);
                            *reinterpret_cast<uint4*>(dst + sw128_off(srow, (hh & 1) * 4 + ch)) = v;
                        }
                    } else {
                        uint8_t* base = mop + (srow >> 5) * 8192 + ((srow & 3) << 2);
                        const int cch = (srow & 31) >> 2;
#pragma unroll
                        for (int j = 0; j < DH; ++j)
                            *reinterpret_cast<float*>(base + sw128_off(hh * DH + j, cch)) = tf32r(vals[j]);
                    }
                }
                if constexpr (NORM) {
                    if (tid < D) sZP[tid] = sER[tid] * sZ[tid];
                }
                tmem_wait_st();
                fence_proxy_async_smem();
                tc_fence_before();
                if constexpr (NORM) named_bar_sync(1, NM);
                mbar_arrive(xf);
            }
            if (tid == 0) trace_mark(p, c, 3);
            // (4) P = S . mask  (+ row sums, q~ . z' for the normaliser)
            mbar_wait(s_full, c & 1);
            if (tid == 0) trace_mark(p, c, 4);
            tc_fence_after();
            {
                // this thread's 128 / NQ columns of the S row (bf16: 32, tf32: 64)
                constexpr int SC = 128 / NQ;
                uint32_t r0[32], r1[32];
                tmem_ld32(tS + lane_off + hh * SC, r0);
                if constexpr (SC == 64) tmem_ld32(tS + lane_off + hh * SC + 32, r1);
                tmem_wait_ld();
                float rs = 0.f;
#pragma unroll
                for (int j = 0; j < SC; ++j) {
                    const int cc = hh * SC + j;
                    float v = __uint_as_float(j < 32 ? r0[j] : r1[j - 32]);
                    v = (cc <= row) ? v : 0.f;
                    if constexpr (TR) v = tf32r(v);
                    rs += v;
                    if (j < 32) r0[j] = __float_as_uint(v); else r1[j - 32] = __float_as_uint(v);
                }
                float qz = 0.f;
                if constexpr (NORM) {
#pragma unroll 8
                    for (int j = 0; j < DH; ++j) qz += ld_elem<T>(qt, row, hh * DH + j) * sZP[hh * DH + j];
                }
                const uint32_t tpart = kBF16 ? tS + lane_off + 64 : tmem + 384 + lane_off;
                if constexpr (kBF16) {
                    uint32_t pk[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
                    named_bar_sync(1, NM);
                    tmem_st16(tS + lane_off + hh * 16, pk);
                } else {
                    tmem_st32(tS + lane_off + hh * 64, r0);
                    tmem_st32(tS + lane_off + hh * 64 + 32, r1);
                }
                if constexpr (NORM) {
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tpart + hh),
                                 "r"(__float_as_uint(rs)) : "memory");
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tpart + NQ + hh),
                                 "r"(__float_as_uint(qz)) : "memory");
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(p_full);
            }
            if (tid == 0) trace_mark(p, c, 5);
            // (5) state: M_next = diag(e^{G_end - r}) M'
            mbar_wait(mo_full, c & 1);
            if (tid == 0) trace_mark(p, c, 6);
            tc_fence_after();
            {
                const int kr = srow < D ? srow : 0;
                const float f = sEG[kr];
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    uint32_t rr[32];
                    tmem_ld32(tM + lane_off + hh * DH + cb * 32, rr);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) rr[j] = __float_as_uint(__uint_as_float(rr[j]) * f);
                    tmem_st32(tM + lane_off + hh * DH + cb * 32, rr);
                }
                tmem_wait_st();
                if constexpr (NORM) {
                    if (tid < D) {
                        sZ[tid] = sEG[tid] * (sZP[tid] + sZC[tid]);
                        sZC[tid] = 0.f;
                    }
                }
            }
            // (6) O epilogue -> global
            {
                float inv = 1.f;
                if constexpr (NORM) {
                    const uint32_t tpart = kBF16 ? tS + lane_off + 64 : tmem + 384 + lane_off;
                    uint32_t pr[8];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(pr[0]), "=r"(pr[1]), "=r"(pr[2]), "=r"(pr[3]), "=r"(pr[4]), "=r"(pr[5]),
                                   "=r"(pr[6]), "=r"(pr[7]) : "r"(tpart));
                    tmem_wait_ld();
                    float den = 0.f;
#pragma unroll
                    for (int i = 0; i < 2 * NQ; ++i) den += __uint_as_float(pr[i]);
                    if (fabsf(den) < 1e-12f && row < nvalid) atomicOr(&p.err[0], 1);
                    inv = 1.f / den;
                }
                // bf16: stage O (this thread's 32 columns of its row); one TMA bulk tensor store
                // per chunk (rows past the sequence end are clipped).  tf32 (no smem left for a
                // staging tile): direct row stores.
                if constexpr (!kBF16) {
                    uint32_t rr[32];
                    tmem_ld32(tO + lane_off + hh * DH, rr);
                    tmem_wait_ld();
                    if (row < nvalid) {
                        T* dst = reinterpret_cast<T*>(p.o) + (((size_t)b * p.Nstride + t0 + row) * p.H + h) * D + hh * DH;
#pragma unroll
                        for (int ch = 0; ch < 8; ++ch)
                            *reinterpret_cast<float4*>(dst + ch * 4) =
                                make_float4(__uint_as_float(rr[ch * 4]) * inv, __uint_as_float(rr[ch * 4 + 1]) * inv,
                                            __uint_as_float(rr[ch * 4 + 2]) * inv, __uint_as_float(rr[ch * 4 + 3]) * inv);
                    }
                } else {
                    uint32_t rr[32];
                    tmem_ld32(tO + lane_off + hh * DH, rr);
                    tmem_wait_ld();
                    constexpr int CPT = DH / TT::EPC;  // 16-byte chunks per thread
#pragma unroll
                    for (int ch = 0; ch < CPT; ++ch) {
                        uint4 v;
                        if constexpr (kBF16) {
                            v.x = pack_bf16(__uint_as_float(rr[ch * 8 + 0]) * inv, __uint_as_float(rr[ch * 8 + 1]) * inv);
                            v.y = pack_bf16(__uint_as_float(rr[ch * 8 + 2]) * inv, __uint_as_float(rr[ch * 8 + 3]) * inv);
                            v.z = pack_bf16(__uint_as_float(rr[ch * 8 + 4]) * inv, __uint_as_float(rr[ch * 8 + 5]) * inv);
                            v.w = pack_bf16(__uint_as_float(rr[ch * 8 + 6]) * inv, __uint_as_float(rr[ch * 8 + 7]) * inv);
                        } else {
                            v = make_uint4(__float_as_uint(__uint_as_float(rr[ch * 4]) * inv),
                                           __float_as_uint(__uint_as_float(rr[ch * 4 + 1]) * inv),
                                           __float_as_uint(__uint_as_float(rr[ch * 4 + 2]) * inv),
                                           __float_as_uint(__uint_as_float(rr[ch * 4 + 3]) * inv));
                        }
                        const int cgi = hh * CPT + ch;
                        *reinterpret_cast<uint4*>(ostg + (cgi >> 3) * kBlockBytes + sw128_off(row, cgi & 7)) = v;
                    }
                }
                tc_fence_before();
                fence_proxy_async_smem();
            }
            if (tid == 0) trace_mark(p, c, 7);
            named_bar_sync(1, NM);  // everyone done with this chunk's tiles and sZ; O staged
            if (kBF16 && tid == 0) {
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) tma_store_4d(&tmO, ostg + blk * kBlockBytes, blk * TT::EPB, h, t0, b);
                bulk_commit();
            }
            if (tid == 0) trace_mark(p, c, 8);
        }
        if constexpr (kBF16) {
            if (local) {  // the segment's state from zero and its per-column log decay (combine inputs)
                float* dst = p.Sseg + (((size_t)bh * p.nseg + seg) * D + srow) * D + hh * DH;
                uint32_t r[32];
                tmem_ld32(tM + lane_off + hh * DH, r);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                                      __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                if (tid < D) p.logDseg[((size_t)bh * p.nseg + seg) * D + tid] = gtot;
            }
        }
    }
    if (threadIdx.x == 128) bulk_wait_read0();  // smem must outlive the last O store's read of it
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// ====================================================================================
// Local-state correction, TokenVector decays (bf16, identity feature map; the vector
// counterpart of lsm_local_fix, lsm_kernels.cuh).  The output pass ran every segment from a
// zero state; with M_in(s) from the segment combine
//     o_t = o_t^local + (q_t . E_t) M_in(s),   E_t[k] = prod_{u in seg, u <= t} sigmoid(a_u[k])
// E_t only decreases along the segment, so the correction stops after the first chunk that
// leaves every column below e^{-88}.  With a ~ N(0, 1) gates a column decays by ~e^{-0.8} per
// token: one or two chunks per segment.  Thread (column d = tid % 128, row half tid / 128)
// scans E down its column in linear space (sigmoid products; an underflow to zero is the
// exact value's fp32 image) -- pass 1 the half's product, pass 2 the prefix and q~ = q E.
// ====================================================================================
constexpr int kFixVecThreads = 256;
constexpr int fix_vec_smem() { return 4 * kTileBytes + 3 * 128 * 4 + 64; }

template <int D>  // 128 (a template: this header is included by several translation units)
__global__ void __launch_bounds__(kFixVecThreads, 1)
    lsm_local_fix_vec(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmO, LsmFwdParams p) {
    using T = __nv_bfloat16;
    using TT = TileTraits<T>;
    static_assert(D == TT::D, "bf16 tiles are 128 columns");
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* qt = smem;                    // Q~ tile
    uint8_t* at = smem + kTileBytes;       // gate tile
    uint8_t* ot = smem + 2 * kTileBytes;   // O tile (read, updated, stored)
    uint8_t* mop = smem + 3 * kTileBytes;  // bf16 M_in operand
    float* sP = reinterpret_cast<float*>(smem + 4 * kTileBytes);  // [D] E at the chunk start
    float* sH = sP + D;                                           // [2][D] half products
    uint64_t* bars = reinterpret_cast<uint64_t*>(sH + 2 * D);
    uint64_t* full = bars;
    uint64_t* mma_done = bars + 1;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 2);

    const int seg = p.nseg - (int)gridDim.x + blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id(), tid = threadIdx.x;
    const int d = tid & 127, hf = tid >> 7;
    if (tid == 0) {
        mbar_init(full, 1);
        mbar_init(mma_done, 1);
        fence_barrier_init();
    }
    if (tid < D) sP[tid] = 1.f;
    if (warp == 0) tmem_alloc<128>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    pdl_wait();
    pdl_trigger();
    {  // M_in(seg) -> bf16 operand: thread (row, column half)
        const int row = tid & 127, half = tid >> 7;
        const float* src = p.Min + (((size_t)bh * p.nseg + seg) * D + row) * D + half * 64;
        uint8_t* dst = mop + half * (D * 128);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
            const float4 a = *reinterpret_cast<const float4*>(src + ch * 8);
            const float4 c = *reinterpret_cast<const float4*>(src + ch * 8 + 4);
            uint4 v;
            v.x = pack_bf16(a.x, a.y); v.y = pack_bf16(a.z, a.w);
            v.z = pack_bf16(c.x, c.y); v.w = pack_bf16(c.z, c.w);
            *reinterpret_cast<uint4*>(dst + sw128_off(row, ch)) = v;
        }
    }
    const int q4 = warp & 3, half = warp >> 2;  // TMEM lane quarter, column half
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    bool alive = true;
    for (int c = 0; c < nchunks; ++c) {
        // the previous chunk's E update and O store read; stop once every column is below e^{-88}
        if (!__syncthreads_or(alive)) break;
        const int t0 = t_begin + c * kC;
        const int nvalid = min(kC, t_end - t0);
        if (tid == 0) {
            bulk_wait_read0();
            mbar_expect_tx(full, 6 * kBlockBytes);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                tma_load_4d(qt + blk * kBlockBytes, &tmQ, full, blk * TT::EPB, h, t0, b);
                tma_load_4d(at + blk * kBlockBytes, &tmA, full, blk * TT::EPB, h, t0, b);
                tma_load_4d(ot + blk * kBlockBytes, &tmO, full, blk * TT::EPB, h, t0, b);
            }
        }
        mbar_wait(full, c & 1);
        const int r0 = hf * 64, r1 = min(r0 + 64, nvalid);
        auto sig = [&](int r) {
            const float ex = ex2_ftz(-ld_elem<T>(at, r, d) * 1.4426950408889634f);
            return rcp_ftz(1.f + ex);
        };
        {  // pass 1: this half's product
            float pr = 1.f;
            for (int r = r0; r < r1; ++r) pr *= sig(r);
            sH[hf * D + d] = pr;
        }
        __syncthreads();
        {  // pass 2: inclusive prefix, q~ = q E (rows past the sequence end: 0)
            float e = sP[d] * (hf ? sH[d] : 1.f);
            for (int r = r0; r < r0 + 64; ++r) {
                float x = 0.f;
                if (r < r1) {
                    e *= sig(r);
                    x = ld_elem<T>(qt, r, d) * e;
                }
                st_elem<T>(qt, r, d, x);
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            constexpr uint32_t idQM = umma_idesc(1, 0, 1, 128, D);
            const uint32_t qa = smem_u32(qt), mb = smem_u32(mop);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                mma_ss_f16(tmem, umma_desc_sw128(qa + off, 16, 1024), umma_desc_sw128(mb + kk * 16 * 128, D * 128, 1024),
                           idQM, kk > 0 ? 1u : 0u);
            }
            mma_commit(mma_done);
        }
        if (tid < D) {
            const float e = sP[d] * sH[d] * sH[D + d];
            sP[d] = e;
            alive = e > 6.05e-39f;  // e^{-88}
        } else {
            alive = false;
        }
        mbar_wait(mma_done, c & 1);
        tc_fence_after();
        {  // O += Q~ M_in for this thread's row and 64 columns, in the O tile, then one bulk store
            uint32_t r[64];
            tmem_ld32(tmem + lane_off + half * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
            tmem_ld32(tmem + lane_off + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            tmem_wait_ld();
            uint8_t* ob = ot + half * kBlockBytes;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                uint4* ptr = reinterpret_cast<uint4*>(ob + sw128_off(row, ch));
                uint4 v = *ptr;
                uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = unpack_bf16(w[e]);
                    w[e] = pack_bf16(f.x + __uint_as_float(r[ch * 8 + 2 * e]), f.y + __uint_as_float(r[ch * 8 + 2 * e + 1]));
                }
                *ptr = v;
            }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tma_store_4d(&tmO, ot, 0, h, t0, b);
            tma_store_4d(&tmO, ot + kBlockBytes, TT::EPB, h, t0, b);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait0();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
}

template <typename T>
constexpr int output_pass_vec_smem() {
    using TT = TileTraits<T>;
    // + group offsets 2 x [RG][D], sER, sEG, sZ, sZP, sZC + 6 barriers + TMEM slot
    // Q | K | V | NAB gate / M' buffers (| tf32 K~^T, V^T) (| bf16 O staging) + group factors
    // [RG][D] + sER, sEG, sZ, sZP, sZC + 10 barriers + TMEM slot
    return (sizeof(T) == 2 ? 6 : 4) * kTileBytes + (TT::kTransposed ? 2 * kTileBytes : 0) +
           ((vec_math_threads<T>() / 16) + 5) * TT::D * 4 + 128;
}
template <typename T>
constexpr int state_pass_vec_smem() {
    using TT = TileTraits<T>;
    // + sTot [16][D], sR, sGe, sG0, sCar, sZ, barriers
    return (TT::kTransposed ? 1 : 2) * 3 * kTileBytes + (TT::kTransposed ? 2 * kTileBytes : 0) +
           (16 + 5) * TT::D * 4 + 128;
}

}  // namespace lmoe_dev
