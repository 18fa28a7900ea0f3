// lsm_kernels.cuh -- device code of the chunkwise LSM forward (v3), see lsm_fwd.cuh.
// Included by the per-dtype instantiation units lsm_inst_{bf16,f32}.cu.
#pragma once
#include "lsm_fwd.cuh"

namespace lmoe_dev {

// Round-to-nearest fp32 -> tf32 (the tensor core would truncate the low mantissa bits).
__device__ __forceinline__ float tf32r(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Gate pre-activations of one chunk (lane l owns tokens 4l..4l+3); issued two chunks ahead
// of their use so the dependent global-load latency is hidden.
template <int DECAY>
__device__ __forceinline__ void load_gates(const LsmFwdParams& p, int b, int h, int t0, int nvalid,
                                           int lane, float (&bv)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int t = lane * 4 + u;
        bv[u] = (DECAY == kDecayTokenScalar && t < nvalid)
                    ? __ldg(p.b_pre + ((size_t)b * p.Nstride + t0 + t) * p.H + h)
                    : 0.f;
    }
}

// Per-token log decay la and keff factor kf (lsm.hpp:483-518) of lane-owned tokens, then
// the inclusive chunk-local scan: returns G_end, leaves G_t in la.
template <int DECAY>
__device__ __forceinline__ float chunk_scan(const LsmFwdParams& p, const float (&bv)[4], int nvalid,
                                            float spa, int lane, float (&la)[4], float (&kf)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const bool valid = lane * 4 + u < nvalid;
        la[u] = 0.f;
        kf[u] = valid ? 1.f : 0.f;
        if constexpr (DECAY == kDecayConst) la[u] = valid ? p.log_a : 0.f;
        if constexpr (DECAY == kDecayTokenScalar) {
            const float spb = softplus_f(bv[u]);
            la[u] = valid ? -spb * spa : 0.f;
            kf[u] = valid ? spb : 0.f;
        }
    }
    float own[4];
    float run = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) { own[u] = la[u]; run += la[u]; la[u] = run; }
    float x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    const float excl = x - run;
#pragma unroll
    for (int u = 0; u < 4; ++u) la[u] += excl;
    if (p.fault) {  // TEST ONLY: the reference's off-by-one hook (lsm.hpp:566-572), p_t = prod_{s<t}
#pragma unroll
        for (int u = 0; u < 4; ++u) la[u] -= own[u];
    }
    return __shfl_sync(0xFFFFFFFFu, x, 31);
}

// One 16-byte chunk (8 bf16 / 4 fp32 values) in registers: x <- round(phi(x) * scale).
template <typename T, int FM, bool RND>
__device__ __forceinline__ void xform_chunk(uint4& v, float scale) {
    if constexpr (sizeof(T) == 2) {
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f = unpack_bf16(w[i]);
            w[i] = pack_bf16(fmap_t<FM>(f.x) * scale, fmap_t<FM>(f.y) * scale);
        }
    } else {
        float* f = reinterpret_cast<float*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float x = fmap_t<FM>(f[i]) * scale;
            f[i] = RND ? tf32r(x) : x;
        }
    }
}

// Row-owner transform of NCH 16-byte chunks (starting at chunk ch0) of one SW128 row, in
// place.  All shared loads issue before the first store: with load / transform / store per
// chunk the compiler cannot prove the swizzled addresses distinct, so every load waited for
// the previous chunk's store (8 exposed shared-memory round trips per row).
template <typename T, int FM, bool RND, int NCH>
__device__ __forceinline__ void xform_chunks(uint8_t* blk, int row, int ch0, float scale) {
    uint4 v[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) v[ch] = *reinterpret_cast<const uint4*>(blk + sw128_off(row, ch0 + ch));
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) xform_chunk<T, FM, RND>(v[ch], scale);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) *reinterpret_cast<uint4*>(blk + sw128_off(row, ch0 + ch)) = v[ch];
}

// Row-owner transform of one 128-byte half row (8 x 16B chunks) in place:
// x <- round(phi(x) * scale); rows beyond the sequence get scale 0.
template <typename T, int FM, bool RND>
__device__ __forceinline__ void xform_half_row(uint8_t* blk, int row, float scale) {
    xform_chunks<T, FM, RND, 8>(blk, row, 0, scale);
}

// Row-owner transform of NCOLS columns starting at col0 of a two-block SW128 tile (the
// range stays inside one 128-byte block).
template <typename T, int FM, bool RND, int NCOLS>
__device__ __forceinline__ void xform_row_part(uint8_t* tile, int row, int col0, float scale) {
    using TT = TileTraits<T>;
    static_assert(NCOLS % TT::EPC == 0 && NCOLS <= TT::EPB, "one block, whole chunks");
    xform_chunks<T, FM, RND, NCOLS / TT::EPC>(tile + (col0 / TT::EPB) * kBlockBytes, row,
                                             (col0 % TT::EPB) / TT::EPC, scale);
}

// fp32 only: write one token row's 32 values of column block `hb` (already scaled) into a
// transposed K-major tile [64 d rows x 128 tok] (4 SW128 blocks of 32 tokens, 8 KB apart).
__device__ __forceinline__ void store_transposed_f32(uint8_t* dstT, int tok, int hb,
                                                     const float (&vals)[32]) {
    uint8_t* base = dstT + (tok >> 5) * 8192 + ((tok & 3) << 2);
    const int cchunk = (tok & 31) >> 2;
#pragma unroll
    for (int c = 0; c < 32; ++c)
        *reinterpret_cast<float*>(base + sw128_off(hb * 32 + c, cchunk)) = tf32r(vals[c]);
}
__device__ __forceinline__ void load_half_row_f32(const uint8_t* blk, int row, float (&vals)[32]) {
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
        const float4 v = *reinterpret_cast<const float4*>(blk + sw128_off(row, ch));
        vals[ch * 4] = v.x; vals[ch * 4 + 1] = v.y; vals[ch * 4 + 2] = v.z; vals[ch * 4 + 3] = v.w;
    }
}

// ====================================================================================
// Phase 1: per-segment state S_seg = sum_j exp(L_j) keff_j v_j^T accumulated in TMEM.
// warps: 0 TMA, 1 MMA, 2 decay, 3 idle, 4..7 transform (row owners, 128 threads)
// ====================================================================================
template <typename T, int DECAY, int FM, bool NORM, bool REV>
__global__ void __launch_bounds__(kStatePassThreads, 1)
    lsm_state_pass(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   LsmFwdParams p) {
    using TT = TileTraits<T>;
    constexpr int D = TT::D;
    constexpr int NST = TT::SP_STAGES;
    constexpr bool TR = TT::kTransposed;
    constexpr bool kXform = TR || DECAY != kDecayNone || FM != 0 || NORM;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* tiles = smem;                                   // NST x [K | V]
    uint8_t* kT = tiles + NST * 2 * kTileBytes;              // fp32 transposed tiles
    uint8_t* vT = kT + (TR ? kTileBytes : 0);
    float* ringW = reinterpret_cast<float*>(vT + (TR ? kTileBytes : 0));  // [2][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(ringW + 256);
    uint64_t* full = bars;              // [NST]
    uint64_t* empty = bars + NST;       // [NST]
    uint64_t* wfull = bars + 2 * NST;   // [2]
    uint64_t* wfree = wfull + 2;        // [2]
    // K~ transformed, one barrier per stage: the four math warps are not synchronised with
    // each other per chunk, so a fast warp may transform chunk it+1 (its stage is already
    // loaded) before a slow one finishes chunk it; with a single barrier its arrival would
    // complete chunk it's phase early (the race measured in lsm_fused.cuh).  A warp reaches
    // chunk it+NST only after the MMA consumed chunk it (its stage was reloaded).
    uint64_t* xf = wfree + 2;           // [NST]
    uint64_t* acc_full = xf + NST;
    uint64_t* kt_free = acc_full + 1;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(kt_free + 1);

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&wfull[i], 32); mbar_init(&wfree[i], 128); }
        for (int i = 0; i < NST; ++i) mbar_init(&xf[i], 128);
        mbar_init(acc_full, 1);
        mbar_init(kt_free, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<128>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    trace_cta(p, 0, 1);
    pdl_wait();  // predecessor's outputs (segment states / prefixes) are visible from here
    pdl_trigger();
    trace_cta(p, 1, 2);
    // forward: last chunk first (weights e^{G_end - G_j} need no pre-pass); REV: first first
    auto chunk_t0 = [&](int it) { return t_begin + (REV ? it : nchunks - 1 - it) * kC; };

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % NST;
                if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
                const int t0 = chunk_t0(it);
                uint8_t* kt = tiles + s * 2 * kTileBytes;
                uint8_t* vt = kt + kTileBytes;
                mbar_expect_tx(&full[s], 2 * kTileBytes);
                tma_load_4d(kt, &tmK, &full[s], 0, h, t0, b);
                tma_load_4d(kt + kBlockBytes, &tmK, &full[s], TT::EPB, h, t0, b);
                tma_load_4d(vt, &tmV, &full[s], 0, h, t0, b);
                tma_load_4d(vt + kBlockBytes, &tmV, &full[s], TT::EPB, h, t0, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % NST;
                mbar_wait(&full[s], (it / NST) & 1);
                mbar_wait(&xf[s], (it / NST) & 1);
                tc_fence_after();
                const uint32_t kt = smem_u32(tiles + s * 2 * kTileBytes);
                const uint32_t vt = kt + kTileBytes;
                if constexpr (!TR) {
                    constexpr uint32_t idesc = umma_idesc(TT::FMT, 1, 1, 128, D);
#pragma unroll
                    for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                        const uint64_t a = umma_desc_sw128(kt + kk * TT::KSTEP * 128, kBlockBytes, 1024);
                        const uint64_t bd = umma_desc_sw128(vt + kk * TT::KSTEP * 128, kBlockBytes, 1024);
                        mma_ss_f16(tmem, a, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
                    }
                } else {
                    constexpr uint32_t idesc = umma_idesc(TT::FMT, 0, 0, 64, D);
                    const uint32_t ka = smem_u32(kT), va = smem_u32(vT);
#pragma unroll
                    for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                        const uint32_t off = (kk >> 2) * 8192 + (kk & 3) * 32;
                        mma_ss_tf32(tmem, umma_desc_sw128(ka + off, 16, 1024),
                                    umma_desc_sw128(va + off, 16, 1024), idesc,
                                    (it > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(kt_free);
                }
                mma_commit(&empty[s]);
            }
            mma_commit(acc_full);
        }
    } else if (warp == 2) {
        // decay warp: per-token weights w_t = exp(L_t) kf_t, L_t = log decay from token t
        // (exclusive) to the segment end = (G_end - G_t) + decay of the later chunks.
        // REV: w_t = exp(G_t + decay of the earlier chunks) (from the segment start), no kf.
        const float spa = (DECAY == kDecayTokenScalar) ? softplus_f(p.a_raw[h]) : 0.f;
        float suffix = 0.f;
        float bvA[4], bvB[4], bvC[4];
        auto nval = [&](int it) { return min(kC, t_end - chunk_t0(it)); };
        load_gates<DECAY>(p, b, h, chunk_t0(0), nval(0), lane, bvA);
        if (nchunks > 1) load_gates<DECAY>(p, b, h, chunk_t0(1), nval(1), lane, bvB);
        for (int it = 0; it < nchunks; ++it) {
            const int slot = it & 1;
            if (it + 2 < nchunks) load_gates<DECAY>(p, b, h, chunk_t0(it + 2), nval(it + 2), lane, bvC);
            // the math warps release a ring slot only when they read it (kXform); without the
            // transform nothing reads the ring, and waiting here deadlocked every decay-free bf16
            // segment of three or more chunks
            if (kXform && it >= 2) mbar_wait(&wfree[slot], ((it >> 1) - 1) & 1);
            float la[4], kf[4];
            const float gend = chunk_scan<DECAY>(p, bvA, nval(it), spa, lane, la, kf);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                ringW[slot * 128 + lane * 4 + u] =
                    REV ? __expf(la[u] + suffix) : __expf(gend - la[u] + suffix) * kf[u];
            suffix += gend;
            __syncwarp();
            mbar_arrive(&wfull[slot]);
#pragma unroll
            for (int u = 0; u < 4; ++u) { bvA[u] = bvB[u]; bvB[u] = bvC[u]; }
        }
        if (lane == 0) p.logDseg[(size_t)bh * p.nseg + seg] = suffix;
    } else if (warp >= 4) {
        const int tid = threadIdx.x - 128;  // 0..127 == token row of the chunk
        const int q = warp & 3;
        float zacc = 0.f;                   // normaliser colsum, column tid
        for (int it = 0; it < nchunks; ++it) {
            const int s = it % NST, slot = it & 1;
            uint8_t* kt = tiles + s * 2 * kTileBytes;
            uint8_t* vt = kt + kTileBytes;
            if constexpr (kXform) {
                mbar_wait(&wfull[slot], (it >> 1) & 1);
                const float w = ringW[slot * 128 + tid];
                mbar_wait(&full[s], (it / NST) & 1);
                if constexpr (!TR) {
                    xform_half_row<T, FM, false>(kt, tid, w);
                    xform_half_row<T, FM, false>(kt + kBlockBytes, tid, w);
                } else {
                    if (it >= 1) mbar_wait(kt_free, (it - 1) & 1);
#pragma unroll
                    for (int hb = 0; hb < 2; ++hb) {
                        float vals[32];
                        load_half_row_f32(kt + hb * kBlockBytes, tid, vals);
#pragma unroll
                        for (int c = 0; c < 32; ++c) vals[c] = fmap_t<FM>(vals[c]) * w;
                        store_transposed_f32(kT, tid, hb, vals);
                        load_half_row_f32(vt + hb * kBlockBytes, tid, vals);
                        store_transposed_f32(vT, tid, hb, vals);
                    }
                }
                fence_proxy_async_smem();
                mbar_arrive(&wfree[slot]);
                if constexpr (NORM) {
                    named_bar_sync(1, 128);
                    if (tid < D) {
                        float acc = 0.f;
                        if constexpr (!TR) {
                            const int blk = tid / TT::EPB, cin = tid % TT::EPB;
                            const uint8_t* base = kt + blk * kBlockBytes;
                            for (int r = 0; r < kC; ++r)
                                acc += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                                    base + sw128_off(r, cin / TT::EPC) + (cin % TT::EPC) * 2));
                        } else {
#pragma unroll 4
                            for (int blk = 0; blk < 4; ++blk)
                                for (int ch = 0; ch < 8; ++ch) {
                                    const float4 v = *reinterpret_cast<const float4*>(kT + blk * 8192 + sw128_off(tid, ch));
                                    acc += v.x + v.y + v.z + v.w;
                                }
                        }
                        zacc += acc;
                    }
                    named_bar_sync(1, 128);  // colsum reads done before the next transform
                }
            }
            mbar_arrive(&xf[s]);
        }
        // epilogue: S (d_k rows x d_v cols) from TMEM to global
        mbar_wait(acc_full, 0);
        tc_fence_after();
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
        if constexpr (NORM) {
            if (tid < D) p.zseg[((size_t)bh * p.nseg + seg) * D + tid] = zacc;
        }
    }
    tc_fence_before();
    __syncthreads();
    trace_cta(p, 1, 1);
    if (warp == 1) tmem_dealloc<128>(tmem);
}

// ====================================================================================
// Phase 3: output pass.
// warps: 0 TMA producer, 1 MMA, 2 decay factors, 3 idle, 4..11 math (256 threads)
// Per chunk c the MMA issues QM(c) and dM(c) as soon as the transforms land, then PV(c)
// once P is in TMEM, then S(c+1); the math warps overlap the P epilogue with QM/dM and
// store O straight from registers, so a stage is recycled as soon as its MMAs complete.
// TMEM (bf16): S0 [0,128) S1 [128,256) O [256,384) M [384,512); row partials in the
//              current S buffer's columns 64..67 once P (packed bf16) occupies 0..63.
//      (tf32): S0, S1, O [256,320), M [320,384) (M=64 layout), partials [384,388).
// ====================================================================================
template <typename T, int DECAY, int FM, bool NORM, bool REV>
__global__ void __launch_bounds__(output_pass_threads<T>(), 1)
    lsm_output_pass(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    LsmFwdParams p) {
    using TT = TileTraits<T>;
    constexpr int D = TT::D;
    constexpr bool kBF16 = sizeof(T) == 2;
    constexpr int NST = TT::OUT_STAGES;
    constexpr bool TR = TT::kTransposed;
    constexpr bool kPrep = FM != 0 || TR;  // phi and/or tf32 rounding before S
    constexpr int NQ = TT::NQ;             // column groups per row (math warpgroups)
    constexpr int MT = 128 * NQ;           // math threads
    constexpr int DH = D / NQ;             // d_v columns per math thread (O, M)
    constexpr int KC = 128 / NQ;           // key columns per math thread (S, P)
    static_assert(!TR || NQ == 2, "the tf32 transposed path is written for two column halves");
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* tiles = smem;                                 // NST x [Q | K | V]
    uint8_t* kT = tiles + NST * 3 * kTileBytes;            // fp32: K~^T, V^T tiles
    uint8_t* vT = kT + (TR ? kTileBytes : 0);
    uint8_t* mop = vT + (TR ? kTileBytes : 0);             // state MMA operand
    float* ringG = reinterpret_cast<float*>(mop + TT::MOP_BYTES);  // [2][128]
    float* ringF = ringG + 256;                                     // [2][128]
    float* ringS = ringF + 256;                                     // [2][8]
    float* sZ = ringS + 16;                                         // [128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sZ + 128);
    uint64_t* full = bars;         // [2]
    uint64_t* empty = bars + 2;    // [2]
    uint64_t* s_full = bars + 4;   // [2]
    uint64_t* p_full = bars + 6;
    uint64_t* xf2 = bars + 7;
    uint64_t* m_ready = bars + 8;
    uint64_t* mo_full = bars + 9;
    uint64_t* gfull = bars + 10;   // [2]
    uint64_t* gfree = bars + 12;   // [2]
    uint64_t* xf1 = bars + 14;
    uint64_t* o_staged = bars + 15;  // bf16 O of the chunk staged in its Q tile (store warp)
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 16);

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id();
    // processing order: first-to-last, or last-to-first for the reverse-time (REV) passes
    auto chunk_t0 = [&](int c) { return t_begin + (REV ? nchunks - 1 - c : c) * kC; };

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 2);  // MMA commit + the O epilogue (it stages O in the Q tile)
            mbar_init(&s_full[i], 1);
            mbar_init(&gfull[i], 32);
            mbar_init(&gfree[i], MT);
        }
        mbar_init(p_full, MT);
        mbar_init(xf2, MT);
        mbar_init(m_ready, MT);
        mbar_init(mo_full, 1);
        mbar_init(xf1, MT);
        mbar_init(o_staged, MT);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    trace_cta(p, 0);
    pdl_wait();  // predecessor's outputs (segment states / prefixes) are visible from here
    pdl_trigger();
    trace_cta(p, 0, 2);
    const uint32_t tO = tmem + 256;
    const uint32_t tM = tmem + (kBF16 ? 384 : 320);

    if (warp == 0) {
        // ---------------- producer ---------------------------------------------------------
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % NST;
                if (c >= NST) mbar_wait(&empty[s], ((c / NST) - 1) & 1);
                const int t0 = chunk_t0(c);
                uint8_t* st = tiles + s * 3 * kTileBytes;
                mbar_expect_tx(&full[s], 3 * kTileBytes);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    tma_load_4d(st + blk * kBlockBytes, &tmQ, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + kTileBytes + blk * kBlockBytes, &tmK, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + 2 * kTileBytes + blk * kBlockBytes, &tmV, &full[s], blk * TT::EPB, h, t0, b);
                }
                trace_mark(p, c, 10);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ------------------------------------------------------
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc(TT::FMT, 0, 0, 128, 128);
            constexpr uint32_t idPV = umma_idesc(TT::FMT, 0, TR ? 0 : 1, 128, D);
            constexpr uint32_t idQM = umma_idesc(TT::FMT, 0, TR ? 0 : 1, 128, D);
            constexpr uint32_t idDM = TR ? umma_idesc(TT::FMT, 0, 0, 64, D) : umma_idesc(TT::FMT, 1, 1, 128, D);
            const uint32_t mb = smem_u32(mop), ka = smem_u32(kT), va = smem_u32(vT);
            auto issue_S = [&](int c) {
                const int s = c % NST, bb = c & 1;
                mbar_wait(&full[s], (c / NST) & 1);
                if constexpr (kPrep) mbar_wait(xf1, c & 1);
                tc_fence_after();
                const uint32_t qt = smem_u32(tiles + s * 3 * kTileBytes), kt = qt + kTileBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    const uint64_t a = umma_desc_sw128(qt + off, 16, 1024);
                    const uint64_t bd = umma_desc_sw128(kt + off, 16, 1024);
                    if constexpr (kBF16) mma_ss_f16(tmem + bb * 128, a, bd, idS, kk > 0);
                    else mma_ss_tf32(tmem + bb * 128, a, bd, idS, kk > 0);
                }
                mma_commit(&s_full[bb]);
            };
            issue_S(0);
            trace_mark(p, 0, 9);
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % NST, bb = c & 1;
                const uint32_t qt = smem_u32(tiles + s * 3 * kTileBytes);
                const uint32_t kt = qt + kTileBytes, vt = qt + 2 * kTileBytes;
                // O (+)= Q~ M ; M += K~^T V  (onto e^{G_end} M already in TMEM)
                auto qm_dm = [&](bool first) {
                    mbar_wait(xf2, c & 1);
                    mbar_wait(m_ready, c & 1);
                    tc_fence_after();
                    trace_mark(p, c, 6);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                        const uint64_t a = umma_desc_sw128(qt + off, 16, 1024);
                        const uint32_t acc = (first && kk == 0) ? 0u : 1u;
                        if constexpr (!TR) {
                            const uint64_t bd = umma_desc_sw128(mb + kk * TT::KSTEP * 128, D * 128, 1024);
                            mma_ss_f16(tO, a, bd, idQM, acc);
                        } else {
                            const uint64_t bd = umma_desc_sw128(mb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
                            mma_ss_tf32(tO, a, bd, idQM, acc);
                        }
                    }
                    if (p.nomask) return;  // the state is the global sum, never updated
#pragma unroll
                    for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                        if constexpr (!TR) {
                            const uint64_t a = umma_desc_sw128(kt + kk * TT::KSTEP * 128, kBlockBytes, 1024);
                            const uint64_t bd = umma_desc_sw128(vt + kk * TT::KSTEP * 128, kBlockBytes, 1024);
                            mma_ss_f16(tM, a, bd, idDM, 1u);
                        } else {
                            const uint32_t off = (kk >> 2) * 8192 + (kk & 3) * 32;
                            mma_ss_tf32(tM, umma_desc_sw128(ka + off, 16, 1024),
                                        umma_desc_sw128(va + off, 16, 1024), idDM, 1u);
                        }
                    }
                };
                // O (+)= P V   (P from TMEM, +8 columns per K step)
                auto pv = [&](bool first) {
                    mbar_wait(p_full, c & 1);
                    tc_fence_after();
                    trace_mark(p, c, 7);
#pragma unroll
                    for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                        const uint32_t acc = (first && kk == 0) ? 0u : 1u;
                        if constexpr (!TR) {
                            const uint64_t bd = umma_desc_sw128(vt + kk * TT::KSTEP * 128, kBlockBytes, 1024);
                            mma_ts_f16(tO, tmem + bb * 128 + kk * 8, bd, idPV, acc);
                        } else {
                            const uint64_t bd = umma_desc_sw128(va + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
                            mma_ts_tf32(tO, tmem + bb * 128 + kk * 8, bd, idPV, acc);
                        }
                    }
                };
                if (p.order == 1) {
                    qm_dm(true);
                    pv(false);
                } else {
                    pv(true);
                    if (NST == 2 && c + 1 < nchunks) { issue_S(c + 1); trace_mark(p, c + 1, 9); }
                    qm_dm(false);
                }
                mma_commit(mo_full);
                mma_commit(&empty[s]);  // stage s (Q, K, V) fully consumed
                trace_mark(p, c, 8);
                if ((p.order == 1 || NST == 1) && c + 1 < nchunks) { issue_S(c + 1); trace_mark(p, c + 1, 9); }
            }
        }
    } else if (warp == 2) {
        // ---------------- decay factors, one ring slot per chunk ------------------------
        //   ringG = G (inclusive log decay), ringF = e^{r_Q - G} kf (safe) | kf (unsafe),
        //   ringS = {G_end, safe, -, -, r_0..r_3}: r_Q the log decay at the last row of key
        //   quarter Q (REV: its first row, and ringF = e^{G - r_Q})
        const float spa = (DECAY == kDecayTokenScalar) ? softplus_f(p.a_raw[h]) : 0.f;
        float bvA[4], bvB[4], bvC[4];
        auto nval = [&](int c) { return min(kC, t_end - chunk_t0(c)); };
        load_gates<DECAY>(p, b, h, chunk_t0(0), nval(0), lane, bvA);
        if (nchunks > 1) load_gates<DECAY>(p, b, h, chunk_t0(1), nval(1), lane, bvB);
        float gtot = 0.f;  // the segment's total log decay (local-state mode)
        for (int c = 0; c < nchunks; ++c) {
            const int slot = c & 1;
            if (c + 2 < nchunks) load_gates<DECAY>(p, b, h, chunk_t0(c + 2), nval(c + 2), lane, bvC);
            if (c >= 2) mbar_wait(&gfree[slot], ((c >> 1) - 1) & 1);
            float G[4], kf[4];
            const float gend = chunk_scan<DECAY>(p, bvA, nval(c), spa, lane, G, kf);
            gtot += gend;
            // split e^{G_i - G_j} = e^{G_i - r_Q} e^{r_Q - G_j} per 32-key quarter Q (lane / 8),
            // r_Q = G at the quarter's last key: the key factor is <= 1 and the query factor
            // only exceeds 1 on the diagonal block, so both stay finite while every quarter's
            // decay span is < 80 (REV mirrors it with r_Q at the quarter's first key)
            const float qfirst = __shfl_sync(0xFFFFFFFFu, G[0], lane & ~7);
            const float qlast = __shfl_sync(0xFFFFFFFFu, G[3], lane | 7);
            const float r = REV ? qfirst : qlast;
            const bool safe = __all_sync(0xFFFFFFFFu, (qfirst - qlast) < -kSafeLogDecay);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                ringG[slot * 128 + lane * 4 + u] = G[u];
                if constexpr (REV)  // column factor e^{G_j - r_Q} of e^{G_j - G_i}; no key kf
                    ringF[slot * 128 + lane * 4 + u] = (DECAY != kDecayNone && safe) ? __expf(G[u] - r) : 1.f;
                else
                    ringF[slot * 128 + lane * 4 + u] =
                        (DECAY != kDecayNone && safe) ? __expf(r - G[u]) * kf[u] : kf[u];
            }
            if (lane == 0) {
                ringS[slot * 8] = gend;
                ringS[slot * 8 + 1] = safe ? 1.f : 0.f;
            }
            if ((lane & 7) == 0) ringS[slot * 8 + 4 + (lane >> 3)] = r;
            __syncwarp();
            mbar_arrive(&gfull[slot]);
#pragma unroll
            for (int u = 0; u < 4; ++u) { bvA[u] = bvB[u]; bvB[u] = bvC[u]; }
        }
        if (p.local && lane == 0) p.logDseg[(size_t)bh * p.nseg + seg] = gtot;
    } else if (warp == 3) {
        // ---------------- O store warp (bf16 O): bulk-store each staged chunk, then release
        // its stage once the store has read the tile, off the math warps' path
        if (lane == 0 && kBF16 && !p.out_f32) {
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % NST;
                uint8_t* qt = tiles + s * 3 * kTileBytes;
                mbar_wait(o_staged, c & 1);
                tma_store_4d(&tmO, qt, 0, h, chunk_t0(c), b);
                tma_store_4d(&tmO, qt + kBlockBytes, TT::EPB, h, chunk_t0(c), b);
                bulk_commit();
                bulk_wait_read0();
                mbar_arrive(&empty[s]);
            }
        }
    } else if (warp >= 4) {
        // ---------------- math warps ----------------------------------------------------
        const int mw = warp - 4;
        const int tid = threadIdx.x - 128;  // 0..MT-1
        const int q = warp & 3;             // TMEM lane quarter
        const int hh = mw >> 2;             // column group (0..NQ-1)
        const int row = q * 32 + lane;      // token row of S / O / Q / K tiles
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        // state rows: d_k index (M=128 layout for bf16, M=64 layout for tf32)
        const int srow = TR ? q * 16 + lane : row;
        const bool sown = TR ? lane < 16 : true;
        T* const obase = reinterpret_cast<T*>(p.o);
        auto tpart = [&](int c) -> uint32_t {
            return kBF16 ? tmem + (c & 1) * 128 + 64 + lane_off : tmem + 384 + lane_off;
        };

        auto prep = [&](int c) {  // phi(Q), phi(K) [+ tf32 rounding] in place; zero rows past the end
            const int s = c % NST;
            mbar_wait(&full[s], (c / NST) & 1);
            const int nvalid = min(kC, t_end - chunk_t0(c));
            const float sc = row < nvalid ? 1.f : 0.f;
            uint8_t* qt = tiles + s * 3 * kTileBytes;
            xform_row_part<T, FM, TR, DH>(qt, row, hh * DH, sc);
            xform_row_part<T, FM, TR, DH>(qt + kTileBytes, row, hh * DH, sc);
            fence_proxy_async_smem();
            mbar_arrive(xf1);
        };
        auto write_state_operand = [&](const float* vals) {  // DH values of row srow
            if (!sown) return;
            if constexpr (!TR) {
                uint8_t* dst = mop + (hh * DH / TT::EPB) * (D * 128);
                const int ch0 = (hh * DH % TT::EPB) / TT::EPC;
#pragma unroll
                for (int ch = 0; ch < DH / 8; ++ch) {
                    uint4 v;
                    v.x = pack_bf16(vals[ch * 8 + 0], vals[ch * 8 + 1]);
                    v.y = pack_bf16(vals[ch * 8 + 2], vals[ch * 8 + 3]);
                    v.z = pack_bf16(vals[ch * 8 + 4], vals[ch * 8 + 5]);
                    v.w = pack_bf16(vals[ch * 8 + 6], vals[ch * 8 + 7]);
                    *reinterpret_cast<uint4*>(dst + sw128_off(srow, ch0 + ch)) = v;
                }
            } else {
                // M^T K-major: element (d_v j, d_k i) -> block i/32, row j
                uint8_t* base = mop + (srow >> 5) * 8192 + ((srow & 3) << 2);
                const int cch = (srow & 31) >> 2;
#pragma unroll
                for (int j = 0; j < DH; ++j)
                    *reinterpret_cast<float*>(base + sw128_off(hh * DH + j, cch)) = tf32r(vals[j]);
            }
        };

        // backward side channel (see LsmFwdParams::mst): vals = this thread's DH state values
        // of row srow, the operand of processing step cidx
        auto state_hook = [&](const float* vals, int cidx) {
            if (p.mst == nullptr || !sown) return;
            const int cg = chunk_t0(cidx) / kC;
            T* dst = reinterpret_cast<T*>(p.mst) + (((size_t)bh * p.nchunk_tot + cg) * D + srow) * D + hh * DH;
#pragma unroll
            for (int j = 0; j < DH; j += 8) {
                if constexpr (kBF16) {
                    uint4 w;
                    w.x = pack_bf16(vals[j], vals[j + 1]); w.y = pack_bf16(vals[j + 2], vals[j + 3]);
                    w.z = pack_bf16(vals[j + 4], vals[j + 5]); w.w = pack_bf16(vals[j + 6], vals[j + 7]);
                    *reinterpret_cast<uint4*>(dst + j) = w;
                } else {
                    *reinterpret_cast<float4*>(dst + j) = make_float4(vals[j], vals[j + 1], vals[j + 2], vals[j + 3]);
                    *reinterpret_cast<float4*>(dst + j + 4) = make_float4(vals[j + 4], vals[j + 5], vals[j + 6], vals[j + 7]);
                }
            }
        };

        if constexpr (kPrep) prep(0);
        // initial state: operand M_0, TMEM M = e^{G_end(0)} M_0
        {
            // the entering state's load does not depend on the decay warp: issue it first
            float vals[DH];
            const size_t mslot = p.nomask ? (size_t)bh : (size_t)bh * p.nseg + seg;
            const float* src = p.Min + (mslot * D + (sown ? srow : 0)) * D + hh * DH;
            bool have = sown;
            if (p.local) {  // local-state mode: only segment 0 enters with a state (Mloc0)
                have = sown && seg == 0 && p.Mloc0 != nullptr;
                src = have ? p.Mloc0 + ((size_t)bh * D + srow) * D + hh * DH : nullptr;
            }
#pragma unroll
            for (int j = 0; j < DH; j += 4) {
                const float4 v = have ? *reinterpret_cast<const float4*>(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                vals[j] = v.x; vals[j + 1] = v.y; vals[j + 2] = v.z; vals[j + 3] = v.w;
            }
            mbar_wait(&gfull[0], 0);
            const float g0 = __expf(ringS[0]);  // G_end of chunk 0
            write_state_operand(vals);
            state_hook(vals, 0);
#pragma unroll
            for (int cb = 0; cb < DH / 32; ++cb) {
                uint32_t r[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(vals[cb * 32 + j] * g0);
                tmem_st32(tM + lane_off + hh * DH + cb * 32, r);
            }
            if constexpr (NORM) {
                if (tid < D) sZ[tid] = p.zin[((size_t)bh * p.nseg + seg) * D + tid];
                named_bar_sync(1, MT);
            }
            tmem_wait_st();
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(m_ready);
        }

        for (int c = 0; c < nchunks; ++c) {
            const int s = c % NST, bb = c & 1, slot = c & 1;
            const int t0 = chunk_t0(c);
            const int nvalid = min(kC, t_end - t0);
            // REV with Mamba2 keff queries (dv pass): kf_i = softplus(b_i) scales output row i
            float qf = 1.f;
            if constexpr (REV && DECAY == kDecayTokenScalar) {
                if (p.rev_kfq && row < nvalid)
                    qf = softplus_f(__ldg(p.b_pre + ((size_t)b * p.Nstride + t0 + row) * p.H + h));
            }
            uint8_t* qt = tiles + s * 3 * kTileBytes;
            uint8_t* kt = qt + kTileBytes;
            mbar_wait(&gfull[slot], (c >> 1) & 1);
            const float gend = ringS[slot * 8];
            const bool safe = ringS[slot * 8 + 1] != 0.f;
            const float* rQ = ringS + slot * 8 + 4;  // per-key-quarter factorisation references
            const float gi = ringG[slot * 128 + row];
            const float* Fs = ringF + slot * 128;
            const float* Gs = ringG + slot * 128;
            mbar_wait(&s_full[bb], (c >> 1) & 1);  // S(c) done: raw Q, K no longer needed
            tc_fence_after();
            if (tid == 0) trace_mark(p, c, 0);
            if constexpr (!kPrep) mbar_wait(&full[s], (c / NST) & 1);  // tile visibility
            if constexpr (TR) {
                // V^T (K-major B operand of PV and dM) before anything is published
                float vals[32];
                load_half_row_f32(qt + 2 * kTileBytes + hh * kBlockBytes, row, vals);
                store_transposed_f32(vT, row, hh, vals);
                fence_proxy_async_smem();
            }
            float zcol = 0.f;
            float qz = 0.f;  // q~_i . z_in partial (normaliser)
            // (b) Q~ = phiQ e^{G_i}, K~ = phiK kf e^{G_end - G_i}  (row owners; fp32: K~^T)
            auto do_b = [&]() {
                // forward: query cross factor e^{G_i}, key state factor e^{G_end - G_j} kf_j;
                // REV: e^{G_end - G_i} and e^{G_j}
                const float fq = (DECAY != kDecayNone) ? __expf(REV ? gend - gi : gi) : 1.f;
                float fk = 1.f;
                if constexpr (DECAY != kDecayNone && REV) fk = __expf(gi);
                if constexpr (DECAY != kDecayNone && !REV)
                    fk = safe ? __expf(gend - rQ[q]) * Fs[row] : __expf(gend - gi) * Fs[row];
                uint8_t* qb = qt + (hh * DH / TT::EPB) * kBlockBytes;
                const int qch0 = (hh * DH % TT::EPB) / TT::EPC;
                constexpr int NCH = DH / TT::EPC;
                // all of this row part's Q (and, bf16, K) chunks are loaded before any store
                // (see xform_chunks): one shared-memory round trip instead of 2 NCH
                constexpr bool kBothK = !TR && DECAY != kDecayNone;
                uint4 vq[NCH], vk[kBothK ? NCH : 1];
                if constexpr (DECAY != kDecayNone || NORM) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) vq[ch] = *reinterpret_cast<const uint4*>(qb + sw128_off(row, qch0 + ch));
                }
                if constexpr (kBothK) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) vk[ch] = *reinterpret_cast<const uint4*>(kt + (qb - qt) + sw128_off(row, qch0 + ch));
                }
                if constexpr (DECAY != kDecayNone || NORM) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) {
                        uint4& v = vq[ch];
                        if constexpr (kBF16) {
                            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float2 f = unpack_bf16(w[e]);
                                f.x *= fq; f.y *= fq;
                                if constexpr (NORM) qz += f.x * sZ[hh * DH + ch * 8 + 2 * e] + f.y * sZ[hh * DH + ch * 8 + 2 * e + 1];
                                w[e] = pack_bf16(f.x, f.y);
                            }
                        } else {
                            float* f = reinterpret_cast<float*>(&v);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                f[e] = tf32r(f[e] * fq);
                                if constexpr (NORM) qz += f[e] * sZ[hh * DH + ch * 4 + e];
                            }
                        }
                    }
                }
                if constexpr (kBothK) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) xform_chunk<T, 0, false>(vk[ch], fk);
                }
                if constexpr (DECAY != kDecayNone) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) *reinterpret_cast<uint4*>(qb + sw128_off(row, qch0 + ch)) = vq[ch];
                }
                if constexpr (kBothK) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch)
                        *reinterpret_cast<uint4*>(kt + (qb - qt) + sw128_off(row, qch0 + ch)) = vk[ch];
                }
                if constexpr (TR) {
                    float vals[32];
                    load_half_row_f32(kt + hh * kBlockBytes, row, vals);
#pragma unroll
                    for (int j = 0; j < 32; ++j) vals[j] *= fk;
                    store_transposed_f32(kT, row, hh, vals);
                }
                fence_proxy_async_smem();
                if constexpr (NORM) {
                    if (p.order == 0) {  // P already occupies the S buffer: partial slot is free
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tpart(c) + NQ + hh),
                                     "r"(__float_as_uint(qz)) : "memory");
                        tmem_wait_st();
                    }
                    named_bar_sync(1, MT);
                    if (tid < D) {
                        if constexpr (!TR) {
                            const int blk = tid / TT::EPB, cin = tid % TT::EPB;
                            const uint8_t* base = kt + blk * kBlockBytes;
                            for (int r = 0; r < kC; ++r)
                                zcol += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                                    base + sw128_off(r, cin / TT::EPC) + (cin % TT::EPC) * 2));
                        } else {
                            for (int blk = 0; blk < 4; ++blk)
#pragma unroll
                                for (int ch = 0; ch < 8; ++ch) {
                                    const float4 v = *reinterpret_cast<const float4*>(kT + blk * 8192 + sw128_off(tid, ch));
                                    zcol += v.x + v.y + v.z + v.w;
                                }
                        }
                    }
                }
                mbar_arrive(xf2);
                if (tid == 0) trace_mark(p, c, 1);
            };
            // (a) S -> P
            auto do_a = [&]() {
                uint32_t r[KC / 32][32];
                const uint32_t tS = tmem + bb * 128 + lane_off + hh * KC;
                // causal mask col <= row (REV: col >= row): a warp's KC key columns against its
                // 32 rows are all kept, all masked (no TMEM read, P = 0) or the diagonal block.
                // nomask (Alg. 1): no intra-chunk term at all (the gathered state holds every key)
                const bool zero = p.nomask || (REV ? hh * KC + KC - 1 < q * 32 : hh * KC > q * 32 + 31);
                float rs = 0.f;
                if (!zero) {
#pragma unroll
                    for (int i = 0; i < KC / 32; ++i) tmem_ld32(tS + i * 32, r[i]);
                    tmem_wait_ld();
                    // decay factor per column, the branch on `safe` (uniform per chunk) hoisted out
                    // of the column loop and the ring rows read as float4
                    if constexpr (DECAY != kDecayNone) {
                        if (safe) {
#pragma unroll
                            for (int i = 0; i < KC / 32; ++i) {
                                const float rr = rQ[hh * (KC / 32) + i];
                                const float eq = __expf(REV ? rr - gi : gi - rr);  // query factor of the key quarter
#pragma unroll
                                for (int j = 0; j < 32; j += 4) {
                                    const float4 F = *reinterpret_cast<const float4*>(Fs + hh * KC + i * 32 + j);
                                    r[i][j] = __float_as_uint(__uint_as_float(r[i][j]) * (eq * F.x));
                                    r[i][j + 1] = __float_as_uint(__uint_as_float(r[i][j + 1]) * (eq * F.y));
                                    r[i][j + 2] = __float_as_uint(__uint_as_float(r[i][j + 2]) * (eq * F.z));
                                    r[i][j + 3] = __float_as_uint(__uint_as_float(r[i][j + 3]) * (eq * F.w));
                                }
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < KC / 32; ++i) {
#pragma unroll
                                for (int j = 0; j < 32; j += 4) {
                                    const float4 G = *reinterpret_cast<const float4*>(Gs + hh * KC + i * 32 + j);
                                    const float g4[4] = {G.x, G.y, G.z, G.w};
                                    float f4[4];
                                    if constexpr (REV) {
#pragma unroll
                                        for (int u = 0; u < 4; ++u) f4[u] = __expf(g4[u] - gi);
                                    } else {
                                        const float4 F = *reinterpret_cast<const float4*>(Fs + hh * KC + i * 32 + j);
                                        f4[0] = __expf(gi - g4[0]) * F.x; f4[1] = __expf(gi - g4[1]) * F.y;
                                        f4[2] = __expf(gi - g4[2]) * F.z; f4[3] = __expf(gi - g4[3]) * F.w;
                                    }
#pragma unroll
                                    for (int u = 0; u < 4; ++u) r[i][j + u] = __float_as_uint(__uint_as_float(r[i][j + u]) * f4[u]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int j = 0; j < KC; ++j) {
                        const int col = hh * KC + j;
                        float v = (REV ? col >= row : col <= row) ? __uint_as_float(r[j / 32][j % 32]) : 0.f;
                        if constexpr (TR) v = tf32r(v);
                        rs += v;
                        r[j / 32][j % 32] = __float_as_uint(v);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < KC; ++j) r[j / 32][j % 32] = 0u;
                }
                if constexpr (kBF16) {
                    uint32_t pk[KC / 2];
#pragma unroll
                    for (int j = 0; j < KC / 2; ++j)
                        pk[j] = pack_bf16(__uint_as_float(r[(2 * j) / 32][(2 * j) % 32]),
                                          __uint_as_float(r[(2 * j + 1) / 32][(2 * j + 1) % 32]));
                    // all S reads of this TMEM lane quarter done before P overwrites them: only the
                    // NQ warps of quarter q share these lanes
                    named_bar_sync(2 + q, 32 * NQ);
                    if constexpr (KC == 32) {
                        tmem_st16(tmem + bb * 128 + lane_off + hh * 16, pk);
                    } else {
                        tmem_st32(tmem + bb * 128 + lane_off + hh * 32, pk);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < KC / 32; ++i) tmem_st32(tS + i * 32, r[i]);
                }
                if constexpr (NORM) {
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tpart(c) + hh),
                                 "r"(__float_as_uint(rs)) : "memory");
                    if (p.order == 1)
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tpart(c) + NQ + hh),
                                     "r"(__float_as_uint(qz)) : "memory");
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(p_full);
                if (tid == 0) trace_mark(p, c, 2);
            };
            if (p.order == 1) { do_b(); do_a(); }
            else { do_a(); do_b(); }
            mbar_arrive(&gfree[slot]);
            if (NST == 2 && kPrep && c + 1 < nchunks) prep(c + 1);
            // (c) state: M_{c+1} from TMEM -> operand; TMEM <- e^{G_end(c+1)} M_{c+1}
            mbar_wait(mo_full, c & 1);
            tc_fence_after();
            if (tid == 0) trace_mark(p, c, 3);
            if (c + 1 < nchunks) {
                const int ns = (c + 1) & 1;
                mbar_wait(&gfull[ns], ((c + 1) >> 1) & 1);
                const float gnext = __expf(ringS[ns * 8]);
                float vals[DH];
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    uint32_t r[32];
                    tmem_ld32(tM + lane_off + hh * DH + cb * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) vals[cb * 32 + j] = __uint_as_float(r[j]);
                }
                write_state_operand(vals);
                state_hook(vals, c + 1);
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    uint32_t r[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(vals[cb * 32 + j] * gnext);
                    tmem_st32(tM + lane_off + hh * DH + cb * 32, r);
                }
                if constexpr (NORM) {
                    if (tid < D) sZ[tid] = __expf(gend) * sZ[tid] + zcol;
                }
                tmem_wait_st();
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(m_ready);
                if (tid == 0) trace_mark(p, c, 4);
            }
            // (d) O epilogue: registers -> global (this row's 128-byte half, 8 x 16 B)
            {
                float inv = 1.f;
                if constexpr (NORM) {
                    float den = 0.f;
#pragma unroll
                    for (int i = 0; i < 2 * NQ; ++i) {
                        uint32_t pr;
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(pr) : "r"(tpart(c) + i));
                        tmem_wait_ld();
                        den += __uint_as_float(pr);
                    }
                    if (fabsf(den) < 1e-12f && row < nvalid) atomicOr(&p.err[0], 1);
                    inv = 1.f / den;
                }
                if constexpr (REV) inv = qf;
                const bool vrow = row < nvalid;
                if (kBF16 && !p.out_f32) {
                    // bf16 O: stage this thread's half row in the (consumed) Q tile in the TMA
                    // SW128 layout, then one thread bulk-stores the tile (rows >= N clipped)
#pragma unroll
                    for (int cb = 0; cb < DH / 32; ++cb) {
                        uint32_t r[32];
                        tmem_ld32(tO + lane_off + hh * DH + cb * 32, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            uint4 v;
                            v.x = pack_bf16(__uint_as_float(r[ch * 8 + 0]) * inv, __uint_as_float(r[ch * 8 + 1]) * inv);
                            v.y = pack_bf16(__uint_as_float(r[ch * 8 + 2]) * inv, __uint_as_float(r[ch * 8 + 3]) * inv);
                            v.z = pack_bf16(__uint_as_float(r[ch * 8 + 4]) * inv, __uint_as_float(r[ch * 8 + 5]) * inv);
                            v.w = pack_bf16(__uint_as_float(r[ch * 8 + 6]) * inv, __uint_as_float(r[ch * 8 + 7]) * inv);
                            *reinterpret_cast<uint4*>(qt + (hh * DH / TT::EPB) * kBlockBytes +
                                                      sw128_off(row, (hh * DH % TT::EPB) / TT::EPC + cb * 4 + ch)) = v;
                        }
                    }
                    tc_fence_before();
                    fence_proxy_async_smem();
                    mbar_arrive(o_staged);  // warp 3 stores the tile and releases the stage
                } else if (kBF16 && p.out_f32) {  // fp32 rows (backward intermediates)
                    float* dstf = reinterpret_cast<float*>(p.o) +
                                  (((size_t)b * p.Nstride + t0 + (vrow ? row : 0)) * p.H + h) * D + hh * DH;
#pragma unroll
                    for (int cb = 0; cb < DH / 32; ++cb) {
                        uint32_t r[32];
                        tmem_ld32(tO + lane_off + hh * DH + cb * 32, r);
                        tmem_wait_ld();
                        if (vrow) {
#pragma unroll
                            for (int ch = 0; ch < 8; ++ch)
                                *reinterpret_cast<float4*>(dstf + cb * 32 + ch * 4) =
                                    make_float4(__uint_as_float(r[ch * 4]) * inv, __uint_as_float(r[ch * 4 + 1]) * inv,
                                                __uint_as_float(r[ch * 4 + 2]) * inv, __uint_as_float(r[ch * 4 + 3]) * inv);
                        }
                    }
                } else {
                T* dst = obase + (((size_t)b * p.Nstride + t0 + (vrow ? row : 0)) * p.H + h) * D + hh * DH;
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    uint32_t r[32];
                    tmem_ld32(tO + lane_off + hh * DH + cb * 32, r);
                    tmem_wait_ld();
                    if (vrow) {
                        if constexpr (kBF16) {
#pragma unroll
                            for (int ch = 0; ch < 4; ++ch) {
                                uint4 v;
                                v.x = pack_bf16(__uint_as_float(r[ch * 8 + 0]) * inv, __uint_as_float(r[ch * 8 + 1]) * inv);
                                v.y = pack_bf16(__uint_as_float(r[ch * 8 + 2]) * inv, __uint_as_float(r[ch * 8 + 3]) * inv);
                                v.z = pack_bf16(__uint_as_float(r[ch * 8 + 4]) * inv, __uint_as_float(r[ch * 8 + 5]) * inv);
                                v.w = pack_bf16(__uint_as_float(r[ch * 8 + 6]) * inv, __uint_as_float(r[ch * 8 + 7]) * inv);
                                *reinterpret_cast<uint4*>(dst + cb * 32 + ch * 8) = v;
                            }
                        } else {
#pragma unroll
                            for (int ch = 0; ch < 8; ++ch)
                                *reinterpret_cast<float4*>(dst + cb * 32 + ch * 4) =
                                    make_float4(__uint_as_float(r[ch * 4]) * inv, __uint_as_float(r[ch * 4 + 1]) * inv,
                                                __uint_as_float(r[ch * 4 + 2]) * inv, __uint_as_float(r[ch * 4 + 3]) * inv);
                        }
                    }
                }
                }
                if (!(kBF16 && !p.out_f32) && tid == 0) mbar_arrive(&empty[s]);  // stage untouched
                tc_fence_before();
                if (tid == 0) trace_mark(p, c, 5);
            }
            if (NST == 1 && kPrep && c + 1 < nchunks) prep(c + 1);
        }
        // local-state mode: the segment's final state (TMEM M after the last chunk's dM, which
        // the last iteration's mo_full wait covered) -> Sseg, the combine's input
        if (p.local && sown) {
            float* dst = p.Sseg + (((size_t)bh * p.nseg + seg) * D + srow) * D + hh * DH;
#pragma unroll
            for (int cb = 0; cb < DH / 32; ++cb) {
                uint32_t r[32];
                tmem_ld32(tM + lane_off + hh * DH + cb * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + cb * 32 + j) =
                        make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                    __uint_as_float(r[j + 3]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    trace_cta(p, 1);
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// ====================================================================================
// Local-state correction (decaying scalar kinds, bf16, identity feature map).  The output
// pass ran every segment from a zero state; with M_in(s) from the segment combine the exact
// output is
//     o_t = o_t^local + (q_t e^{Gseg_t}) M_in(s),   Gseg_t = log decay from the segment start
//                                                   through token t (inclusive)
// and e^{Gseg_t} only decreases along the segment, so the correction stops at the first chunk
// that starts below e^{-88} (the fp32 normal range: below it the term is smaller than any
// representable output difference).  For Mamba2 / Lightning / RetNet that is a few chunks
// per segment, so the step reads q, k, v once (no state pass).  One CTA per (segment, head):
// thread 0 issues TMA and the MMAs; the 8 warps transform Q~ and add the product to O.
// ====================================================================================
constexpr int kFixThreads = 256;
constexpr int fix_smem() { return 3 * kTileBytes + 128 * 4 + 64; }

template <int DECAY>
__global__ void __launch_bounds__(kFixThreads, 1)
    lsm_local_fix(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO, LsmFwdParams p) {
    using T = __nv_bfloat16;
    using TT = TileTraits<T>;
    constexpr int D = 128;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* qt = smem;                   // Q~ tile
    uint8_t* ot = smem + kTileBytes;      // O tile (read, updated, stored)
    uint8_t* mop = smem + 2 * kTileBytes; // bf16 M_in operand (the output pass's layout)
    float* sG = reinterpret_cast<float*>(smem + 3 * kTileBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sG + 128);
    uint64_t* full = bars;
    uint64_t* mma_done = bars + 1;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 2);
    __shared__ float sGcum, sGend;

    const int seg = p.nseg - (int)gridDim.x + blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // the last gridDim.x segments
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id(), tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(full, 1);
        mbar_init(mma_done, 1);
        fence_barrier_init();
        sGcum = 0.f;
    }
    if (warp == 0) tmem_alloc<128>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    pdl_wait();
    pdl_trigger();
    // M_in(seg) -> bf16 operand: thread (row, column half)
    {
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
    const float spa = (DECAY == kDecayTokenScalar) ? softplus_f(p.a_raw[h]) : 0.f;
    const int q = warp & 3, half = warp >> 2;  // TMEM lane quarter, column half
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    for (int c = 0; c < nchunks; ++c) {
        __syncthreads();  // sGcum of the previous chunk, previous O store read
        if (sGcum < -88.f) break;  // every later factor is below the fp32 normal range
        const int t0 = t_begin + c * kC;
        const int nvalid = min(kC, t_end - t0);
        if (tid == 0) {
            bulk_wait_read0();  // the previous chunk's O store has read the tile
            mbar_expect_tx(full, 4 * kBlockBytes);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                tma_load_4d(qt + blk * kBlockBytes, &tmQ, full, blk * TT::EPB, h, t0, b);
                tma_load_4d(ot + blk * kBlockBytes, &tmO, full, blk * TT::EPB, h, t0, b);
            }
        }
        if (warp == 0) {  // the chunk's inclusive log decay G_t (chunk-local), as the decay warp
            float bv[4], G[4], kf[4];
            load_gates<DECAY>(p, b, h, t0, nvalid, lane, bv);
            const float gend = chunk_scan<DECAY>(p, bv, nvalid, spa, lane, G, kf);
#pragma unroll
            for (int u = 0; u < 4; ++u) sG[lane * 4 + u] = G[u];
            if (lane == 0) sGend = gend;
        }
        __syncthreads();
        mbar_wait(full, c & 1);
        // Q~ = q e^{Gcum + G_t} in place: thread (row = tid % 128, column half)
        {
            const int r2 = tid & 127, hf = tid >> 7;
            const float f = r2 < nvalid ? __expf(sGcum + sG[r2]) : 0.f;
            xform_chunks<T, 0, false, 8>(qt + hf * kBlockBytes, r2, 0, f);
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
        mbar_wait(mma_done, c & 1);
        tc_fence_after();
        // O += Q~ M_in for this thread's row and 64 columns, in the O tile, then one bulk store
        {
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
            sGcum += sGend;
        }
    }
    if (tid == 0) bulk_wait0();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
}

}  // namespace lmoe_dev
