// lsm_fwd.cu -- device kernels of the chunkwise LSM forward (see lsm_fwd.cuh for the math).
#include "lsm_fwd.cuh"

namespace lmoe_dev {

// ------------------------------------------------------------------------------------
// Phase 1: per-segment state  S_seg = sum_j exp(L_j) keff_j v_j^T   (TMEM accumulator)
// warps: 0 = TMA producer, 1 = MMA issuer, 2..5 = transform (128 threads)
// ------------------------------------------------------------------------------------
constexpr int kSPStages = 3;
constexpr int kSPThreads = 192;

template <typename T>
__global__ void __launch_bounds__(kSPThreads, 1)
    lsm_state_pass(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   LsmFwdParams p) {
    using TT = TileTraits<T>;
    constexpr int D = TT::D;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* tiles = smem;  // stage s: K at s*64K, V at s*64K+32K
    float* sG = reinterpret_cast<float*>(smem + kSPStages * 2 * kTileBytes);  // 128
    float* sTmp = sG + 128;                                                 // 8
    float* sZ = sTmp + 8;                                                   // 128 colsum acc
    uint64_t* bars = reinterpret_cast<uint64_t*>(sZ + 128);
    uint64_t* full = bars;                 // [kSPStages]
    uint64_t* empty = bars + kSPStages;    // [kSPStages]
    uint64_t* xf = bars + 2 * kSPStages;   // transform done (128 arrivals)
    uint64_t* acc_full = xf + 1;           // MMA accumulation finished
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        for (int i = 0; i < kSPStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(xf, 128);
        mbar_init(acc_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<128>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % kSPStages;
                if (it >= kSPStages) mbar_wait(&empty[s], ((it / kSPStages) - 1) & 1);
                const int c = nchunks - 1 - it;  // reverse order
                const int t0 = t_begin + c * kC;
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
            constexpr uint32_t idesc = umma_idesc(TT::FMT, 1, 1, 128, D);
            constexpr int ksteps = kC / TT::KSTEP;
            constexpr uint32_t kstep_bytes = TT::KSTEP * 128;
            for (int it = 0; it < nchunks; ++it) {
                const int s = it % kSPStages;
                mbar_wait(&full[s], (it / kSPStages) & 1);
                mbar_wait(xf, it & 1);
                tc_fence_after();
                const uint32_t kt = smem_u32(tiles + s * 2 * kTileBytes);
                const uint32_t vt = kt + kTileBytes;
#pragma unroll
                for (int kk = 0; kk < ksteps; ++kk) {
                    uint64_t a = umma_desc_sw128(kt + kk * kstep_bytes, kBlockBytes, 1024);
                    uint64_t bd = umma_desc_sw128(vt + kk * kstep_bytes, kBlockBytes, 1024);
                    if constexpr (sizeof(T) == 2)
                        mma_ss_f16(tmem, a, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
                    else
                        mma_ss_tf32(tmem, a, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&empty[s]);
            }
            mma_commit(acc_full);
        }
    } else {
        // transform warps: K <- keff(phi(K)) * exp(L_j); L_j = log decay from token j
        // (exclusive) to the segment end.
        const int tid = threadIdx.x - 64;  // 0..127
        float suffix = 0.f;                // log decay of the already-visited (later) chunks
        float zacc = 0.f;                  // normaliser colsum, column tid
        const bool need_fm = p.fm != 0 || p.mamba2_keff;
        const float spa = (p.decay == kDecayTokenScalar) ? softplus_f(p.a_raw[h]) : 0.f;
        for (int it = 0; it < nchunks; ++it) {
            const int s = it % kSPStages;
            const int c = nchunks - 1 - it;
            const int t0 = t_begin + c * kC;
            const int nvalid = min(kC, t_end - t0);
            // per-token log decay and keff multiplier
            float la = 0.f, kf = 1.f;
            {
                const int tok = t0 + tid;
                const bool valid = tid < nvalid;
                if (p.decay == kDecayConst) la = valid ? p.log_a : 0.f;
                if (p.decay == kDecayTokenScalar || p.mamba2_keff) {
                    const float bv = valid ? p.b_pre[((size_t)b * p.N + tok) * p.H + h] : 0.f;
                    const float spb = softplus_f(bv);
                    if (p.decay == kDecayTokenScalar) la = valid ? -spb * spa : 0.f;
                    if (p.mamba2_keff) kf = spb;
                }
                if (!valid) kf = 0.f;
            }
            const float G = group_inclusive_scan(la, sTmp, tid, 1, 128);
            // chunk total log decay (thread 127 holds it)
            if (tid == 127) sTmp[4] = G;
            named_bar_sync(1, 128);
            const float gend = sTmp[4];
            // weight for own token row tid: exp(gend - G + suffix) * kf
            sG[tid] = __expf(gend - G + suffix) * kf;
            mbar_wait(&full[s], (it / kSPStages) & 1);
            named_bar_sync(1, 128);
            uint8_t* kt = tiles + s * 2 * kTileBytes;
            if (p.decay != kDecayNone || need_fm || nvalid < kC) {
#pragma unroll 4
                for (int i = 0; i < 2 * kC * 8 / 128; ++i) {  // 2048 chunks / 128 threads
                    const int g = i * 128 + tid;
                    const int blk = g >> 10, row = (g >> 3) & 127;
                    xform_chunk<T>(kt + blk * kBlockBytes + (g & 1023) * 16, p.fm, sG[row],
                                   need_fm && p.fm != 0);
                }
                fence_proxy_async_smem();
            }
            if (p.norm) {
                named_bar_sync(1, 128);
                if (tid < D) {
                    const int blk = tid / TT::EPB, cin = tid % TT::EPB;
                    const int ch = cin / TT::EPC, e = cin % TT::EPC;
                    const uint8_t* base = kt + blk * kBlockBytes;
                    float acc = 0.f;
                    for (int r = 0; r < kC; ++r) {
                        const uint8_t* q = base + sw128_off(r, ch) + e * sizeof(T);
                        if constexpr (sizeof(T) == 2)
                            acc += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(q));
                        else
                            acc += *reinterpret_cast<const float*>(q);
                    }
                    zacc += acc;
                }
            }
            mbar_arrive(xf);
            suffix += gend;
        }
        // epilogue: S (d_k rows x d_v cols) from TMEM to global
        mbar_wait(acc_full, 0);
        tc_fence_after();
        const int q = warp & 3;  // TMEM lane quarter of this warp
        const int row = q * 32 + lane;
        float* dst = p.Sseg + (((size_t)bh * p.nseg + seg) * D + row) * D;
        if (row < D) {
#pragma unroll
            for (int cb = 0; cb < D / 32; ++cb) {
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + cb * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + cb * 32 + j) =
                        make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                    __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
            }
        } else {
            // warps whose lane quarter lies beyond d_k (fp32 d=64) still take part in the
            // warp-collective TMEM loads' convention: nothing to do.
        }
        if (tid < D && p.norm) p.zseg[((size_t)bh * p.nseg + seg) * D + tid] = zacc;
        if (tid == 0) p.logDseg[(size_t)bh * p.nseg + seg] = suffix;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<128>(tmem);
}

// ------------------------------------------------------------------------------------
// Phase 2: decayed exclusive prefix over segments (and ranks, for SP)
//   Min[s] = acc ; acc = exp(logD[s]) * acc + S[s]        per element of [M | z]
// ------------------------------------------------------------------------------------
__global__ void lsm_seg_combine(const float* __restrict__ S, const float* __restrict__ zS,
                                const float* __restrict__ logD, const float* __restrict__ M0,
                                const float* __restrict__ z0, float* __restrict__ Min,
                                float* __restrict__ zin, float* __restrict__ Mfin,
                                float* __restrict__ zfin, int nseg, int dk, int dv, int norm,
                                int* err) {
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int nm = dk * dv;
    const int total = nm + (norm ? dk : 0);
    if (e >= total) return;
    const bool isz = e >= nm;
    const int ee = isz ? e - nm : e;
    const int stride = isz ? dk : nm;
    const float* src = isz ? zS : S;
    float* dst = isz ? zin : Min;
    float acc = 0.f;
    if (isz) { if (z0) acc = z0[(size_t)bh * dk + ee]; }
    else if (M0) acc = M0[(size_t)bh * nm + ee];
    const size_t base = (size_t)bh * nseg * stride + ee;
    for (int s = 0; s < nseg; ++s) {
        if (dst) dst[base + (size_t)s * stride] = acc;
        acc = __expf(logD[(size_t)bh * nseg + s]) * acc + src[base + (size_t)s * stride];
    }
    if (!isfinite(acc)) atomicOr(&err[1], 1);
    float* fin = isz ? zfin : Mfin;
    if (fin) fin[(size_t)bh * (isz ? dk : nm) + ee] = acc;
}

// ------------------------------------------------------------------------------------
// Phase 3: output pass.  warps: 0 = TMA, 1 = MMA, 2..9 = math (256 threads)
// TMEM columns: [0,128) S / P,  [128,256) O,  [256,384) dM,  384/385 row partials
// ------------------------------------------------------------------------------------
constexpr int kOPThreads = 320;

template <typename T>
__global__ void __launch_bounds__(kOPThreads, 1)
    lsm_output_pass(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    LsmFwdParams p) {
    using TT = TileTraits<T>;
    constexpr int D = TT::D;
    constexpr bool kBF16 = sizeof(T) == 2;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* tiles = smem;  // stage s: Q, K, V at s*96K + {0, 32K, 64K}
    uint8_t* mbuf = smem + 2 * 3 * kTileBytes;
    float* sG = reinterpret_cast<float*>(mbuf + TT::MBUF_BYTES);  // 128
    float* sZ = sG + 128;                                          // 128
    float* sTmp = sZ + 128;                                        // 16
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTmp + 16);
    uint64_t* full = bars;         // [2]
    uint64_t* empty = bars + 2;    // [2]
    uint64_t* xf1 = bars + 4;      // math -> MMA: tiles transformed (phi / keff)
    uint64_t* s_full = bars + 5;   // MMA -> math: S in TMEM
    uint64_t* p_full = bars + 6;   // math -> MMA: P in TMEM
    uint64_t* xf2 = bars + 7;      // math -> MMA: Q~, K~ ready
    uint64_t* m_full = bars + 8;   // math -> MMA: bf16/tf32 state operand ready
    uint64_t* mo_full = bars + 9;  // MMA -> math: O and dM complete
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 10);

    const int seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int bh = b * p.H + h;
    const int t_begin = seg * p.seg_len;
    const int t_end = min(p.N, t_begin + p.seg_len);
    const int nchunks = (t_end - t_begin + kC - 1) / kC;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(xf1, kMathThreads);
        mbar_init(s_full, 1);
        mbar_init(p_full, kMathThreads);
        mbar_init(xf2, kMathThreads);
        mbar_init(m_full, kMathThreads);
        mbar_init(mo_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    const uint32_t tS = tmem, tO = tmem + 128, tM = tmem + 256, tR = tmem + 384;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmO);
            for (int c = 0; c < nchunks; ++c) {
                const int s = c & 1;
                if (c >= 2) mbar_wait(&empty[s], ((c >> 1) - 1) & 1);
                const int t0 = t_begin + c * kC;
                uint8_t* st = tiles + s * 3 * kTileBytes;
                mbar_expect_tx(&full[s], 3 * kTileBytes);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    tma_load_4d(st + blk * kBlockBytes, &tmQ, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + kTileBytes + blk * kBlockBytes, &tmK, &full[s], blk * TT::EPB, h, t0, b);
                    tma_load_4d(st + 2 * kTileBytes + blk * kBlockBytes, &tmV, &full[s], blk * TT::EPB, h, t0, b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc(TT::FMT, 0, 0, 128, 128);
            constexpr uint32_t idPV = umma_idesc(TT::FMT, 0, 1, 128, D);
            constexpr uint32_t idQM = umma_idesc(TT::FMT, 0, 1, 128, D);
            constexpr uint32_t idDM = umma_idesc(TT::FMT, 1, 1, 128, D);
            constexpr uint32_t kstep_mn = TT::KSTEP * 128;  // MN-major K advance (bytes)
            const uint32_t mb = smem_u32(mbuf);
            for (int c = 0; c < nchunks; ++c) {
                const int s = c & 1;
                const uint32_t qt = smem_u32(tiles + s * 3 * kTileBytes);
                const uint32_t kt = qt + kTileBytes, vt = qt + 2 * kTileBytes;
                mbar_wait(&full[s], (c >> 1) & 1);
                mbar_wait(xf1, c & 1);
                tc_fence_after();
                // S = phiQ . Keff^T      (K-major A and B, K = head dim: 8 steps of 32 B)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    const uint64_t a = umma_desc_sw128(qt + off, 16, 1024);
                    const uint64_t bd = umma_desc_sw128(kt + off, 16, 1024);
                    if constexpr (kBF16) mma_ss_f16(tS, a, bd, idS, kk > 0);
                    else mma_ss_tf32(tS, a, bd, idS, kk > 0);
                }
                mma_commit(s_full);
                // O = P V      (A = P from TMEM, +8 columns per K step; B = V MN-major)
                mbar_wait(p_full, c & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                    const uint64_t bd = umma_desc_sw128(vt + kk * kstep_mn, kBlockBytes, 1024);
                    if constexpr (kBF16) mma_ts_f16(tO, tS + kk * 8, bd, idPV, kk > 0);
                    else mma_ts_tf32(tO, tS + kk * 8, bd, idPV, kk > 0);
                }
                mbar_wait(xf2, c & 1);
                mbar_wait(m_full, c & 1);
                tc_fence_after();
                // O += Q~ M      (A = Q~ K-major; B = state MN-major [d_k rows][d_v])
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                    const uint64_t a = umma_desc_sw128(qt + off, 16, 1024);
                    const uint64_t bd = umma_desc_sw128(mb + kk * kstep_mn, D * 128, 1024);
                    if constexpr (kBF16) mma_ss_f16(tO, a, bd, idQM, 1u);
                    else mma_ss_tf32(tO, a, bd, idQM, 1u);
                }
                // dM = K~^T V  (A = K~ MN-major over d_k, B = V MN-major; K = tokens)
#pragma unroll
                for (int kk = 0; kk < kC / TT::KSTEP; ++kk) {
                    const uint64_t a = umma_desc_sw128(kt + kk * kstep_mn, kBlockBytes, 1024);
                    const uint64_t bd = umma_desc_sw128(vt + kk * kstep_mn, kBlockBytes, 1024);
                    if constexpr (kBF16) mma_ss_f16(tM, a, bd, idDM, kk > 0);
                    else mma_ss_tf32(tM, a, bd, idDM, kk > 0);
                }
                mma_commit(mo_full);
            }
        }
    } else {
        // ---------------- math warps ----------------
        const int mw = warp - 2;           // 0..7
        const int tid = threadIdx.x - 64;  // 0..255
        const int q = warp & 3;            // TMEM lane quarter
        const int hh = mw >> 2;            // column half
        const int row = q * 32 + lane;     // tile row owned in TMEM epilogues
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        constexpr int DH = D / 2;          // d_v columns per half
        constexpr int MROWS = D;           // d_k rows of the state
        const bool own_state_row = row < MROWS;
        const bool need_fm = p.fm != 0;
        const float spa = (p.decay == kDecayTokenScalar) ? softplus_f(p.a_raw[h]) : 0.f;

        // fp32 master state: row `row`, columns [hh*DH, hh*DH + DH)
        float Mreg[DH];
        {
            const float* src = p.Min + (((size_t)bh * p.nseg + seg) * D + (own_state_row ? row : 0)) * D + hh * DH;
#pragma unroll
            for (int j = 0; j < DH; j += 4) {
                float4 v = own_state_row ? *reinterpret_cast<const float4*>(src + j) : make_float4(0, 0, 0, 0);
                Mreg[j] = v.x; Mreg[j + 1] = v.y; Mreg[j + 2] = v.z; Mreg[j + 3] = v.w;
            }
        }
        auto write_state_operand = [&]() {
            if (!own_state_row) return;
            // MN-major B operand [d_k rows][d_v]: column block = hh, row = row
            uint8_t* dst = mbuf + hh * (D * 128);
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                uint4 v;
                if constexpr (kBF16) {
                    v.x = pack_bf16(Mreg[ch * 8 + 0], Mreg[ch * 8 + 1]);
                    v.y = pack_bf16(Mreg[ch * 8 + 2], Mreg[ch * 8 + 3]);
                    v.z = pack_bf16(Mreg[ch * 8 + 4], Mreg[ch * 8 + 5]);
                    v.w = pack_bf16(Mreg[ch * 8 + 6], Mreg[ch * 8 + 7]);
                } else {
                    v = make_uint4(__float_as_uint(Mreg[ch * 4]), __float_as_uint(Mreg[ch * 4 + 1]),
                                   __float_as_uint(Mreg[ch * 4 + 2]), __float_as_uint(Mreg[ch * 4 + 3]));
                }
                *reinterpret_cast<uint4*>(dst + sw128_off(row, ch)) = v;
            }
        };
        write_state_operand();
        if (p.norm && tid < D) sZ[tid] = p.zin[((size_t)bh * p.nseg + seg) * D + tid];
        fence_proxy_async_smem();
        mbar_arrive(m_full);  // state operand for chunk 0

        for (int c = 0; c < nchunks; ++c) {
            const int s = c & 1;
            const int t0 = t_begin + c * kC;
            const int nvalid = min(kC, t_end - t0);
            uint8_t* qt = tiles + s * 3 * kTileBytes;
            uint8_t* kt = qt + kTileBytes;
            // (1) per-token cumulative log decay G (inclusive) and Mamba2 keff factor
            float la = 0.f, kf = 1.f;
            if (tid < kC) {
                const int tok = t0 + tid;
                const bool valid = tid < nvalid;
                if (p.decay == kDecayConst) la = valid ? p.log_a : 0.f;
                if (p.decay == kDecayTokenScalar || p.mamba2_keff) {
                    const float bv = valid ? p.b_pre[((size_t)b * p.N + tok) * p.H + h] : 0.f;
                    const float spb = softplus_f(bv);
                    if (p.decay == kDecayTokenScalar) la = valid ? -spb * spa : 0.f;
                    if (p.mamba2_keff) kf = spb;
                }
                if (!valid) kf = 0.f;
            }
            const float Gt = group_inclusive_scan(la, sTmp, tid, 1, kMathThreads);
            if (tid < kC) sG[tid] = Gt;
            if (tid == kC - 1) sTmp[8] = Gt;
            // keff factor per row kept in the (otherwise unused) upper half of sTmp? No:
            // stash it in TMEM-free smem: reuse sZ's tail is unsafe; keep a second array.
            named_bar_sync(1, kMathThreads);
            const float gend = sTmp[8];
            mbar_wait(&full[s], (c >> 1) & 1);
            // (2) transform 1: phi(Q), keff(phi(K)); zero rows beyond the sequence end
            const bool xf1_needed = need_fm || p.mamba2_keff || nvalid < kC;
            if (xf1_needed) {
                // keff multipliers for K rows travel through the scan scratch: recompute
                // per row from b_pre (cheap, L1-resident) to keep shared memory free.
#pragma unroll 2
                for (int i = 0; i < 2 * 2 * kC * 8 / kMathThreads; ++i) {  // Q and K tiles
                    const int g = i * kMathThreads + tid;                  // 0..4095
                    const int tile = g >> 11;                              // 0 = Q, 1 = K
                    const int gg = g & 2047;
                    const int blk = gg >> 10, r = (gg >> 3) & 127;
                    float scale = r < nvalid ? 1.f : 0.f;
                    if (tile == 1 && p.mamba2_keff && r < nvalid)
                        scale = softplus_f(p.b_pre[((size_t)b * p.N + t0 + r) * p.H + h]);
                    xform_chunk<T>((tile ? kt : qt) + blk * kBlockBytes + (gg & 1023) * 16, p.fm,
                                   scale, need_fm);
                }
                fence_proxy_async_smem();
            }
            mbar_arrive(xf1);
            // (3) S -> P: exact pairwise decay exp(G_i - G_j), causal mask j <= i
            mbar_wait(s_full, c & 1);
            tc_fence_after();
            {
                uint32_t r0[32], r1[32];
                tmem_ld32(tS + lane_off + hh * 64, r0);
                tmem_ld32(tS + lane_off + hh * 64 + 32, r1);
                tmem_wait_ld();
                const float gi = sG[row];
                float rs = 0.f;
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    const int col = hh * 64 + j;
                    float v = __uint_as_float(j < 32 ? r0[j] : r1[j - 32]);
                    float f = (col <= row) ? 1.f : 0.f;
                    if (p.decay != kDecayNone && col <= row) f = __expf(gi - sG[col]);
                    v *= f;
                    rs += v;
                    if (j < 32) r0[j] = __float_as_uint(v); else r1[j - 32] = __float_as_uint(v);
                }
                if constexpr (kBF16) {
                    uint32_t pk[32];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        pk[j] = pack_bf16(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
                        pk[16 + j] = pack_bf16(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
                    }
                    // every warp must finish reading S before P (half width) overwrites it
                    named_bar_sync(1, kMathThreads);
                    tmem_st32(tS + lane_off + hh * 32, pk);
                } else {
                    tmem_st32(tS + lane_off + hh * 64, r0);
                    tmem_st32(tS + lane_off + hh * 64 + 32, r1);
                }
                uint32_t rsv[1] = {__float_as_uint(rs)};
                asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tR + lane_off + hh),
                             "r"(rsv[0]) : "memory");
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(p_full);
            }
            // (4) transform 2: Q~ = Q e^{G_i},  K~ = K e^{G_end - G_j}
            if (p.decay != kDecayNone) {
#pragma unroll 2
                for (int i = 0; i < 2 * 2 * kC * 8 / kMathThreads; ++i) {
                    const int g = i * kMathThreads + tid;
                    const int tile = g >> 11;
                    const int gg = g & 2047;
                    const int blk = gg >> 10, r = (gg >> 3) & 127;
                    const float scale = tile ? __expf(gend - sG[r]) : __expf(sG[r]);
                    xform_chunk<T>((tile ? kt : qt) + blk * kBlockBytes + (gg & 1023) * 16, 0,
                                   scale, false);
                }
                fence_proxy_async_smem();
            }
            float zcol = 0.f;
            if (p.norm) {
                named_bar_sync(1, kMathThreads);
                // q~_i . z_in partial over this half's d_k columns (block hh of the Q tile)
                {
                    float acc = 0.f;
                    const uint8_t* qb = qt + hh * kBlockBytes;
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch) {
                        const uint4 v = *reinterpret_cast<const uint4*>(qb + sw128_off(row, ch));
                        if constexpr (kBF16) {
                            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float2 f = unpack_bf16(w[e]);
                                acc += f.x * sZ[hh * 64 + ch * 8 + 2 * e] + f.y * sZ[hh * 64 + ch * 8 + 2 * e + 1];
                            }
                        } else {
                            acc += __uint_as_float(v.x) * sZ[hh * 32 + ch * 4] +
                                   __uint_as_float(v.y) * sZ[hh * 32 + ch * 4 + 1] +
                                   __uint_as_float(v.z) * sZ[hh * 32 + ch * 4 + 2] +
                                   __uint_as_float(v.w) * sZ[hh * 32 + ch * 4 + 3];
                        }
                    }
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(
                                     tR + lane_off + 2 + hh),
                                 "r"(__float_as_uint(acc)) : "memory");
                    tmem_wait_st();
                }
                // colsum of K~ for the normaliser state, column tid
                if (tid < D) {
                    const int blk = tid / TT::EPB, cin = tid % TT::EPB;
                    const int ch = cin / TT::EPC, e = cin % TT::EPC;
                    const uint8_t* base = kt + blk * kBlockBytes;
                    for (int r = 0; r < kC; ++r) {
                        const uint8_t* ptr = base + sw128_off(r, ch) + e * sizeof(T);
                        if constexpr (kBF16) zcol += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(ptr));
                        else zcol += *reinterpret_cast<const float*>(ptr);
                    }
                }
            }
            mbar_arrive(xf2);
            // (5) state update M = e^{G_end} M + dM ; refresh the MMA operand
            mbar_wait(mo_full, c & 1);
            tc_fence_after();
            const float gamma = __expf(gend);
            if (own_state_row || kBF16) {
                uint32_t r[32];
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    tmem_ld32(tM + lane_off + hh * DH + cb * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) Mreg[cb * 32 + j] = gamma * Mreg[cb * 32 + j] + __uint_as_float(r[j]);
                }
            } else {
                // fp32 d=64: lanes 64..127 of dM hold no state rows; keep the warp-collective
                // load shape uniform anyway
                uint32_t r[32];
                tmem_ld32(tM + lane_off + hh * DH, r);
                tmem_wait_ld();
            }
            if (c + 1 < nchunks) {
                write_state_operand();
                if (p.norm && tid < D) sZ[tid] = gamma * sZ[tid] + zcol;
                fence_proxy_async_smem();
                mbar_arrive(m_full);
            } else if (p.norm && tid < D) {
                sZ[tid] = gamma * sZ[tid] + zcol;
            }
            // (6) O epilogue -> staging (Q tile buffer) -> TMA store
            {
                float den = 1.f;
                if (p.norm) {
                    uint32_t pr[4];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(pr[0]), "=r"(pr[1]), "=r"(pr[2]), "=r"(pr[3])
                                 : "r"(tR + lane_off));
                    tmem_wait_ld();
                    den = __uint_as_float(pr[0]) + __uint_as_float(pr[1]) + __uint_as_float(pr[2]) +
                          __uint_as_float(pr[3]);
                    if (fabsf(den) < 1e-12f && row < nvalid) atomicOr(&p.err[0], 1);
                }
                const float inv = 1.f / den;
                uint8_t* stg = qt + hh * kBlockBytes;
#pragma unroll
                for (int cb = 0; cb < DH / 32; ++cb) {
                    uint32_t r[32];
                    tmem_ld32(tO + lane_off + hh * DH + cb * 32, r);
                    tmem_wait_ld();
                    if constexpr (kBF16) {
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            uint4 v;
                            v.x = pack_bf16(__uint_as_float(r[ch * 8 + 0]) * inv, __uint_as_float(r[ch * 8 + 1]) * inv);
                            v.y = pack_bf16(__uint_as_float(r[ch * 8 + 2]) * inv, __uint_as_float(r[ch * 8 + 3]) * inv);
                            v.z = pack_bf16(__uint_as_float(r[ch * 8 + 4]) * inv, __uint_as_float(r[ch * 8 + 5]) * inv);
                            v.w = pack_bf16(__uint_as_float(r[ch * 8 + 6]) * inv, __uint_as_float(r[ch * 8 + 7]) * inv);
                            *reinterpret_cast<uint4*>(stg + sw128_off(row, cb * 4 + ch)) = v;
                        }
                    } else {
#pragma unroll
                        for (int ch = 0; ch < 8; ++ch) {
                            uint4 v = make_uint4(__float_as_uint(__uint_as_float(r[ch * 4]) * inv),
                                                 __float_as_uint(__uint_as_float(r[ch * 4 + 1]) * inv),
                                                 __float_as_uint(__uint_as_float(r[ch * 4 + 2]) * inv),
                                                 __float_as_uint(__uint_as_float(r[ch * 4 + 3]) * inv));
                            *reinterpret_cast<uint4*>(stg + sw128_off(row, ch)) = v;
                        }
                    }
                }
                tc_fence_before();
                fence_proxy_async_smem();
                named_bar_sync(1, kMathThreads);
                if (tid == 0) {
                    tma_store_4d(&tmO, qt, 0, h, t0, b);
                    tma_store_4d(&tmO, qt + kBlockBytes, TT::EPB, h, t0, b);
                    bulk_commit();
                    bulk_wait_read0();
                    mbar_arrive(&empty[s]);
                }
            }
        }
        if (tid == 0) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

template __global__ void lsm_state_pass<__nv_bfloat16>(const __grid_constant__ CUtensorMap,
                                                       const __grid_constant__ CUtensorMap, LsmFwdParams);
template __global__ void lsm_state_pass<float>(const __grid_constant__ CUtensorMap,
                                               const __grid_constant__ CUtensorMap, LsmFwdParams);
template __global__ void lsm_output_pass<__nv_bfloat16>(const __grid_constant__ CUtensorMap,
                                                        const __grid_constant__ CUtensorMap,
                                                        const __grid_constant__ CUtensorMap,
                                                        const __grid_constant__ CUtensorMap, LsmFwdParams);
template __global__ void lsm_output_pass<float>(const __grid_constant__ CUtensorMap,
                                                const __grid_constant__ CUtensorMap,
                                                const __grid_constant__ CUtensorMap,
                                                const __grid_constant__ CUtensorMap, LsmFwdParams);

}  // namespace lmoe_dev
