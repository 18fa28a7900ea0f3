// lsm_fused.cuh -- single-read persistent LSM forward (bf16, head_dim 128, scalar decays).
//
// Restates lsm_forward_chunked (/root/reference/proj/include/lmoe/lsm.hpp:668-708) over
// chunk_forward_separable (lsm.hpp:554-598) for DecayKind None / ConstScalar / TokenScalar
// (BLA and Rebased without normaliser, Lightning, RetNet, Mamba2) in ONE launch that reads
// q, k, v (and the gates) from HBM once and writes o once.
//
// Work split.  Each (b,h) sequence is cut into nseg segments of seg_len tokens; P CTAs
// (one per SM, P * B * H <= #SMs, all co-resident: cooperative launch) own a head, CTA j
// taking segments j, j+P, j+2P, ...  For one segment a CTA runs
//   A  state steps (chunks last to first): K~ = keff e^{L}, S_seg = K~^T V accumulated in
//      TMEM -- the segment's own state from zero (the phase-1 state pass of lsm_kernels.cuh);
//      K and V are loaded with an L2 evict_last policy;
//   chain  M_in(s) = the inclusive prefix of segment s-1, handed over by the CTA that owns
//      s-1 through ring[bh][(s-1) % R] and a release/acquire flag; this CTA then publishes
//      incl(s) = D_s M_in(s) + S_seg (D_s = the segment's total decay) for segment s+1.
//      The chain carries one d x d fp32 state per segment (64 KB written + read in L2), and
//      only the hand-off is serial: the A steps, the next segment's loads and its first
//      S = QK^T / P tiles run before the wait;
//   C  output steps (chunks first to last), the output pass of lsm_kernels.cuh:
//      S = phiQ phiK^T, P = S . e^{G_i - G_j} kf_j . [j <= i], O = P V + (phiQ e^{G}) M,
//      M' = e^{G_end} M + K~^T V; q, k, v loaded evict_first -- the k, v tiles are the ones
//      the A steps just read, so they come from L2.
// Segments are sized so that all CTAs' K/V between their A and C reads fit in L2
// (148 x seg_len x 512 B), so HBM sees 3 d s_in + d s_out + g bytes per (token, head).
//
// warps: 0 TMA producer, 1 MMA issuer, 2 decay factors, 3 O bulk-store, 4..19 math (512)
// TMEM: S0 [0,128) S1 [128,256) O [256,384) M [384,512); the A steps accumulate S_seg in M.
#pragma once
#include "lsm_kernels.cuh"

namespace lmoe_dev {

constexpr int kFusedThreads = 128 + 512;

// developer trace (LMOE_TRACE): globaltimer per (CTA jj of head 0, segment unit, event):
// 0 A steps start, 1 look-back start (A accumulated, C chunk 0's P done), 2 window's flags
// observed, 3 entering state folded, 4 C steps done
__device__ __forceinline__ void fused_mark(const LsmFwdParams& p, int bh, int jj, int un, int ev) {
    if (p.trace != nullptr && bh == 0 && jj < 16 && un < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[64 * 16 + (jj * 64 + un) * 5 + ev] = t;
    }
}
constexpr int fused_smem() { return 2 * 3 * kTileBytes + 128 * 128 * 2 + 2 * 256 * 4 + 16 * 4 + 24 * 8; }

template <int DECAY, int FM>
__global__ void __launch_bounds__(kFusedThreads, 1)
    lsm_fused_fwd(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                  LsmFwdParams p) {
    using T = __nv_bfloat16;
    constexpr int D = 128, NST = 2, NQ = 4, MT = 128 * NQ, DH = D / NQ, KC = 128 / NQ;
    constexpr int EPB = 64, EPC = 8;
    constexpr bool kPrep = FM != 0;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (smem_u32(smem) & 1023) __trap();
    uint8_t* tiles = smem;                                   // NST x [Q | K | V]
    uint8_t* mop = tiles + NST * 3 * kTileBytes;             // bf16 state operand (MN-major)
    float* ringG = reinterpret_cast<float*>(mop + D * D * 2);  // [2][128]: A: weights, C: G
    float* ringF = ringG + 256;                                // [2][128]
    float* ringS = ringF + 256;                                // [2][8]
    uint64_t* bars = reinterpret_cast<uint64_t*>(ringS + 16);
    uint64_t* full = bars;          // [2]
    uint64_t* empty = bars + 2;     // [2]
    uint64_t* s_full = bars + 4;    // [2]
    uint64_t* p_full = bars + 6;
    uint64_t* xf2 = bars + 7;
    uint64_t* m_ready = bars + 8;
    uint64_t* mo_full = bars + 9;
    uint64_t* gfull = bars + 10;    // [2]
    uint64_t* gfree = bars + 12;    // [2]
    uint64_t* xf1 = bars + 14;
    uint64_t* o_staged = bars + 15;
    // A step: K~ transformed.  Two barriers, alternating by A-step parity: the math warps
    // are not synchronised among themselves during the A steps, so with one barrier a fast
    // warp's arrival for step i+1 could complete step i's phase while a slow warp was still
    // transforming (measured: one warp's 32 x 32 block of K left unweighted).  A warp reaches
    // step i+2 only after the stage of step i was reloaded, i.e. after the MMA consumed step i.
    uint64_t* xfA = bars + 16;      // [2]
    uint64_t* accA = bars + 18;     // A steps of a segment accumulated
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bars + 19);

    const int BH = p.B * p.H;
    const int bh = blockIdx.x % BH, jj = blockIdx.x / BH;
    const int b = bh / p.H, h = bh % p.H;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 2);  // A: MMA commit + MMA arrive; C: MMA commit + O store
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
        mbar_init(&xfA[0], MT);
        mbar_init(&xfA[1], MT);
        mbar_init(accA, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(sTmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;
    pdl_wait();
    pdl_trigger();
    const uint32_t tO = tmem + 256, tM = tmem + 384;
    // the segments of this CTA: seg = jj + k * P
    auto span = [&](int seg, int& tb, int& te, int& n) {
        tb = seg * p.seg_len;
        te = min(p.N, tb + p.seg_len);
        n = (te - tb + kC - 1) / kC;
    };

    if (warp == 0) {
        // ---------------- TMA producer: per segment n (K, V) loads, then n (Q, K, V) loads
        if (lane == 0) {
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
            // p.order bit 0: L2 eviction hints (developer A/B knob LMOE_FUSED_HINT=0 turns them off)
            const uint64_t keep = (p.order & 1) ? l2_policy_evict_last() : l2_policy_evict_normal();
            const uint64_t drop = (p.order & 1) ? l2_policy_evict_first() : l2_policy_evict_normal();
            int g = 0;
            for (int seg = jj; seg < p.nseg; seg += p.fP) {
                int tb, te, n;
                span(seg, tb, te, n);
                for (int st = 0; st < 2 * n; ++st, ++g) {
                    const int s = g % NST;
                    if (g >= NST) mbar_wait(&empty[s], ((g / NST) - 1) & 1);
                    uint8_t* base = tiles + s * 3 * kTileBytes;
                    if (st < n) {
                        const int t0 = tb + (n - 1 - st) * kC;
                        mbar_expect_tx(&full[s], 2 * kTileBytes);
#pragma unroll
                        for (int blk = 0; blk < 2; ++blk) {
                            tma_load_4d_hint(base + kTileBytes + blk * kBlockBytes, &tmK, &full[s], blk * EPB, h, t0, b, keep);
                            tma_load_4d_hint(base + 2 * kTileBytes + blk * kBlockBytes, &tmV, &full[s], blk * EPB, h, t0, b, keep);
                        }
                    } else {
                        const int t0 = tb + (st - n) * kC;
                        mbar_expect_tx(&full[s], 3 * kTileBytes);
#pragma unroll
                        for (int blk = 0; blk < 2; ++blk) {
                            tma_load_4d_hint(base + blk * kBlockBytes, &tmQ, &full[s], blk * EPB, h, t0, b, drop);
                            tma_load_4d_hint(base + kTileBytes + blk * kBlockBytes, &tmK, &full[s], blk * EPB, h, t0, b, drop);
                            tma_load_4d_hint(base + 2 * kTileBytes + blk * kBlockBytes, &tmV, &full[s], blk * EPB, h, t0, b, drop);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ------------------------------------------------------
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc(1, 0, 0, 128, 128);
            constexpr uint32_t idPV = umma_idesc(1, 0, 1, 128, D);
            constexpr uint32_t idQM = umma_idesc(1, 0, 1, 128, D);
            constexpr uint32_t idDM = umma_idesc(1, 1, 1, 128, D);
            const uint32_t mb = smem_u32(mop);
            int g = 0, cg = 0, ag = 0;
            for (int seg = jj; seg < p.nseg; seg += p.fP) {
                int tb, te, n;
                span(seg, tb, te, n);
                // A: S_seg = sum over the segment's chunks of K~^T V
                for (int it = 0; it < n; ++it, ++g, ++ag) {
                    const int s = g % NST;
                    mbar_wait(&full[s], (g / NST) & 1);
                    mbar_wait(&xfA[ag & 1], (ag >> 1) & 1);
                    tc_fence_after();
                    const uint32_t kt = smem_u32(tiles + s * 3 * kTileBytes) + kTileBytes, vt = kt + kTileBytes;
#pragma unroll
                    for (int kk = 0; kk < kC / 16; ++kk)
                        mma_ss_f16(tM, umma_desc_sw128(kt + kk * 16 * 128, kBlockBytes, 1024),
                                   umma_desc_sw128(vt + kk * 16 * 128, kBlockBytes, 1024), idDM,
                                   (it > 0 || kk > 0) ? 1u : 0u);
                    mma_commit(&empty[s]);
                    mbar_arrive(&empty[s]);
                }
                mma_commit(accA);
                // C: the output steps
                auto issue_S = [&](int c) {
                    const int gc = g + c, cc = cg + c;
                    const int s = gc % NST, bb = cc & 1;
                    mbar_wait(&full[s], (gc / NST) & 1);
                    if constexpr (kPrep) mbar_wait(xf1, cc & 1);
                    tc_fence_after();
                    const uint32_t qt = smem_u32(tiles + s * 3 * kTileBytes), kt = qt + kTileBytes;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                        mma_ss_f16(tmem + bb * 128, umma_desc_sw128(qt + off, 16, 1024),
                                   umma_desc_sw128(kt + off, 16, 1024), idS, kk > 0);
                    }
                    mma_commit(&s_full[bb]);
                };
                issue_S(0);
                for (int c = 0; c < n; ++c) {
                    const int gc = g + c, cc = cg + c;
                    const int s = gc % NST, bb = cc & 1;
                    const uint32_t qt = smem_u32(tiles + s * 3 * kTileBytes);
                    const uint32_t kt = qt + kTileBytes, vt = qt + 2 * kTileBytes;
                    // O = Q~ M ; M += K~^T V (onto e^{G_end} M already in TMEM; not after the last chunk)
                    mbar_wait(xf2, cc & 1);
                    mbar_wait(m_ready, cc & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kBlockBytes + (kk & 3) * 32;
                        mma_ss_f16(tO, umma_desc_sw128(qt + off, 16, 1024),
                                   umma_desc_sw128(mb + kk * 16 * 128, D * 128, 1024), idQM, kk > 0 ? 1u : 0u);
                    }
                    if (c + 1 < n) {
#pragma unroll
                        for (int kk = 0; kk < kC / 16; ++kk)
                            mma_ss_f16(tM, umma_desc_sw128(kt + kk * 16 * 128, kBlockBytes, 1024),
                                       umma_desc_sw128(vt + kk * 16 * 128, kBlockBytes, 1024), idDM, 1u);
                    }
                    // O += P V (P packed bf16 in TMEM, 8 columns per K step)
                    mbar_wait(p_full, cc & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kC / 16; ++kk)
                        mma_ts_f16(tO, tmem + bb * 128 + kk * 8, umma_desc_sw128(vt + kk * 16 * 128, kBlockBytes, 1024),
                                   idPV, 1u);
                    mma_commit(mo_full);
                    mma_commit(&empty[s]);
                    if (c + 1 < n) issue_S(c + 1);
                }
                g += n;
                cg += n;
            }
        }
    } else if (warp == 2) {
        // ---------------- decay factors: one ring slot per step ---------------------------
        //  A step: ringG = e^{G_end - G_t + suffix} kf_t (weight of token t in S_seg); the last
        //          A step also leaves the segment's total log decay in ringS[3]
        //  C step: ringG = G, ringF = e^{r_Q - G} kf (safe) | kf, ringS = {G_end, safe, -, -, r_0..r_3}
        const float spa = (DECAY == kDecayTokenScalar) ? softplus_f(p.a_raw[h]) : 0.f;
        int g = 0;
        for (int seg = jj; seg < p.nseg; seg += p.fP) {
            int tb, te, n;
            span(seg, tb, te, n);
            auto t0_of = [&](int st) { return st < n ? tb + (n - 1 - st) * kC : tb + (st - n) * kC; };
            auto nval = [&](int st) { return min(kC, te - t0_of(st)); };
            float bvA[4], bvB[4], bvC[4];
            load_gates<DECAY>(p, b, h, t0_of(0), nval(0), lane, bvA);
            load_gates<DECAY>(p, b, h, t0_of(1), nval(1), lane, bvB);  // 2n >= 2 steps
            float suffix = 0.f;
            for (int st = 0; st < 2 * n; ++st, ++g) {
                const int slot = g & 1;
                if (st + 2 < 2 * n) load_gates<DECAY>(p, b, h, t0_of(st + 2), nval(st + 2), lane, bvC);
                if (g >= 2) mbar_wait(&gfree[slot], ((g >> 1) - 1) & 1);
                float G[4], kf[4];
                const float gend = chunk_scan<DECAY>(p, bvA, nval(st), spa, lane, G, kf);
                if (st < n) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) ringG[slot * 128 + lane * 4 + u] = __expf(gend - G[u] + suffix) * kf[u];
                    suffix += gend;
                    if (st == n - 1 && lane == 0) ringS[slot * 8 + 3] = suffix;
                } else {
                    const float qfirst = __shfl_sync(0xFFFFFFFFu, G[0], lane & ~7);
                    const float qlast = __shfl_sync(0xFFFFFFFFu, G[3], lane | 7);
                    const bool safe = __all_sync(0xFFFFFFFFu, (qfirst - qlast) < -kSafeLogDecay);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        ringG[slot * 128 + lane * 4 + u] = G[u];
                        ringF[slot * 128 + lane * 4 + u] =
                            (DECAY != kDecayNone && safe) ? __expf(qlast - G[u]) * kf[u] : kf[u];
                    }
                    if (lane == 0) {
                        ringS[slot * 8] = gend;
                        ringS[slot * 8 + 1] = safe ? 1.f : 0.f;
                    }
                    if ((lane & 7) == 0) ringS[slot * 8 + 4 + (lane >> 3)] = qlast;
                }
                if (p.fdbg && lane == 0) ringS[slot * 8 + 2] = __int_as_float(g);  // developer aid: step tag
                __syncwarp();
                mbar_arrive(&gfull[slot]);
#pragma unroll
                for (int u = 0; u < 4; ++u) { bvA[u] = bvB[u]; bvB[u] = bvC[u]; }
            }
        }
    } else if (warp == 3) {
        // ---------------- O store: bulk-store each staged chunk, then release its stage
        if (lane == 0) {
            const uint64_t drop = (p.order & 1) ? l2_policy_evict_first() : l2_policy_evict_normal();
            int g = 0, cg = 0;
            for (int seg = jj; seg < p.nseg; seg += p.fP) {
                int tb, te, n;
                span(seg, tb, te, n);
                for (int c = 0; c < n; ++c) {
                    const int gc = g + n + c, s = gc % NST;
                    uint8_t* qt = tiles + s * 3 * kTileBytes;
                    mbar_wait(o_staged, (cg + c) & 1);
                    tma_store_4d_hint(&tmO, qt, 0, h, tb + c * kC, b, drop);
                    tma_store_4d_hint(&tmO, qt + kBlockBytes, EPB, h, tb + c * kC, b, drop);
                    bulk_commit();
                    bulk_wait_read0();
                    mbar_arrive(&empty[s]);
                }
                g += 2 * n;
                cg += n;
            }
            bulk_wait0();
        }
    } else if (warp >= 4) {
        // ---------------- math warps ----------------------------------------------------
        const int mw = warp - 4;
        const int tid = threadIdx.x - 128;  // 0..MT-1
        const int q = warp & 3;             // TMEM lane quarter
        const int hh = mw >> 2;             // column group
        const int row = q * 32 + lane;      // token row (S, O, Q, K tiles) / d_k row (state)
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int R = p.fR;  // aggregate ring slots per (b,h)
        auto write_state_operand = [&](const float* vals) {  // DH values of state row `row`
            uint8_t* dst = mop + (hh * DH / EPB) * (D * 128);
            const int ch0 = (hh * DH % EPB) / EPC;
#pragma unroll
            for (int ch = 0; ch < DH / 8; ++ch) {
                uint4 v;
                v.x = pack_bf16(vals[ch * 8 + 0], vals[ch * 8 + 1]);
                v.y = pack_bf16(vals[ch * 8 + 2], vals[ch * 8 + 3]);
                v.z = pack_bf16(vals[ch * 8 + 4], vals[ch * 8 + 5]);
                v.w = pack_bf16(vals[ch * 8 + 6], vals[ch * 8 + 7]);
                *reinterpret_cast<uint4*>(dst + sw128_off(row, ch0 + ch)) = v;
            }
        };
        int g = 0, cg = 0, un = 0, ga = 0;
        for (int seg = jj; seg < p.nseg; seg += p.fP, ++un) {
            int tb, te, n;
            span(seg, tb, te, n);
            // ---- A steps: K~ = phi(K) . w (row owners, in place) -----------------------
            float logD = 0.f;
            if (tid == 0) fused_mark(p, bh, jj, un, 0);
            for (int it = 0; it < n; ++it, ++g, ++ga) {
                const int slot = g & 1, s = g % NST;
                mbar_wait(&gfull[slot], (g >> 1) & 1);
                const float w = ringG[slot * 128 + row];
                if (it == n - 1) logD = ringS[slot * 8 + 3];
                if (p.fdbg) {  // developer aid: count stale ring reads and non-positive weights
                    const size_t base = (size_t)p.B * p.H * p.nseg * 2 * D * D + (size_t)p.B * p.H * p.nseg;
                    if (__float_as_int(ringS[slot * 8 + 2]) != g) atomicAdd(reinterpret_cast<int*>(p.fdbg + base), 1);
                    if (!(w >= 0.f)) atomicAdd(reinterpret_cast<int*>(p.fdbg + base + 1), 1);
                }
                mbar_wait(&full[s], (g / NST) & 1);
                xform_row_part<T, FM, false, DH>(tiles + s * 3 * kTileBytes + kTileBytes, row, hh * DH, w);
                fence_proxy_async_smem();
                mbar_arrive(&xfA[ga & 1]);
                mbar_arrive(&gfree[slot]);
            }
            // ---- look-back: publish this segment's aggregate (S_seg, log D_seg); the entering
            // state is this CTA's own inclusive prefix of segment seg - P (or M0 in the first
            // round) carried through the other CTAs' aggregates of segments (seg - P, seg):
            //   M_in(seg) = D_{seg-1} (... (D_{seg-P+1} incl(seg-P) + S_{seg-P+1}) ...) + S_{seg-1}
            // No serial hand-off chain: a segment waits only for the state steps of the P - 1
            // segments before it, which run concurrently.  The order of the additions is fixed,
            // so the result does not depend on timing.
            auto chain = [&](float gend0) {
                mbar_wait(accA, un & 1);
                tc_fence_after();
                if (tid == 0) fused_mark(p, bh, jj, un, 1);
                uint32_t r[32];
                tmem_ld32(tM + lane_off + hh * DH, r);
                tmem_wait_ld();
                const int P = p.fP;
                {
                    const int slot = bh * R + seg % R;
                    float* dst = p.ring + ((size_t)slot * D + row) * D + hh * DH;
#pragma unroll
                    for (int j = 0; j < DH; j += 4)
                        __stcg(reinterpret_cast<float4*>(dst + j),
                               make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                           __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
                    if (tid == 0) __stcg(p.ringD + slot, logD);
                    // the barrier orders every thread's stores before thread 0's fence; the fence
                    // is cumulative, so the release publishes them all
                    named_bar_sync(2, MT);
                    if (tid == 0) {
                        __threadfence();
                        st_release_gpu(p.flags + slot, seg + 1);
                    }
                }
                float X[DH];
                int s0 = 0;
                const float* own = p.incl + ((size_t)(bh * P + jj) * D + row) * D + hh * DH;
                if (seg >= P) {
                    s0 = seg - P + 1;
#pragma unroll
                    for (int j = 0; j < DH; j += 4) {
                        const float4 v = __ldcg(reinterpret_cast<const float4*>(own + j));
                        X[j] = v.x; X[j + 1] = v.y; X[j + 2] = v.z; X[j + 3] = v.w;
                    }
                } else {
                    const float* m0 = p.Min ? p.Min + ((size_t)bh * D + row) * D + hh * DH : nullptr;
#pragma unroll
                    for (int j = 0; j < DH; j += 4) {
                        const float4 v = m0 ? __ldcg(reinterpret_cast<const float4*>(m0 + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
                        X[j] = v.x; X[j + 1] = v.y; X[j + 2] = v.z; X[j + 3] = v.w;
                    }
                }
                // one thread observes every flag of the window (relaxed polls, then a fence: the
                // acquire), the barrier carries that to all math threads, and then the aggregates
                // are read with no flag wait between them
                if (tid == 0) {
                    for (int s2 = s0; s2 < seg; ++s2)
                        while (ld_relaxed_gpu(p.flags + bh * R + s2 % R) != s2 + 1) __nanosleep(20);
                    __threadfence();
                }
                named_bar_sync(2, MT);
                if (tid == 0) fused_mark(p, bh, jj, un, 2);  // window observed
                for (int s2 = s0; s2 < seg; ++s2) {
                    const int slot = bh * R + s2 % R;
                    const float dl = __expf(__ldcg(p.ringD + slot));
                    const float* src = p.ring + ((size_t)slot * D + row) * D + hh * DH;
#pragma unroll
                    for (int j = 0; j < DH; j += 4) {
                        const float4 v = __ldcg(reinterpret_cast<const float4*>(src + j));
                        X[j] = fmaf(dl, X[j], v.x);
                        X[j + 1] = fmaf(dl, X[j + 1], v.y);
                        X[j + 2] = fmaf(dl, X[j + 2], v.z);
                        X[j + 3] = fmaf(dl, X[j + 3], v.w);
                    }
                }
                if (tid == 0) fused_mark(p, bh, jj, un, 3);  // M_in folded
                if (p.fdbg) {  // developer aid: [bh][seg][S_seg | M_in] + logD at the end
                    float* dbg = p.fdbg + ((size_t)bh * p.nseg + seg) * 2 * D * D + (size_t)row * D + hh * DH;
                    for (int j = 0; j < DH; ++j) { dbg[j] = __uint_as_float(r[j]); dbg[D * D + j] = X[j]; }
                    if (tid == 0) p.fdbg[(size_t)p.B * p.H * p.nseg * 2 * D * D + (size_t)bh * p.nseg + seg] = logD;
                }
                // own inclusive prefix (read back by this thread next round), or the final state
                const float dl = __expf(logD);
                const bool last = seg + 1 == p.nseg;
                float* idst = last ? (p.Mfin ? p.Mfin + ((size_t)bh * D + row) * D + hh * DH : nullptr) : const_cast<float*>(own);
                bool bad = false;
#pragma unroll
                for (int j = 0; j < DH; j += 4) {
                    float4 v;
                    v.x = fmaf(dl, X[j], __uint_as_float(r[j]));
                    v.y = fmaf(dl, X[j + 1], __uint_as_float(r[j + 1]));
                    v.z = fmaf(dl, X[j + 2], __uint_as_float(r[j + 2]));
                    v.w = fmaf(dl, X[j + 3], __uint_as_float(r[j + 3]));
                    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
                    if (idst) __stcg(reinterpret_cast<float4*>(idst + j), v);
                }
                if (bad) atomicOr(&p.err[1], 1);
                // the entering state: operand M_in, TMEM M = e^{G_end(chunk 0)} M_in
                write_state_operand(X);
                const float g0 = __expf(gend0);
                uint32_t w32[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) w32[j] = __float_as_uint(X[j] * g0);
                tmem_st32(tM + lane_off + hh * DH, w32);
                tmem_wait_st();
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(m_ready);
            };
            // ---- C steps ---------------------------------------------------------------
            auto prep = [&](int c) {  // phi(Q), phi(K) in place; zero rows past the end
                const int gc = g + c, s = gc % NST;
                mbar_wait(&full[s], (gc / NST) & 1);
                const int nvalid = min(kC, te - (tb + c * kC));
                const float sc = row < nvalid ? 1.f : 0.f;
                uint8_t* qt = tiles + s * 3 * kTileBytes;
                xform_row_part<T, FM, false, DH>(qt, row, hh * DH, sc);
                xform_row_part<T, FM, false, DH>(qt + kTileBytes, row, hh * DH, sc);
                fence_proxy_async_smem();
                mbar_arrive(xf1);
            };
            if constexpr (kPrep) prep(0);
            for (int c = 0; c < n; ++c) {
                const int gc = g + c, cc = cg + c;
                const int s = gc % NST, bb = cc & 1, slot = gc & 1;
                uint8_t* qt = tiles + s * 3 * kTileBytes;
                uint8_t* kt = qt + kTileBytes;
                mbar_wait(&gfull[slot], (gc >> 1) & 1);
                if (p.fdbg && __float_as_int(ringS[slot * 8 + 2]) != gc)
                    atomicAdd(reinterpret_cast<int*>(p.fdbg + (size_t)p.B * p.H * p.nseg * 2 * D * D + (size_t)p.B * p.H * p.nseg + 2), 1);
                const float gend = ringS[slot * 8];
                const bool safe = ringS[slot * 8 + 1] != 0.f;
                const float* rQ = ringS + slot * 8 + 4;
                const float gi = ringG[slot * 128 + row];
                const float* Fs = ringF + slot * 128;
                const float* Gs = ringG + slot * 128;
                mbar_wait(&s_full[bb], (cc >> 1) & 1);
                tc_fence_after();
                if constexpr (!kPrep) mbar_wait(&full[s], (gc / NST) & 1);
                // (b) Q~ = phiQ e^{G_i}, K~ = phiK kf e^{G_end - G_i}: this row part's Q and K
                // chunks all loaded before any store (see xform_chunks, lsm_kernels.cuh)
                {
                    if constexpr (DECAY != kDecayNone) {
                        const float fq = __expf(gi);
                        const float fk = safe ? __expf(gend - rQ[q]) * Fs[row] : __expf(gend - gi) * Fs[row];
                        uint8_t* qb = qt + (hh * DH / EPB) * kBlockBytes;
                        uint8_t* kb = kt + (hh * DH / EPB) * kBlockBytes;
                        const int qch0 = (hh * DH % EPB) / EPC;
                        constexpr int NCH = DH / EPC;
                        uint4 vq[NCH], vk[NCH];
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch) {
                            vq[ch] = *reinterpret_cast<const uint4*>(qb + sw128_off(row, qch0 + ch));
                            vk[ch] = *reinterpret_cast<const uint4*>(kb + sw128_off(row, qch0 + ch));
                        }
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch) {
                            xform_chunk<T, 0, false>(vq[ch], fq);
                            xform_chunk<T, 0, false>(vk[ch], fk);
                        }
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch) {
                            *reinterpret_cast<uint4*>(qb + sw128_off(row, qch0 + ch)) = vq[ch];
                            *reinterpret_cast<uint4*>(kb + sw128_off(row, qch0 + ch)) = vk[ch];
                        }
                    }
                    fence_proxy_async_smem();
                    mbar_arrive(xf2);
                }
                // (a) S -> P (packed bf16 into the S buffer): warps above the diagonal skip the
                // TMEM read; the `safe` branch is hoisted out of the column loop
                {
                    uint32_t r[32];
                    const uint32_t tS = tmem + bb * 128 + lane_off + hh * KC;
                    if (hh <= q) {
                        tmem_ld32(tS, r);
                        tmem_wait_ld();
                        if (DECAY == kDecayNone || safe) {
                            const float eq = (DECAY != kDecayNone) ? __expf(gi - rQ[hh]) : 1.f;
#pragma unroll
                            for (int j = 0; j < KC; j += 4) {
                                const float4 F = *reinterpret_cast<const float4*>(Fs + hh * KC + j);
                                r[j] = __float_as_uint(__uint_as_float(r[j]) * (eq * F.x));
                                r[j + 1] = __float_as_uint(__uint_as_float(r[j + 1]) * (eq * F.y));
                                r[j + 2] = __float_as_uint(__uint_as_float(r[j + 2]) * (eq * F.z));
                                r[j + 3] = __float_as_uint(__uint_as_float(r[j + 3]) * (eq * F.w));
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < KC; j += 4) {
                                const float4 G = *reinterpret_cast<const float4*>(Gs + hh * KC + j);
                                const float4 F = *reinterpret_cast<const float4*>(Fs + hh * KC + j);
                                r[j] = __float_as_uint(__uint_as_float(r[j]) * (__expf(gi - G.x) * F.x));
                                r[j + 1] = __float_as_uint(__uint_as_float(r[j + 1]) * (__expf(gi - G.y) * F.y));
                                r[j + 2] = __float_as_uint(__uint_as_float(r[j + 2]) * (__expf(gi - G.z) * F.z));
                                r[j + 3] = __float_as_uint(__uint_as_float(r[j + 3]) * (__expf(gi - G.w) * F.w));
                            }
                        }
#pragma unroll
                        for (int j = 0; j < KC; ++j)
                            if (hh * KC + j > row) r[j] = 0u;
                    } else {
#pragma unroll
                        for (int j = 0; j < KC; ++j) r[j] = 0u;
                    }
                    uint32_t pk[KC / 2];
#pragma unroll
                    for (int j = 0; j < KC / 2; ++j) pk[j] = pack_bf16(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
                    named_bar_sync(3 + q, 32 * NQ);  // this lane quarter's S reads done before P overwrites
                    tmem_st16(tmem + bb * 128 + lane_off + hh * 16, pk);
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(p_full);
                }
                mbar_arrive(&gfree[slot]);
                if (kPrep && c + 1 < n) prep(c + 1);
                if (c == 0) chain(gend);
                // (c) state: M_{c+1} from TMEM -> operand; TMEM <- e^{G_end(c+1)} M_{c+1}
                mbar_wait(mo_full, cc & 1);
                tc_fence_after();
                if (c + 1 < n) {
                    const int ns = (gc + 1) & 1;
                    mbar_wait(&gfull[ns], ((gc + 1) >> 1) & 1);
                    const float gnext = __expf(ringS[ns * 8]);
                    float vals[DH];
                    uint32_t r[32];
                    tmem_ld32(tM + lane_off + hh * DH, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) vals[j] = __uint_as_float(r[j]);
                    write_state_operand(vals);
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(vals[j] * gnext);
                    tmem_st32(tM + lane_off + hh * DH, r);
                    tmem_wait_st();
                    fence_proxy_async_smem();
                    tc_fence_before();
                    mbar_arrive(m_ready);
                }
                // (d) O epilogue: bf16 staged in the consumed Q tile, bulk-stored by warp 3
                {
                    uint32_t r[32];
                    tmem_ld32(tO + lane_off + hh * DH, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        uint4 v;
                        v.x = pack_bf16(__uint_as_float(r[ch * 8 + 0]), __uint_as_float(r[ch * 8 + 1]));
                        v.y = pack_bf16(__uint_as_float(r[ch * 8 + 2]), __uint_as_float(r[ch * 8 + 3]));
                        v.z = pack_bf16(__uint_as_float(r[ch * 8 + 4]), __uint_as_float(r[ch * 8 + 5]));
                        v.w = pack_bf16(__uint_as_float(r[ch * 8 + 6]), __uint_as_float(r[ch * 8 + 7]));
                        *reinterpret_cast<uint4*>(qt + (hh * DH / EPB) * kBlockBytes +
                                                  sw128_off(row, (hh * DH % EPB) / EPC + ch)) = v;
                    }
                    tc_fence_before();
                    fence_proxy_async_smem();
                    mbar_arrive(o_staged);
                }
            }
            if (tid == 0) fused_mark(p, bh, jj, un, 4);
            g += n;
            cg += n;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace lmoe_dev
