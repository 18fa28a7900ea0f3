// lsm_fwd.cuh -- chunkwise unified-LSM forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Restates lsm_forward_chunked / chunk_forward_separable
// (/root/reference/proj/include/lmoe/lsm.hpp:554-598, 668-708) for the scalar-decay
// families (DecayKind None / ConstScalar / TokenScalar: BLA, Rebased, Lightning, RetNet,
// Mamba2) as a three-phase segment-parallel scan -- the same algorithm as LSM sequence
// parallelism (parallel.hpp:303-376), applied inside one GPU:
//
//   phase 1  lsm_state_pass   per (b,h,segment): S_seg = sum_j exp(L_j) keff_j v_j^T
//                             (L_j = log-decay from token j to the segment end), z_seg,
//                             log D_seg.  Chunks are visited last-to-first so the decay
//                             weights are known without a pre-pass; S accumulates in TMEM.
//   phase 2  lsm_seg_combine  per (b,h): decayed exclusive prefix over segments
//                             M_in(s+1) = D_s M_in(s) + S_s (+ initial state M0).
//   phase 3  lsm_output_pass  per (b,h,segment), chunk by chunk (C = 128 tokens), with
//            G_t = inclusive chunk-local log decay, kf_t = Mamba2 softplus(b_t) (else 1):
//                S  = phiQ phiK^T                               (tcgen05 -> TMEM, 2 buffers)
//                P  = S . e^{G_i} . (e^{-G_j} kf_j) . [j <= i]  (registers -> TMEM)
//                O  = P V + (phiQ . e^{G}) M                    (tcgen05; P read from TMEM)
//                M' = e^{G_end} M + (phiK . kf . e^{G_end-G})^T V (tcgen05, accumulated
//                                                              onto the TMEM-resident state)
//            The pairwise factor is split as e^{G_i} e^{-G_j} when the chunk's total decay
//            is > e^-80 (no overflow); otherwise P uses exact e^{G_i - G_j} per element.
//
// Tile layout in shared memory: every Q/K/V tile is 128 token rows x 256 bytes, two
// SWIZZLE_128B column blocks of [128 rows x 128 B] exactly as TMA writes them; this covers
// bf16 d=128 and fp32 (tf32 MMA) d=64 with the same byte arithmetic.  tf32 operands must be
// K-major (measured: MN-major tf32 descriptors yield zeros), so the fp32 path transposes
// K~ and V into K-major [d rows x 128 tokens] tiles and keeps the state operand as M^T.
#pragma once
#include "ptx.cuh"

namespace lmoe_dev {

constexpr int kC = 128;                         // chunk rows (tokens) per device tile
constexpr int kRowBytes = 256;                  // head_dim * sizeof(T)
constexpr int kTileBytes = kC * kRowBytes;      // 32 KB
constexpr int kBlockBytes = kC * 128;           // one SW128 column block of a tile: 16 KB
constexpr int kMathThreads = 256;               // 8 epilogue warps (output pass)
constexpr float kSafeLogDecay = -80.f;          // e^{-G} stays finite in fp32 above this

// single-read forward: the aggregate of segment s lives in ring slot s % fR with fR = 2 fP.  Its
// readers are the segments (s, s + fP); the writer of s + 2 fP first needs the aggregate of a
// segment that each of those readers publishes only after its look-back has read slot s.
enum DecayMode { kDecayNone = 0, kDecayConst = 1, kDecayTokenScalar = 2, kDecayTokenVector = 3 };

struct LsmFwdParams {
    int B, N, H;
    int Nstride;       // sequence length of the underlying [B, Nstride, H] gate buffer
    int seg_len;       // tokens per segment, multiple of kC
    int nseg;          // segments per (b,h)
    float log_a;       // ConstScalar: log(a)
    const float* b_pre;  // [B,N,H]   TokenScalar gate pre-activation
    const float* a_raw;  // [H]       Mamba2 static parameter
    float* Sseg;         // [B*H][nseg][dk][dv]
    float* zseg;         // [B*H][nseg][dk]
    float* logDseg;      // [B*H][nseg][lw]  (lw = 1, or d_k for TokenVector decays)
    const float* Min;    // [B*H][nseg][dk][dv]  (phase 3 input)
    const float* zin;    // [B*H][nseg][dk]
    void* o;             // [B, Nstride, H, D] output (phase 3), written from registers
    int* err;            // [0] degenerate normaliser, [1] non-finite state
    int order;           // phase-3 schedule: 0 = P epilogue first, 1 = transforms first
    int out_f32;         // bf16 inputs, fp32 output rows (backward intermediates)
    int rev_kfq;         // REV passes: scale output rows by kf_i = softplus(b_i) (Mamba2 keff query)
    int nomask;          // unmasked SP (sp_lsm_nomask_rank): O = phiQ M_in[bh], no intra term,
                         // no state update; Min is [B*H][dk][dv] (shared by all segments)
    // backward side channel (Mamba2 gate gradients, lsm_dgate.cu): the state operand of every
    // chunk (the state before it in forward order, the state gradient after it in REV order)
    // written to mst [BH][nchunk_tot][D][D] in T
    void* mst;
    int nchunk_tot;
    unsigned long long* trace;  // optional clock64 trace of CTA (0,0,0) [64 chunks][16]
    // local-state forward (decaying scalar kinds, see lsm_local_fix): every segment but the
    // first starts from a zero state; the output pass writes each segment's final state to
    // Sseg and its total log decay to logDseg; Mloc0 = the initial state of segment 0 or null
    int local;
    const float* Mloc0;
    int fault;                  // TEST ONLY (LMOE_FLAG_TEST_DECAY_FAULT): decay shifted by one token
    // single-read persistent forward (lsm_fused.cuh): P CTAs per (b,h) walk its segments
    // j, j+P, j+2P, ...; the inclusive prefix state of segment s is handed to segment s+1
    // through ring[bh][s % R] (fp32 [D][D]) and flags[bh][s % R] = s + 1
    int fP, fR;                 // CTAs per (b,h); aggregate ring slots per (b,h) (2 fP)
    float* ring;                // [B*H][fR][D][D] segment aggregates S_seg
    int* flags;                 // [B*H][fR] = segment + 1 once its aggregate is published
    float* ringD;               // [B*H][fR] segment log decays
    float* incl;                // [B*H][fP][D][D] each CTA's inclusive prefix of its last segment
    float* Mfin;                // [B*H][D][D] final state (inclusive prefix of the last segment)
    float* fdbg;                // developer aid (LMOE_FUSED_DEBUG_PTR): per (bh, seg) S_seg, M_in, logD
};

// per-CTA globaltimer at kernel start (after the prologue) and end, slots after the 64 x 16
// chunk trace: [region][cta][2] for up to 2048 CTAs (region 0 output pass, 1 state pass)
__device__ __forceinline__ void trace_cta(const LsmFwdParams& p, int which, int region = 0) {
    if (p.trace != nullptr && threadIdx.x == 0) {
        const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        if (cta < 2048) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.trace[64 * 16 + region * 4096 + cta * 2 + which] = t;
            uint32_t sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            if (which == 0 && region < 2) p.trace[64 * 16 + 3 * 4096 + cta * 2 + region] = sm;
        }
    }
}
__device__ __forceinline__ void trace_mark(const LsmFwdParams& p, int c, int slot) {
    if (p.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && c < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
        p.trace[c * 16 + slot] = t;
    }
}

template <typename T>
struct TileTraits;
template <>
struct TileTraits<__nv_bfloat16> {
    static constexpr int D = 128;          // head dim
    static constexpr int EPC = 8;          // elements per 16-byte chunk
    static constexpr int EPB = 64;         // elements per 128-byte block row
    static constexpr int KSTEP = 16;       // UMMA K per instruction
    static constexpr uint32_t FMT = 1;     // BF16
    static constexpr int MOP_BYTES = 128 * 128 * 2;   // state operand
    static constexpr int OUT_STAGES = 2;
    static constexpr int SP_STAGES = 3;
    static constexpr bool kTransposed = false;
    static constexpr int NQ = 4;           // output-pass column groups: 16 math warps
};
template <>
struct TileTraits<float> {
    static constexpr int D = 64;
    static constexpr int EPC = 4;
    static constexpr int EPB = 32;
    static constexpr int KSTEP = 8;        // tf32
    static constexpr uint32_t FMT = 2;     // TF32
    static constexpr int MOP_BYTES = 64 * 64 * 4;
    static constexpr int OUT_STAGES = 1;
    static constexpr int SP_STAGES = 2;
    static constexpr bool kTransposed = true;  // K-major-only operands
    static constexpr int NQ = 2;
};

__device__ __forceinline__ float softplus_f(float x) {
    return x > 30.f ? x : log1pf(__expf(x));
}
template <int FM>
__device__ __forceinline__ float fmap_t(float x) {
    if constexpr (FM == 1) return x > 0.f ? x + 1.f : __expf(x);
    else if constexpr (FM == 2) return x * x;
    else return x;
}

// Shared-memory sizes (bytes).
template <typename T>
constexpr int output_pass_smem() {
    using TT = TileTraits<T>;
    return TT::OUT_STAGES * 3 * kTileBytes + (TT::kTransposed ? 2 * kTileBytes : 0) +
           TT::MOP_BYTES + 2800;
}
template <typename T>
constexpr int state_pass_smem() {
    using TT = TileTraits<T>;
    return TT::SP_STAGES * 2 * kTileBytes + (TT::kTransposed ? 2 * kTileBytes : 0) + 4096;
}
constexpr int kStatePassThreads = 256;
constexpr int kOutputPassThreads = 384;  // TokenVector output pass (lsm_vec_kernels.cuh)
// scalar-decay output pass: 4 control warps + NQ warpgroups of math warps
template <typename T>
constexpr int output_pass_threads() { return 128 + 128 * TileTraits<T>::NQ; }

// REV = reverse-time pass of the backward (lsm_bwd.cuh): out_i = sum_{j >= i} e^{G_j - G_i}
// (q'_i . k'_j) v'_j + e^{G_end - G_i} q'_i dM, chunks visited last-to-first, state carried
// towards the sequence start (dM_{c-1} = e^{g(c)} dM_c + sum_j e^{G_j} k'_j^T v'_j).
template <typename T, int DECAY, int FM, bool NORM, bool REV = false>
__global__ void lsm_state_pass(const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV, LsmFwdParams p);
template <typename T, int DECAY, int FM, bool NORM, bool REV = false>
__global__ void lsm_output_pass(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK,
                                const __grid_constant__ CUtensorMap tmV,
                                const __grid_constant__ CUtensorMap tmO, LsmFwdParams p);
__global__ void lsm_seg_combine(const float* __restrict__ S, const float* __restrict__ zS,
                                const float* __restrict__ logD, const float* __restrict__ M0,
                                const float* __restrict__ z0, float* __restrict__ Min,
                                float* __restrict__ zin, float* __restrict__ Mfin,
                                float* __restrict__ zfin, float* __restrict__ logDtot,
                                int fin_stride, int nseg, int dk, int dv, int norm, int lw, int rev,
                                int* err);
__global__ void sp_rank_combine(const float* __restrict__ gathered, int P, int BH, int rank,
                                int dk, int dv, int norm, int lw, float* __restrict__ M0,
                                float* __restrict__ z0);

}  // namespace lmoe_dev
