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
//   phase 3  lsm_output_pass  per (b,h,segment), chunk by chunk (C = 128 tokens):
//                S  = phiQ Keff^T                           (tcgen05, TMEM)
//                P  = S . exp(G_i - G_j) . [j <= i]         (registers -> TMEM, bf16/tf32)
//                O  = P V + (phiQ . e^{G}) M                (tcgen05, P read from TMEM)
//                dM = (Keff . e^{G_end - G})^T V            (tcgen05)
//                M  = e^{G_end} M + dM                      (fp32 master state in registers)
//
// Tile layout in shared memory: every Q/K/V tile is 128 token rows x 256 bytes, stored as
// two SWIZZLE_128B column blocks of [128 rows x 128 B] exactly as TMA writes them; this
// covers bf16 d=128 and fp32 (tf32 MMA) d=64 with the same byte arithmetic.
#pragma once
#include "ptx.cuh"

namespace lmoe_dev {

constexpr int kC = 128;                         // chunk rows (tokens) per device tile
constexpr int kRowBytes = 256;                  // head_dim * sizeof(T)
constexpr int kTileBytes = kC * kRowBytes;      // 32 KB
constexpr int kBlockBytes = kC * 128;           // one SW128 column block of a tile: 16 KB
constexpr int kMathThreads = 256;               // 8 epilogue/transform warps

enum DecayMode { kDecayNone = 0, kDecayConst = 1, kDecayTokenScalar = 2 };

struct LsmFwdParams {
    int B, N, H;
    int seg_len;       // tokens per segment, multiple of kC
    int nseg;          // segments per (b,h)
    int decay;         // DecayMode
    int fm;            // 0 identity, 1 elu+1, 2 squared
    int norm;          // normaliser on
    int mamba2_keff;   // keff = phi(k) * softplus(b)
    float log_a;       // ConstScalar: log(a)
    const float* b_pre;  // [B,N,H]   TokenScalar gate pre-activation
    const float* a_raw;  // [H]       Mamba2 static parameter
    float* Sseg;         // [B*H][nseg][dk][dv]
    float* zseg;         // [B*H][nseg][dk]
    float* logDseg;      // [B*H][nseg]
    const float* Min;    // [B*H][nseg][dk][dv]  (phase 3 input)
    const float* zin;    // [B*H][nseg][dk]
    int* err;            // [0] degenerate normaliser, [1] non-finite state
};

template <typename T>
struct TileTraits;
template <>
struct TileTraits<__nv_bfloat16> {
    static constexpr int D = 128;          // head dim
    static constexpr int EPC = 8;          // elements per 16-byte chunk
    static constexpr int EPB = 64;         // elements per 128-byte block row
    static constexpr int KSTEP = 16;       // UMMA K per instruction
    static constexpr uint32_t FMT = 1;     // BF16
    static constexpr int MBUF_BYTES = 128 * 128 * 2;
};
template <>
struct TileTraits<float> {
    static constexpr int D = 64;
    static constexpr int EPC = 4;
    static constexpr int EPB = 32;
    static constexpr int KSTEP = 8;        // tf32
    static constexpr uint32_t FMT = 2;     // TF32
    static constexpr int MBUF_BYTES = 64 * 64 * 4;
};

__device__ __forceinline__ float softplus_f(float x) {
    return x > 30.f ? x : log1pf(__expf(x));
}
__device__ __forceinline__ float fmap_f(int fm, float x) {
    if (fm == 1) return x > 0.f ? x + 1.f : __expf(x);
    if (fm == 2) return x * x;
    return x;
}

// Elementwise transform of one 16-byte chunk (8 bf16 or 4 fp32) in place.
template <typename T>
__device__ __forceinline__ void xform_chunk(uint8_t* p, int fm, float scale, bool apply_fm) {
    uint4 v = *reinterpret_cast<uint4*>(p);
    if constexpr (sizeof(T) == 2) {
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f = unpack_bf16(w[i]);
            if (apply_fm) { f.x = fmap_f(fm, f.x); f.y = fmap_f(fm, f.y); }
            w[i] = pack_bf16(f.x * scale, f.y * scale);
        }
    } else {
        float* f = reinterpret_cast<float*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float x = apply_fm ? fmap_f(fm, f[i]) : f[i];
            f[i] = x * scale;
        }
    }
    *reinterpret_cast<uint4*>(p) = v;
}

// Inclusive scan of one float per thread over `n` consecutive threads starting at thread 0
// of a group of warps; `tmp` holds >= n/32 floats.  Must be called by all threads of the
// group (count `nthreads`, named barrier `bar_id`).
__device__ __forceinline__ float group_inclusive_scan(float x, float* tmp, int tid,
                                                      uint32_t bar_id, uint32_t nthreads) {
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        float y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[w] = x;
    named_bar_sync(bar_id, nthreads);
    float off = 0.f;
    for (int i = 0; i < w; ++i) off += tmp[i];
    named_bar_sync(bar_id, nthreads);
    return x + off;
}

}  // namespace lmoe_dev

namespace lmoe_dev {
template <typename T>
__global__ void lsm_state_pass(const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV, LsmFwdParams p);
template <typename T>
__global__ void lsm_output_pass(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK,
                                const __grid_constant__ CUtensorMap tmV,
                                const __grid_constant__ CUtensorMap tmO, LsmFwdParams p);
__global__ void lsm_seg_combine(const float* __restrict__ S, const float* __restrict__ zS,
                                const float* __restrict__ logD, const float* __restrict__ M0,
                                const float* __restrict__ z0, float* __restrict__ Min,
                                float* __restrict__ zin, float* __restrict__ Mfin,
                                float* __restrict__ zfin, int nseg, int dk, int dv, int norm,
                                int* err);
constexpr int kStatePassSmem = 3 * 2 * kTileBytes + 2048;
constexpr int kStatePassThreads = 192;
constexpr int kOutputPassThreads = 320;
template <typename T>
constexpr int output_pass_smem() { return 2 * 3 * kTileBytes + TileTraits<T>::MBUF_BYTES + 1280; }
}  // namespace lmoe_dev
