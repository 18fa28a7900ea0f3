// lsm_vec_scan.cuh -- shared 2-D column scans of one 128-token chunk tile for the
// TokenVector-decay kernels (lsm_vec_kernels.cuh, lsm_vec_bwd.cu).
//
// NT = 256 threads own the tile as 16 column chunks (16 bytes = EPC columns) x 16 row groups
// of 8 rows: thread (cg = tid % 16, rg = tid / 16).  A warp touches two full 256-byte rows per
// access (conflict-free 16-byte smem transactions).  The column scan is two-level: each thread
// scans its 8 rows in registers, group totals go through shared memory, and the first D
// threads turn them into exclusive per-group offsets (plus the per-column carry of the
// calling kernel) -- no thread walks a whole column.
#pragma once
#include "lsm_kernels.cuh"

namespace lmoe_dev {

constexpr int kVecNT = 256;  // transform threads of every TokenVector kernel

// MUFU ex2 / lg2 / rcp without the denormal fix-ups of __expf / __logf (flush-to-zero)
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_exp(float x) { return ex2_ftz(x * 1.4426950408889634f); }
// log sigmoid(x) = min(x, 0) - log(1 + e^{-|x|}) (abs error ~1e-7, far below the bf16 / tf32
// operand rounding it feeds)
__device__ __forceinline__ float log_sigmoid_fast(float x) {
    return fminf(x, 0.f) - 0.6931471805599453f * lg2_ftz(1.f + ex2_ftz(-fabsf(x) * 1.4426950408889634f));
}
__device__ __forceinline__ float sigmoid_fast(float x) { return rcp_ftz(1.f + fast_exp(-x)); }

template <typename T, int NT = kVecNT>
struct VecLayout {
    static constexpr int EPC = TileTraits<T>::EPC;  // columns per 16-byte chunk
    static constexpr int D = TileTraits<T>::D;      // 16 chunks per row
    static constexpr int RG = NT / 16;              // row groups
    static constexpr int R = kC / RG;               // rows per thread (8 at NT = 256)
};

// the raw 16-byte chunk (row, cg) of a two-block SW128 tile, and its EPC values
__device__ __forceinline__ uint4 ld_chunk_raw(const uint8_t* tile, int row, int cg) {
    return *reinterpret_cast<const uint4*>(tile + (cg >> 3) * kBlockBytes + sw128_off(row, cg & 7));
}
template <typename T>
__device__ __forceinline__ void unpack_chunk(const uint4& u, float (&x)[TileTraits<T>::EPC]) {
    if constexpr (sizeof(T) == 2) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = unpack_bf16(w[i]);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
    } else {
        x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
        x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
    }
}

// EPC consecutive values of (row, chunk cg) of a two-block SW128 tile
template <typename T>
__device__ __forceinline__ void ld_chunk(const uint8_t* tile, int row, int cg, float (&x)[TileTraits<T>::EPC]) {
    const uint4 u = *reinterpret_cast<const uint4*>(tile + (cg >> 3) * kBlockBytes + sw128_off(row, cg & 7));
    if constexpr (sizeof(T) == 2) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = unpack_bf16(w[i]);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
    } else {
        x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
        x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
    }
}
// store (bf16 round-to-nearest, or fp32 rounded to tf32 for the tensor core)
template <typename T>
__device__ __forceinline__ void st_chunk(uint8_t* tile, int row, int cg, const float (&x)[TileTraits<T>::EPC]) {
    uint4 u;
    if constexpr (sizeof(T) == 2) {
        u.x = pack_bf16(x[0], x[1]); u.y = pack_bf16(x[2], x[3]);
        u.z = pack_bf16(x[4], x[5]); u.w = pack_bf16(x[6], x[7]);
    } else {
        u.x = __float_as_uint(tf32r(x[0])); u.y = __float_as_uint(tf32r(x[1]));
        u.z = __float_as_uint(tf32r(x[2])); u.w = __float_as_uint(tf32r(x[3]));
    }
    *reinterpret_cast<uint4*>(tile + (cg >> 3) * kBlockBytes + sw128_off(row, cg & 7)) = u;
}

// fp32 tiles: store without the tf32 rounding (intermediates that are rounded later)
template <typename T>
__device__ __forceinline__ void st_chunk_raw(uint8_t* tile, int row, int cg, const float (&x)[TileTraits<T>::EPC]) {
    if constexpr (sizeof(T) == 2) {
        st_chunk<T>(tile, row, cg, x);
    } else {
        *reinterpret_cast<uint4*>(tile + (cg >> 3) * kBlockBytes + sw128_off(row, cg & 7)) =
            make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
    }
}

// Inclusive chunk-local log-decay G[ii][j] (row rg*R+ii, column cg*EPC+j) from the gate tile
// `at` (la = log sigmoid(a) on valid rows, 0 beyond nvalid).  Also, per column:
//   sR[c]  = G at row 63 (the midpoint reference), sGe[c] = G at the chunk end,
//   sG0[c] = G at row 0 (range check of the midpoint split),
//   sCar[c] = the caller's running carry before this chunk; carry += G_end afterwards
//   (only threads tid < D hold a meaningful `carry`).
// sTot: [RG][D] scratch.  Two named barriers (id 1, NT threads).
template <typename T, int NT = kVecNT>
__device__ __forceinline__ void vec_log_scan(const uint8_t* at, int nvalid, int tid,
                                             float (&G)[VecLayout<T, NT>::R][VecLayout<T, NT>::EPC], float* sTot,
                                             float* sR, float* sGe, float* sG0, float* sCar, float& carry) {
    using L = VecLayout<T, NT>;
    const int cg = tid & 15, rg = tid >> 4;
    float run[L::EPC];
#pragma unroll
    for (int j = 0; j < L::EPC; ++j) run[j] = 0.f;
#pragma unroll
    for (int ii = 0; ii < L::R; ++ii) {
        const int row = rg * L::R + ii;
        float x[L::EPC];
        ld_chunk<T>(at, row, cg, x);
        const float vm = row < nvalid ? 1.f : 0.f;  // branch-free: rows past the end add 0
#pragma unroll
        for (int j = 0; j < L::EPC; ++j) {
            run[j] = fmaf(log_sigmoid_fast(x[j]), vm, run[j]);
            G[ii][j] = run[j];
        }
    }
#pragma unroll
    for (int j = 0; j < L::EPC; ++j) sTot[rg * L::D + cg * L::EPC + j] = run[j];
    if (rg == 0) {
#pragma unroll
        for (int j = 0; j < L::EPC; ++j) sG0[cg * L::EPC + j] = G[0][j];
    }
    named_bar_sync(1, NT);
    if (tid < L::D) {
        float acc = 0.f, r = 0.f;
#pragma unroll
        for (int g = 0; g < L::RG; ++g) {
            const float v = sTot[g * L::D + tid];
            sTot[g * L::D + tid] = acc;
            acc += v;
            if ((g + 1) * L::R == 64) r = acc;
        }
        sR[tid] = r;
        sGe[tid] = acc;
        if (sCar) sCar[tid] = carry;
        carry += acc;
    }
    named_bar_sync(1, NT);
#pragma unroll
    for (int j = 0; j < L::EPC; ++j) {
        const float off = sTot[rg * L::D + cg * L::EPC + j];
#pragma unroll
        for (int ii = 0; ii < L::R; ++ii) G[ii][j] += off;
    }
}

// Midpoint split range check of one column (the forward's e^{G-r} / e^{r-G} folding).
__device__ __forceinline__ bool vec_split_ok(float g0, float r, float ge) {
    return (g0 - r) < -kSafeLogDecay && (r - ge) < -kSafeLogDecay;
}

}  // namespace lmoe_dev
