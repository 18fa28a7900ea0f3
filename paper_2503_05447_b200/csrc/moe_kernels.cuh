// moe_kernels.cuh -- declarations shared by moe_kernels.cu and moe_host.cu.
#pragma once
#include "ptx.cuh"

namespace lmoe_dev {

enum GemmEpilogue { kEpiBF16 = 0, kEpiSwiGLU = 1, kEpiF32 = 2 };
// routing / dispatch limits of the device kernels (the reference routes any E, top_k)
constexpr int kMoeMaxE = 256;
constexpr int kMoeMaxK = 32;
constexpr int kGemmThreads = 320;  // TMA, MMA, 8 epilogue warps (two per TMEM lane quarter)
constexpr int kGemmEpiThreads = kGemmThreads - 64;

struct GemmParams {
    const int* num_tiles;   // device: number of valid 128-row tiles
    const int* tile_group;  // [tiles] group (expert) of each tile
    const int* tile_row0;   // [tiles] first row of each tile
    const int* group_end;   // [groups] one past the last row of each group
    int K;                  // reduction length (multiple of 64)
    void* C;                // output rows (same row index space as A)
    int ldc;                // elements per output row
    int ntn = 1;            // N tiles per M tile (set by the launcher)
};

template <int BN, int EPI>
constexpr int gemm_stage_bytes() {
    return 128 * 128 + ((EPI == kEpiSwiGLU) ? 2 : 1) * 64 * 2 * BN;
}
template <int BN, int EPI>
constexpr int gemm_stages() {
    return (192 * 1024) / gemm_stage_bytes<BN, EPI>() > 8 ? 8 : (192 * 1024) / gemm_stage_bytes<BN, EPI>();
}
template <int BN, int EPI>
constexpr int gemm_smem() {
    return gemm_stages<BN, EPI>() * gemm_stage_bytes<BN, EPI>() + 512;
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.f + __expf(-x)); }

template <int BN, int EPI>
__global__ void moe_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                         const __grid_constant__ CUtensorMap tmB1, GemmParams p);
template <int NE>
__global__ void moe_route(const float* __restrict__ logits, int T, int E, int K, int* __restrict__ ids,
                          float* __restrict__ gates, float* __restrict__ probs, int* __restrict__ counts,
                          float* __restrict__ prob_colsum);
__global__ void moe_plan(const int* __restrict__ counts, const float* __restrict__ prob_colsum, int nrb, int T,
                         int E, int K, int* __restrict__ offsets, int* __restrict__ group_end,
                         int* __restrict__ tile_group, int* __restrict__ tile_row0,
                         int* __restrict__ num_tiles, float* __restrict__ aux);
__global__ void moe_block_counts(const int* __restrict__ ids, int T, int E, int K, int* __restrict__ blk_cnt);
__global__ void moe_block_scan(const int* __restrict__ blk_cnt, const int* __restrict__ offsets, int nblk,
                               int E, int* __restrict__ blk_base);
template <int KM>
__global__ void moe_assign(const int* __restrict__ ids, int T, int E, int K, const int* __restrict__ blk_base,
                           int* __restrict__ slot_pos, int* __restrict__ perm_token);
__global__ void moe_scatter(const uint4* __restrict__ x, const int* __restrict__ slot_pos, int T, int K,
                            int row_vec, uint4* __restrict__ x_perm);
template <int KM>
__global__ void moe_combine(const __nv_bfloat16* __restrict__ y_perm, const int* __restrict__ slot_pos,
                            const float* __restrict__ gates, int T, int K, int hidden, void* __restrict__ y,
                            int y_f32);

}  // namespace lmoe_dev
