// moe_host.cu -- C-ABI of the Linear-MoE expert layer (moe.hpp) on sm_100a.
#include <algorithm>

#include "common.h"
#include "internal.h"
#include "moe_kernels.cu"  // kernels and their launches in one translation unit

namespace lmoe_host {

// blocks of the routing kernel (a warp per token, 8 per block, at most 8 blocks per SM)
static int route_blocks(int T) { return std::min((T + 7) / 8, num_sms() * 8); }

struct MoePlanWs {
    size_t logits, ids, gates, colsum, counts, offsets, group_end, tile_group, tile_row0, num_tiles,
        aux, blk_cnt, blk_base, slot_pos, perm_token, x_perm, h, y_perm, dense_tiles, total;
    int max_tiles, nblk;
};

static MoePlanWs plan_moe(int T, int hidden, int ffn, int E, int K) {
    MoePlanWs w{};
    const size_t rows = (size_t)T * K;
    w.max_tiles = (int)((rows + 127) / 128 + E);
    w.nblk = (T + 255) / 256;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    w.logits = take((size_t)T * E * 4);
    w.ids = take(rows * 4);
    w.gates = take(rows * 4);
    w.colsum = take((size_t)route_blocks(T) * E * 4);  // per route block partial column sums
    w.counts = take((size_t)E * 4);
    w.offsets = take((size_t)(E + 1) * 4);
    w.group_end = take((size_t)E * 4);
    w.tile_group = take((size_t)w.max_tiles * 4);
    w.tile_row0 = take((size_t)w.max_tiles * 4);
    w.num_tiles = take(4);
    w.aux = take(4);
    w.blk_cnt = take((size_t)w.nblk * E * 4);
    w.blk_base = take((size_t)w.nblk * E * 4);
    w.slot_pos = take(rows * 4);
    w.perm_token = take(rows * 4);
    w.x_perm = take(rows * hidden * 2);
    w.h = take(rows * ffn * 2);
    w.y_perm = take(rows * hidden * 2);
    w.dense_tiles = take((size_t)((T + 127) / 128 + 2) * 3 * 4 + 64);
    w.total = off;
    return w;
}

template <int BN, int EPI>
static void launch_gemm(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                        const lmoe_dev::GemmParams& gp, int max_tiles, int ntiles_n, cudaStream_t st) {
    LMOE_CUDA_CHECK(lmoe_dev::ensure_smem((const void*)lmoe_dev::moe_gemm<BN, EPI>, lmoe_dev::gemm_smem<BN, EPI>()));
    // persistent: one CTA per SM (or fewer when the tile list is short) walks the tile list
    lmoe_dev::GemmParams g = gp;
    g.ntn = ntiles_n;
    const long long upper = (long long)max_tiles * ntiles_n;
    const int grid = (int)std::max<long long>(1, std::min<long long>(num_sms(), upper));
    lmoe_dev::moe_gemm<BN, EPI><<<grid, lmoe_dev::kGemmThreads, lmoe_dev::gemm_smem<BN, EPI>(), st>>>(a, b0, b1, g);
    LMOE_CUDA_CHECK(cudaGetLastError());
    ++g_launch_count;
}

// single-group tile list for a dense [rows x K] GEMM (the router)
__global__ void dense_plan(int rows, int* num_tiles, int* tile_group, int* tile_row0, int* group_end) {
    const int n = (rows + 127) / 128;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { tile_group[i] = 0; tile_row0[i] = i * 128; }
    if (threadIdx.x == 0) { *num_tiles = n; group_end[0] = rows; }
}

// Router logits on CUDA cores for expert counts that are not a multiple of 64.
__global__ void router_small(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr,
                             int T, int hidden, int E, float* __restrict__ logits) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * E) return;
    const int t = i / E, e = i % E;
    float acc = 0.f;
    for (int c = 0; c < hidden; ++c)
        acc += __bfloat162float(x[(size_t)t * hidden + c]) * __bfloat162float(wr[(size_t)c * E + e]);
    logits[i] = acc;
}

static void route_core(const float* logits, int T, int E, int K, int* ids, float* gates, float* probs,
                       int* counts, float* colsum, cudaStream_t st) {
    LMOE_CUDA_CHECK(cudaMemsetAsync(counts, 0, E * 4, st));
    const dim3 grid(route_blocks(T));
    if (E <= 32) lmoe_dev::moe_route<1><<<grid, 256, 0, st>>>(logits, T, E, K, ids, gates, probs, counts, colsum);
    else if (E <= 64) lmoe_dev::moe_route<2><<<grid, 256, 0, st>>>(logits, T, E, K, ids, gates, probs, counts, colsum);
    else if (E <= 128) lmoe_dev::moe_route<4><<<grid, 256, 0, st>>>(logits, T, E, K, ids, gates, probs, counts, colsum);
    else lmoe_dev::moe_route<8><<<grid, 256, 0, st>>>(logits, T, E, K, ids, gates, probs, counts, colsum);
    LMOE_CUDA_CHECK(cudaGetLastError());
    ++g_launch_count;
}

static void check_route_args(int T, int E, int K) {
    if (K < 1 || K > E) throw Error(LMOE_ERR_ARG, "route: bad top_k");
    if (E > lmoe_dev::kMoeMaxE || K > lmoe_dev::kMoeMaxK)
        throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_moe: device routing supports E <= 256, top_k <= 32");
    if (T < 1) throw Error(LMOE_ERR_ARG, "lmoe_moe: need T >= 1");
}

size_t dense_gemm_ws(int M) { return align_up((size_t)((M + 127) / 128 + 2) * 3 * 4 + 64, 256); }

// Dense projection on the grouped tcgen05 GEMM with a single group (the LsmMixer /
// AttentionMixer matmuls, model.hpp:232-246, 266-278, and the LM head).
void dense_gemm(const void* A, int M, int K, int lda, const void* W, int N, void* C, int ldc, bool out_f32,
                void* ws, cudaStream_t st) {
    if (M < 1 || K < 64 || K % 64 != 0) throw Error(LMOE_ERR_UNSUPPORTED, "dense GEMM: need K % 64 == 0");
    if (out_f32 ? N % 64 != 0 : N % 128 != 0)
        throw Error(LMOE_ERR_UNSUPPORTED, "dense GEMM: need N % 128 == 0 (bf16 out) or N % 64 == 0 (fp32 out)");
    constexpr CUtensorMapDataType BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    int* dt = static_cast<int*>(ws);
    const int ntile = (M + 127) / 128;
    int* dgroup = dt + 1;
    int* drow0 = dgroup + ntile + 1;
    int* dend = drow0 + ntile + 1;
    dense_plan<<<1, 256, 0, st>>>(M, dt, dgroup, drow0, dend);
    LMOE_CUDA_CHECK(cudaGetLastError());
    ++g_launch_count;
    lmoe_dev::GemmParams gp{dt, dgroup, drow0, dend, K, C, ldc};
    const CUtensorMap ta = make_tmap_2d(A, BF, 2, K, M, lda, 64, 128);
    const CUtensorMap tb = make_tmap_3d(W, BF, 2, N, K, 1, 64, 64);
    if (out_f32) launch_gemm<64, lmoe_dev::kEpiF32>(ta, tb, tb, gp, ntile, N / 64, st);
    else if (N % 256 == 0 && (size_t)ntile * (N / 256) >= (size_t)num_sms()) launch_gemm<256, lmoe_dev::kEpiBF16>(ta, tb, tb, gp, ntile, N / 256, st);
    else launch_gemm<128, lmoe_dev::kEpiBF16>(ta, tb, tb, gp, ntile, N / 128, st);
}

}  // namespace lmoe_host

using namespace lmoe_host;

extern "C" size_t lmoe_moe_workspace_size(int T, int hidden, int ffn, int E, int top_k) {
    if (T < 1 || E < 1 || top_k < 1) return 0;
    return plan_moe(T, hidden, ffn, E, top_k).total;
}

// route (moe.hpp:58-85) + load_balance_loss (moe.hpp:90-103) on given fp32 logits [T, E].
// ids [T,k] ascending, gates [T,k] renormalised over the selection (compact form of the
// reference's dense (T x E) gates), probs [T,E] full softmax (optional), counts [E].
extern "C" int lmoe_moe_route(const float* logits, int T, int E, int top_k, int* ids, float* gates,
                              float* probs, int* counts, float* aux, void* workspace,
                              size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        check_route_args(T, E, top_k);
        const MoePlanWs w = plan_moe(T, 64, 64, E, top_k);
        if (!workspace || workspace_bytes < w.total) throw Error(LMOE_ERR_ARG, "lmoe_moe_route: workspace too small");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        float* colsum = reinterpret_cast<float*>(ws + w.colsum);
        route_core(logits, T, E, top_k, ids, gates, probs, counts, colsum, st);
        lmoe_dev::moe_plan<<<1, 256, 0, st>>>(counts, colsum, route_blocks(T), T, E, top_k,
                                             reinterpret_cast<int*>(ws + w.offsets),
                                             reinterpret_cast<int*>(ws + w.group_end),
                                             reinterpret_cast<int*>(ws + w.tile_group),
                                             reinterpret_cast<int*>(ws + w.tile_row0),
                                             reinterpret_cast<int*>(ws + w.num_tiles),
                                             aux ? aux : reinterpret_cast<float*>(ws + w.aux));
        LMOE_CUDA_CHECK(cudaGetLastError());
        ++g_launch_count;
    });
}

// MoeLayer::forward (moe.hpp:133-149): router GEMM, route, stable dispatch, grouped SwiGLU
// experts, combine, aux loss.  x [T,hidden] bf16; w_router [hidden,E] bf16;
// w_gate, w_up [E,hidden,ffn] bf16; w_down [E,ffn,hidden] bf16 (reference layouts,
// moe.hpp:31-33, experts stacked); y [T,hidden] bf16 (y_f32 = 0) or fp32 (y_f32 = 1).
extern "C" int lmoe_moe_forward(int T, int hidden, int ffn, int E, int top_k, const void* x,
                                const void* w_router, const void* w_gate, const void* w_up,
                                const void* w_down, void* y, int y_f32, float* aux,
                                float* logits_out, int* ids_out, float* gates_out, void* workspace,
                                size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        check_route_args(T, E, top_k);
        if (hidden % 256 != 0 || ffn % 128 != 0)
            throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_moe_forward: needs hidden % 256 == 0 and ffn % 128 == 0");
        const MoePlanWs w = plan_moe(T, hidden, ffn, E, top_k);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_moe_forward: workspace too small (need " + std::to_string(w.total) + ")");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        auto P = [&](size_t off) { return reinterpret_cast<int*>(ws + off); };
        float* logits = logits_out ? logits_out : reinterpret_cast<float*>(ws + w.logits);
        int* ids = ids_out ? ids_out : P(w.ids);
        float* gates = gates_out ? gates_out : reinterpret_cast<float*>(ws + w.gates);
        float* colsum = reinterpret_cast<float*>(ws + w.colsum);
        const size_t rows = (size_t)T * top_k;
        const CUtensorMapDataType BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;

        // 1. router logits = x W_r  (moe.hpp:136)
        if (E % 64 == 0) {
            int* dt = P(w.dense_tiles);
            const int ntile = (T + 127) / 128;
            int* dgroup = dt + 1;
            int* drow0 = dgroup + ntile + 1;
            int* dend = drow0 + ntile + 1;
            dense_plan<<<1, 256, 0, st>>>(T, dt, dgroup, drow0, dend);
            LMOE_CUDA_CHECK(cudaGetLastError());
            ++g_launch_count;
            lmoe_dev::GemmParams gp{dt, dgroup, drow0, dend, hidden, logits, E};
            const CUtensorMap ta = make_tmap_2d(x, BF, 2, hidden, T, hidden, 64, 128);
            const CUtensorMap tb = make_tmap_3d(w_router, BF, 2, E, hidden, 1, 64, 64);
            launch_gemm<64, lmoe_dev::kEpiF32>(ta, tb, tb, gp, ntile, E / 64, st);
        } else {
            router_small<<<(T * E + 255) / 256, 256, 0, st>>>(
                static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w_router), T, hidden, E, logits);
            LMOE_CUDA_CHECK(cudaGetLastError());
            ++g_launch_count;
        }
        // 2. route + counts + probability column sums
        route_core(logits, T, E, top_k, ids, gates, nullptr, P(w.counts), colsum, st);
        // 3. offsets, GEMM tile list, aux loss
        lmoe_dev::moe_plan<<<1, 256, 0, st>>>(P(w.counts), colsum, route_blocks(T), T, E, top_k, P(w.offsets), P(w.group_end),
                                             P(w.tile_group), P(w.tile_row0), P(w.num_tiles),
                                             aux ? aux : reinterpret_cast<float*>(ws + w.aux));
        // 4. stable dispatch positions (tokens ascending within each expert)
        lmoe_dev::moe_block_counts<<<w.nblk, 256, 0, st>>>(ids, T, E, top_k, P(w.blk_cnt));
        lmoe_dev::moe_block_scan<<<E, 256, 0, st>>>(P(w.blk_cnt), P(w.offsets), w.nblk, E, P(w.blk_base));
        if (top_k <= 8) lmoe_dev::moe_assign<8><<<w.nblk, 256, 0, st>>>(ids, T, E, top_k, P(w.blk_base), P(w.slot_pos), P(w.perm_token));
        else lmoe_dev::moe_assign<32><<<w.nblk, 256, 0, st>>>(ids, T, E, top_k, P(w.blk_base), P(w.slot_pos), P(w.perm_token));
        // 5. permute rows: each token row read once, written to its top_k dispatch rows
        lmoe_dev::moe_scatter<<<(T + 7) / 8, 256, 0, st>>>(static_cast<const uint4*>(x), P(w.slot_pos), T, top_k,
                                                          hidden / 8, reinterpret_cast<uint4*>(ws + w.x_perm));
        LMOE_CUDA_CHECK(cudaGetLastError());
        g_launch_count += 5;
        // 6. H = silu(Xp Wg) * (Xp Wu)   (grouped, per-expert B operands)
        {
            lmoe_dev::GemmParams gp{P(w.num_tiles), P(w.tile_group), P(w.tile_row0), P(w.group_end), hidden,
                                    ws + w.h, ffn};
            const CUtensorMap ta = make_tmap_2d(ws + w.x_perm, BF, 2, hidden, rows, hidden, 64, 128);
            const CUtensorMap tg = make_tmap_3d(w_gate, BF, 2, ffn, hidden, E, 64, 64);
            const CUtensorMap tu = make_tmap_3d(w_up, BF, 2, ffn, hidden, E, 64, 64);
            launch_gemm<128, lmoe_dev::kEpiSwiGLU>(ta, tg, tu, gp, w.max_tiles, ffn / 128, st);
        }
        // 7. Y = H Wd
        {
            lmoe_dev::GemmParams gp{P(w.num_tiles), P(w.tile_group), P(w.tile_row0), P(w.group_end), ffn,
                                    ws + w.y_perm, hidden};
            const CUtensorMap ta = make_tmap_2d(ws + w.h, BF, 2, ffn, rows, ffn, 64, 128);
            const CUtensorMap td = make_tmap_3d(w_down, BF, 2, hidden, ffn, E, 64, 64);
            launch_gemm<256, lmoe_dev::kEpiBF16>(ta, td, td, gp, w.max_tiles, hidden / 256, st);
        }
        // 8. combine in ascending expert order
        if (top_k <= 8)
            lmoe_dev::moe_combine<8><<<(T + 7) / 8, 256, 0, st>>>(
                reinterpret_cast<const __nv_bfloat16*>(ws + w.y_perm), P(w.slot_pos), gates, T, top_k, hidden, y, y_f32);
        else
            lmoe_dev::moe_combine<32><<<(T + 7) / 8, 256, 0, st>>>(
                reinterpret_cast<const __nv_bfloat16*>(ws + w.y_perm), P(w.slot_pos), gates, T, top_k, hidden, y, y_f32);
        LMOE_CUDA_CHECK(cudaGetLastError());
        ++g_launch_count;
    });
}

// Grouped-GEMM rows of the last forward for inspection (tests): slot positions [T,k] and
// the token of every permuted row [T*k].
extern "C" int lmoe_moe_dispatch_read(int T, int hidden, int ffn, int E, int top_k, const void* workspace,
                                      int* slot_pos, int* perm_token, int* offsets, lmoe_stream_t stream) {
    return guarded([&]() {
        const MoePlanWs w = plan_moe(T, hidden, ffn, E, top_k);
        const uint8_t* ws = static_cast<const uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const size_t rows = (size_t)T * top_k;
        if (slot_pos) LMOE_CUDA_CHECK(cudaMemcpyAsync(slot_pos, ws + w.slot_pos, rows * 4, cudaMemcpyDeviceToDevice, st));
        if (perm_token) LMOE_CUDA_CHECK(cudaMemcpyAsync(perm_token, ws + w.perm_token, rows * 4, cudaMemcpyDeviceToDevice, st));
        if (offsets) LMOE_CUDA_CHECK(cudaMemcpyAsync(offsets, ws + w.offsets, (E + 1) * 4, cudaMemcpyDeviceToDevice, st));
    });
}

extern "C" size_t lmoe_gemm_workspace_size(int M) { return M < 1 ? 0 : dense_gemm_ws(M); }

// C[M, N] = A[M, K] W[K, N]: bf16 operands (A rows lda elements apart, W row-major as the
// reference's (in x out) weights), fp32 accumulate, C bf16 or fp32 (out_f32) with row stride ldc.
extern "C" int lmoe_gemm(const void* A, int M, int K, int lda, const void* W, int N, void* C, int ldc,
                         int out_f32, void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        if (!A || !W || !C) throw Error(LMOE_ERR_ARG, "lmoe_gemm: null tensor");
        if (!workspace || workspace_bytes < dense_gemm_ws(M)) throw Error(LMOE_ERR_ARG, "lmoe_gemm: workspace too small");
        dense_gemm(A, M, K, lda, W, N, C, ldc, out_f32 != 0, workspace, reinterpret_cast<cudaStream_t>(stream));
    });
}
