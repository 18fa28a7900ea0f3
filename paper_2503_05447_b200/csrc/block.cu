// block.cu -- one Linear-MoE block on sm_100a, the layer unit of "LSM-layer tokens/s".
//
// Restates Block (/root/reference/proj/include/lmoe/model.hpp:284-304) as the hybrid model
// runs it (model_forward, model.hpp:374-405; hybrid_sp_forward, parallel.hpp:477-506):
//     h  = rms_norm(x, norm_mixer)                         (tensor.hpp:1164-1170)
//     x += mixer(h)     L: LsmMixer::forward (model.hpp:232-246) / lsm_mixer_sp
//                       N: AttentionMixer::forward (model.hpp:266-278) / attn_mixer_sp
//     h2 = rms_norm(x, norm_moe)
//     x += MoeLayer::forward(h2).first                     (moe.hpp:133-149)
// with the residual stream x in fp32 and every matmul a bf16 tcgen05 GEMM:
//   [Wq | Wk | Wv (| W_gate_a)] is ONE GEMM; the LSM / attention kernels read q, k, v (a_pre)
//   as row-strided views of its output through their TMA descriptors (no split copies);
//   Mamba2's b_pre = h W_gate_b is an fp32-output GEMM; o W_o is one GEMM; the residual add
//   and the next RMSNorm are one fused kernel.
#include <algorithm>

#include "common.h"
#include "internal.h"
#include "ptx.cuh"

namespace lmoe_dev {

// x[row] += delta[row] (bf16 or fp32, nullable); out[row] = x * rsqrt(mean(x^2) + eps) * w
// (bf16, nullable).  One warp per row.
__global__ void block_add_rmsnorm(float* __restrict__ x, const void* __restrict__ delta, int delta_f32,
                                  const float* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out,
                                  int rows, int hidden) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float* xr = x + (size_t)row * hidden;
    float ss = 0.f;
    for (int c = lane * 4; c < hidden; c += 128) {
        float4 v = *reinterpret_cast<float4*>(xr + c);
        if (delta) {
            if (delta_f32) {
                const float4 d = *reinterpret_cast<const float4*>(static_cast<const float*>(delta) + (size_t)row * hidden + c);
                v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w;
            } else {
                const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(delta) + (size_t)row * hidden + c);
                const float2 a = unpack_bf16(u.x), b = unpack_bf16(u.y);
                v.x += a.x; v.y += a.y; v.z += b.x; v.w += b.y;
            }
            *reinterpret_cast<float4*>(xr + c) = v;
        }
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    if (!out) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xFFFFFFFFu, ss, o);
    const float inv = rsqrtf(ss / hidden + eps);
    for (int c = lane * 4; c < hidden; c += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + c);
        const float4 g = *reinterpret_cast<const float4*>(w + c);
        uint2 u;
        u.x = pack_bf16(v.x * inv * g.x, v.y * inv * g.y);
        u.y = pack_bf16(v.z * inv * g.z, v.w * inv * g.w);
        *reinterpret_cast<uint2*>(out + (size_t)row * hidden + c) = u;
    }
}

// dst[t, h] = src[t, h] for h < H (src rows are 64 wide): Mamba2 b_pre from the padded GEMM
__global__ void block_compact_cols(const float* __restrict__ src, float* __restrict__ dst, int rows, int H) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)rows * H) return;
    dst[i] = src[(i / H) * 64 + i % H];
}

// x[t] = emb[tok[t]] + pos[pos0 + t % n]  (model.hpp:385-386, hybrid_sp_forward :487-490)
__global__ void block_embed(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ emb,
                            const __nv_bfloat16* __restrict__ pos, int pos0, int n, int rows, int hidden,
                            float* __restrict__ x) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)rows * hidden) return;
    const int t = (int)(i / hidden), c = (int)(i % hidden);
    x[i] = __bfloat162float(emb[(size_t)tok[t] * hidden + c]) +
           __bfloat162float(pos[(size_t)(pos0 + t % n) * hidden + c]);
}

}  // namespace lmoe_dev

namespace lmoe_host {

struct BlockWs {
    size_t h, qkv, bg, bpre, o, mixed, y, tiles, mixer, moe, total;
    size_t mixer_bytes, moe_bytes;
    int nc;  // QKV(+gate) GEMM output columns
};

static int device_decay(int inst) {
    switch (inst) {
        case LMOE_BLA: case LMOE_REBASED: return 0;
        case LMOE_LIGHTNING: case LMOE_RETNET: return 1;
        case LMOE_MAMBA2: return 2;
        case LMOE_GLA: case LMOE_HGRN2: case LMOE_RWKV6: return 3;
        default: return -1;
    }
}

static void block_validate(const lmoe_block_desc* d) {
    if (!d) throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: null descriptor");
    if (d->kind != 'L' && d->kind != 'N')
        throw Error(LMOE_ERR_ARG, std::string("ModelConfig: invalid pattern char '") + (char)d->kind + "' (want L or N)");
    if (d->heads < 1 || d->hidden % d->heads != 0)
        throw Error(LMOE_ERR_ARG, "ModelConfig: hidden must be divisible by num_heads");
    if (d->hidden / d->heads != 128)
        throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_block_fwd: head_dim must be 128 (bf16 kernels)");
    if (d->hidden % 256 != 0 || d->ffn_dim % 128 != 0)
        throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_block_fwd: need hidden % 256 == 0 and ffn_dim % 128 == 0");
    if (d->kind == 'L' && device_decay(d->lsm.instance) < 0)
        throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_block_fwd: LSM instance has no device kernel in this build");
}

static BlockWs plan_block(const lmoe_block_desc* d, int B, int N, int N_total, int world) {
    BlockWs w{};
    const size_t T = (size_t)B * N, hid = d->hidden;
    const bool vec = d->kind == 'L' && device_decay(d->lsm.instance) == 3;
    w.nc = (int)(hid * (vec ? 4 : 3));
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    w.h = take(T * hid * 2);
    w.qkv = take(T * w.nc * 2);
    w.bg = take(T * 64 * 4);
    w.bpre = take(T * d->heads * 4);
    w.o = take(T * hid * 2);
    w.mixed = take(T * hid * 2);
    w.y = take(T * hid * 4);
    w.tiles = take(dense_gemm_ws((int)T));
    w.mixer_bytes = d->kind == 'L' ? lsm_mixer_ws(&d->lsm, B, N, d->heads, 128, world)
                                   : sp_attn_ws(B, N_total, d->heads, 128, world);
    w.mixer = take(w.mixer_bytes);
    w.moe_bytes = d->num_experts == 0 ? 0 : lmoe_moe_workspace_size((int)T, d->hidden, d->ffn_dim, d->num_experts, d->top_k);
    w.moe = take(w.moe_bytes);
    w.total = off;
    return w;
}

static void add_rmsnorm(float* x, const void* delta, bool delta_f32, const float* w, float eps, void* out,
                        int rows, int hidden, cudaStream_t st) {
    lmoe_dev::block_add_rmsnorm<<<(rows + 7) / 8, 256, 0, st>>>(x, delta, delta_f32 ? 1 : 0, w, eps,
                                                               static_cast<__nv_bfloat16*>(out), rows, hidden);
    LMOE_CUDA_CHECK(cudaGetLastError());
    ++g_launch_count;
}

}  // namespace lmoe_host

using namespace lmoe_host;

extern "C" size_t lmoe_block_workspace_size(const lmoe_block_desc* desc, int B, int N_local, int N_total,
                                            int world) {
    if (!desc || B < 1 || N_local < 1 || world < 1) return 0;
    return plan_block(desc, B, N_local, N_total, world).total;
}

namespace lmoe_host {
// One block; cu != nullptr: packed documents (B = 1, N_local = T), the mixer per document.
static void block_core(const lmoe_block_desc* d, const lmoe_block_weights* wt, int B, int N_local, int N_total,
                       float* x, float* aux, void* nccl_comm, int rank, int world, const BlockWs& w,
                       void* workspace, lmoe_stream_t stream, const int* cu, int n_docs) {
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int T = B * N_local, hid = d->hidden, H = d->heads, D = 128;
        void* h = ws + w.h;
        uint8_t* qkv = ws + w.qkv;
        // h = rms_norm(x, norm_mixer)
        add_rmsnorm(x, nullptr, false, wt->norm_mixer, d->norm_eps, h, T, hid, st);
        // [q | k | v (| a_pre)] = h [Wq | Wk | Wv (| W_gate_a)]
        dense_gemm(h, T, hid, hid, wt->w_qkv, w.nc, qkv, w.nc, false, ws + w.tiles, st);
        void* o = ws + w.o;
        const size_t col = (size_t)hid * 2;  // byte offset of the next column block
        if (d->kind == 'L') {
            const int mode = device_decay(d->lsm.instance);
            const float* b_pre = nullptr;
            if (mode == 2) {  // Mamba2: b_pre = h W_gate_b (fp32), heads padded to 64 columns
                if (!wt->w_gate_b || !wt->a_raw) throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: Mamba2 needs w_gate_b and a_raw");
                if (H > 64) throw Error(LMOE_ERR_UNSUPPORTED, "lmoe_block_fwd: Mamba2 with more than 64 heads");
                dense_gemm(h, T, hid, hid, wt->w_gate_b, 64, ws + w.bg, 64, true, ws + w.tiles, st);
                lmoe_dev::block_compact_cols<<<(unsigned)(((size_t)T * H + 255) / 256), 256, 0, st>>>(
                    reinterpret_cast<const float*>(ws + w.bg), reinterpret_cast<float*>(ws + w.bpre), T, H);
                LMOE_CUDA_CHECK(cudaGetLastError());
                ++g_launch_count;
                b_pre = reinterpret_cast<const float*>(ws + w.bpre);
            }
            if (cu) {
                for (int i = 0; i < n_docs; ++i) {
                    const size_t r0 = (size_t)cu[i];
                    uint8_t* qd = qkv + r0 * w.nc * 2;
                    lsm_mixer_core(&d->lsm, 1, cu[i + 1] - cu[i], H, D, LMOE_BF16, qd, qd + col, qd + 2 * col,
                                   mode == 3 ? qd + 3 * col : nullptr, w.nc, b_pre ? b_pre + r0 * H : nullptr,
                                   wt->a_raw, static_cast<uint8_t*>(o) + r0 * hid * 2, nullptr, 0, 1, ws + w.mixer,
                                   w.mixer_bytes, st);
                }
            } else {
                lsm_mixer_core(&d->lsm, B, N_local, H, D, LMOE_BF16, qkv, qkv + col, qkv + 2 * col,
                               mode == 3 ? qkv + 3 * col : nullptr, w.nc, b_pre, wt->a_raw, o, nccl_comm, rank,
                               world, ws + w.mixer, w.mixer_bytes, st);
            }
        } else if (cu) {
            for (int i = 0; i < n_docs; ++i) {
                const size_t r0 = (size_t)cu[i];
                const int len = cu[i + 1] - cu[i];
                uint8_t* qd = qkv + r0 * w.nc * 2;
                attn_core(1, len, len, H, D, qd, qd + col, qd + 2 * col, w.nc, static_cast<uint8_t*>(o) + r0 * hid * 2,
                          0, st);
            }
        } else if (world == 1 && !nccl_comm) {
            attn_core(B, N_local, N_local, H, D, qkv, qkv + col, qkv + 2 * col, w.nc, o, 0, st);
        } else {
            sp_attn_core(B, N_total, H, D, qkv, qkv + col, qkv + 2 * col, w.nc, o, nccl_comm, rank, world,
                         ws + w.mixer, w.mixer_bytes, st);
        }
        // x += o W_o ; h2 = rms_norm(x, norm_moe)
        dense_gemm(o, T, hid, hid, wt->wo, hid, ws + w.mixed, hid, false, ws + w.tiles, st);
        if (d->num_experts == 0) {  // mixer-only LSM layer (SURVEY 8(d) "LSM-layer tokens/s"): x += o W_o
            add_rmsnorm(x, ws + w.mixed, false, nullptr, 0.f, nullptr, T, hid, st);
            return;
        }
        add_rmsnorm(x, ws + w.mixed, false, wt->norm_moe, d->norm_eps, h, T, hid, st);
        // x += MoE(h2)
        const int rc = lmoe_moe_forward(T, hid, d->ffn_dim, d->num_experts, d->top_k, h, wt->router, wt->w_gate,
                                        wt->w_up, wt->w_down, ws + w.y, 1, aux, nullptr, nullptr, nullptr,
                                        ws + w.moe, w.moe_bytes, stream);
        if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
        add_rmsnorm(x, ws + w.y, true, nullptr, 0.f, nullptr, T, hid, st);
}
}  // namespace lmoe_host

extern "C" int lmoe_block_fwd(const lmoe_block_desc* d, const lmoe_block_weights* wt, int B, int N_local,
                              int N_total, float* x, float* aux, void* nccl_comm, int rank, int world,
                              void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        block_validate(d);
        if (!wt || !x) throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: null weights or activations");
        if (world < 1 || rank < 0 || rank >= world) throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: bad rank");
        if (world > 1 && !nccl_comm) throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: null communicator");
        const BlockWs w = plan_block(d, B, N_local, N_total, world);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: workspace too small (need " + std::to_string(w.total) + " bytes)");
        block_core(d, wt, B, N_local, N_total, x, aux, nccl_comm, rank, world, w, workspace, stream, nullptr, 0);
    });
}

namespace lmoe_host {
static BlockWs plan_block_varlen(const lmoe_block_desc* d, int T, const int* cu, int n_docs) {
    BlockWs w = plan_block(d, 1, T, T, 1);
    size_t mix = 0;  // the mixer workspace of the longest document (attention needs none)
    for (int i = 0; i < n_docs; ++i)
        if (d->kind == 'L') mix = std::max(mix, lsm_mixer_ws(&d->lsm, 1, cu[i + 1] - cu[i], d->heads, 128, 1));
    if (mix > w.mixer_bytes) {
        w.total += align_up(mix - w.mixer_bytes, 256);
        w.moe += align_up(mix - w.mixer_bytes, 256);
        w.mixer_bytes = mix;
    }
    return w;
}
}  // namespace lmoe_host

extern "C" size_t lmoe_block_varlen_workspace_size(const lmoe_block_desc* desc, int T, const int* cu_seqlens,
                                                   int n_docs) {
    if (!desc || T < 1 || !cu_seqlens || n_docs < 1) return 0;
    return plan_block_varlen(desc, T, cu_seqlens, n_docs).total;
}

extern "C" int lmoe_block_fwd_varlen(const lmoe_block_desc* d, const lmoe_block_weights* wt, int T,
                                     const int* cu_seqlens, int n_docs, float* x, float* aux, void* workspace,
                                     size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        block_validate(d);
        if (!wt || !x) throw Error(LMOE_ERR_ARG, "lmoe_block_fwd: null weights or activations");
        if (!cu_seqlens || n_docs < 1 || cu_seqlens[0] != 0 || cu_seqlens[n_docs] != T)
            throw Error(LMOE_ERR_ARG, "PackedBatch: boundaries must run from 0 to total length");
        for (int i = 1; i <= n_docs; ++i)
            if (cu_seqlens[i] <= cu_seqlens[i - 1])
                throw Error(LMOE_ERR_ARG, "PackedBatch: boundaries must be strictly ascending");
        const BlockWs w = plan_block_varlen(d, T, cu_seqlens, n_docs);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_block_fwd_varlen: workspace too small (need " + std::to_string(w.total) +
                                          " bytes)");
        block_core(d, wt, 1, T, T, x, aux, nullptr, 0, 1, w, workspace, stream, cu_seqlens, n_docs);
    });
}

// x[t] = embedding[tokens[t]] + pos_embedding[pos0 + t % n]  (fp32 residual stream)
extern "C" int lmoe_embed(const int* tokens, int rows, int n, int pos0, int hidden, const void* embedding,
                          const void* pos_embedding, float* x, lmoe_stream_t stream) {
    return guarded([&]() {
        if (!tokens || !embedding || !pos_embedding || !x || rows < 1 || n < 1)
            throw Error(LMOE_ERR_ARG, "lmoe_embed: bad arguments");
        lmoe_dev::block_embed<<<(unsigned)(((size_t)rows * hidden + 255) / 256), 256, 0,
                                reinterpret_cast<cudaStream_t>(stream)>>>(
            tokens, static_cast<const __nv_bfloat16*>(embedding), static_cast<const __nv_bfloat16*>(pos_embedding),
            pos0, n, rows, hidden, x);
        LMOE_CUDA_CHECK(cudaGetLastError());
        ++g_launch_count;
    });
}

// out = rms_norm(x, w, eps) in bf16 (the final norm before the LM head, model.hpp:402)
extern "C" int lmoe_rmsnorm(const float* x, int rows, int hidden, const float* w, float eps, void* out,
                            lmoe_stream_t stream) {
    return guarded([&]() {
        if (!x || !w || !out || hidden % 128 != 0) throw Error(LMOE_ERR_ARG, "lmoe_rmsnorm: bad arguments");
        add_rmsnorm(const_cast<float*>(x), nullptr, false, w, eps, out, rows, hidden,
                    reinterpret_cast<cudaStream_t>(stream));
    });
}
