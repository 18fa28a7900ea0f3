// lmoe/cuda_tensor.hpp -- Tensor-level drop-in for the reference's hot-path entry points.
//
// For callers written against the reference headers (/root/reference/proj/include/lmoe,
// header-only C++20): the same argument types (lmoe::Tensor, LsmGates, LsmSpec, MemoryState,
// RoutingDecision, MoeLayer), the same results and the same std::runtime_error texts, computed
// on the B200 through liblmoe_cuda.so.  Include AFTER the reference headers are on the include
// path; the functions live in lmoe::cuda so both implementations can sit in one translation
// unit (a caller switches by qualifying the call):
//
//   reference                                            this header
//   lsm_forward_chunked(q,k,v,gates,spec,C,&fs)          lsm.hpp:668-670   lmoe::cuda::lsm_forward_chunked(same)
//   route(logits, top_k) -> RoutingDecision (dense)      moe.hpp:52-85     lmoe::cuda::route(same)
//   MoeLayer::forward(x) -> {y, aux}                     moe.hpp:133-149   lmoe::cuda::moe_forward(layer, x)
//   sp_lsm_masked_rank(RankGroup&, rank, q,k,v,g,spec)   parallel.hpp:303  lmoe::cuda::sp_lsm_masked_rank(comm, rank, world, q,k,v,g,spec)
//
// Bridge rules (all exact except the stated device precision):
//   * head dims are zero-padded to the kernel width (fp32 path D = 64 when d <= 64 and the
//     decay is not per-column; otherwise bf16 D = 128).  Zero columns of q, k, v leave every
//     output and state entry unchanged, so the padding is exact -- provided phi(0) = 0.  The
//     elu+1 map has phi(0) = 1, so with padding the bridge applies it on the host (in f64,
//     lsm.hpp feature map) and runs the device with the identity map.
//   * f64 / f32 Tensors are rounded to the device type (fp32 -> tf32 tensor cores, or bf16);
//     results are returned in the input Tensor's dtype.  North-star bounds: norm-relative
//     1e-3 (fp32 path) / 2e-2 (bf16 path) against the reference in f64.
//   * MoE: hidden is zero-padded to a multiple of 256 and ffn_dim to a multiple of 128
//     (zero rows / columns of the router and expert weights: exact); bf16 operands, fp32
//     accumulation and fp32 output.
//   * routing ids are bit-exact with the reference on the same fp32-representable logits.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "lmoe/cuda.hpp"
#include "lmoe/lsm.hpp"
#include "lmoe/moe.hpp"

namespace lmoe {
namespace cuda {
namespace bridge {

// RAII device buffer.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw Error(LMOE_ERR_CUDA, "device allocation failed");
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

inline void h2d(void* dst, const void* src, size_t bytes) {
    if (cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) throw Error(LMOE_ERR_CUDA, "H2D copy failed");
}
inline void d2h(void* dst, const void* src, size_t bytes) {
    if (cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) throw Error(LMOE_ERR_CUDA, "D2H copy failed");
}

// round-to-nearest-even fp32 -> bf16 bits (host side)
inline uint16_t to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)(u >> 16);  // inf / nan
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
inline float from_bf16(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// (rows x cols) Tensor -> row-major (rows x width) device-typed host image, zero-padded
inline std::vector<uint8_t> pack(const lmoe::Tensor& t, int rows, int cols, int width, bool bf16) {
    const size_t es = bf16 ? 2 : 4;
    std::vector<uint8_t> out((size_t)rows * width * es, 0);
    const std::vector<double>& d = t.data();
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const float f = (float)d[(size_t)r * cols + c];
            if (bf16) {
                const uint16_t b = to_bf16(f);
                std::memcpy(&out[((size_t)r * width + c) * 2], &b, 2);
            } else {
                std::memcpy(&out[((size_t)r * width + c) * 4], &f, 4);
            }
        }
    return out;
}

inline int decay_mode(lmoe::LsmInstance inst) {
    switch (decay_kind(inst)) {
        case lmoe::DecayKind::TokenVector: return 3;
        default: return 0;
    }
}

struct LsmPlan {
    int D;
    bool bf16;
    lmoe_dtype dt;
};
inline LsmPlan plan_for(const lmoe::LsmSpec& spec) {
    const int d = std::max(spec.d_k, spec.d_v);
    if (d <= 64 && decay_mode(spec.instance) != 3) return {64, false, LMOE_F32};
    if (d <= 128) return {128, true, LMOE_BF16};
    throw Error(LMOE_ERR_UNSUPPORTED, "lmoe::cuda: head dims above 128 are not supported by the device kernels");
}

inline lmoe_lsm_desc desc_for(const lmoe::LsmSpec& spec, int chunk_size) {
    lmoe_lsm_desc d{};
    d.instance = static_cast<int>(spec.instance);
    d.feature_map = static_cast<int>(spec.feature_map);
    d.use_normalizer = spec.use_normalizer ? 1 : 0;
    d.scalar_decay = (float)spec.scalar_decay;
    d.chunk_size = chunk_size;
    d.flags = LMOE_FLAG_CHECK;
    return d;
}

// The per-sequence inputs of one head on the device.
struct LsmDev {
    LsmPlan pl;
    int n;
    DevBuf q, k, v, o, a_pre, b_pre, a_raw, M, z;
    bool host_fmap = false;  // elu+1 applied here (padded columns must map to 0)
    LsmDev(const lmoe::Tensor& qm, const lmoe::Tensor& km, const lmoe::Tensor& vm, const lmoe::LsmGates& g, const lmoe::LsmSpec& spec)
        : pl(plan_for(spec)), n(qm.shape()[0]),
          q((size_t)n * pl.D * (pl.bf16 ? 2 : 4)), k((size_t)n * pl.D * (pl.bf16 ? 2 : 4)),
          v((size_t)n * pl.D * (pl.bf16 ? 2 : 4)), o((size_t)n * pl.D * (pl.bf16 ? 2 : 4)),
          a_pre(decay_mode(spec.instance) == 3 ? (size_t)n * pl.D * 2 : 0),
          b_pre(spec.instance == lmoe::LsmInstance::Mamba2 ? (size_t)n * 4 : 0),
          a_raw(spec.instance == lmoe::LsmInstance::Mamba2 ? 4 : 0), M((size_t)pl.D * pl.D * 4),
          z((size_t)pl.D * 4) {
        const int dk = spec.d_k, dv = spec.d_v;
        if (km.shape()[0] != n || vm.shape()[0] != n || qm.shape()[1] != dk || km.shape()[1] != dk ||
            vm.shape()[1] != dv)
            detail::shape_error("lsm_forward_chunked", qm.shape(), vm.shape());
        auto up = [&](DevBuf& b, const lmoe::Tensor& t, int cols) {
            const auto img = pack(t, n, cols, pl.D, pl.bf16);
            h2d(b.p, img.data(), img.size());
        };
        host_fmap = spec.feature_map == lmoe::FeatureMap::EluPlusOne && dk < pl.D;
        if (host_fmap) {
            auto phi = [&](const lmoe::Tensor& t) {
                std::vector<double> y(t.data());
                for (double& e : y) e = e > 0.0 ? e + 1.0 : std::exp(e);  // elu(x) + 1
                return lmoe::Tensor::from_data({n, dk}, std::move(y));
            };
            up(q, phi(qm), dk);
            up(k, phi(km), dk);
        } else {
            up(q, qm, dk);
            up(k, km, dk);
        }
        up(v, vm, dv);
        if (a_pre.p) {
            if (!g.a_pre.defined()) throw Error(LMOE_ERR_ARG, "lsm_forward_chunked: gates.a_pre required for this instance");
            const auto img = pack(g.a_pre, n, dk, pl.D, true);
            h2d(a_pre.p, img.data(), img.size());
        }
        if (b_pre.p) {
            if (!g.b_pre.defined()) throw Error(LMOE_ERR_ARG, "lsm_forward_chunked: gates.b_pre required for this instance");
            std::vector<float> bp(n);
            for (int t = 0; t < n; ++t) bp[t] = (float)g.b_pre.at(t);
            h2d(b_pre.p, bp.data(), bp.size() * 4);
            const float ar = (float)spec.mamba2_a_raw.at(0);
            h2d(a_raw.p, &ar, 4);
        }
    }
    lmoe::Tensor output(int dv, lmoe::DType dt) const {
        const size_t es = pl.bf16 ? 2 : 4;
        std::vector<uint8_t> img((size_t)n * pl.D * es);
        d2h(img.data(), o.p, img.size());
        std::vector<double> out((size_t)n * dv);
        for (int t = 0; t < n; ++t)
            for (int c = 0; c < dv; ++c) {
                const size_t i = (size_t)t * pl.D + c;
                if (pl.bf16) {
                    uint16_t b;
                    std::memcpy(&b, &img[i * 2], 2);
                    out[(size_t)t * dv + c] = from_bf16(b);
                } else {
                    float f;
                    std::memcpy(&f, &img[i * 4], 4);
                    out[(size_t)t * dv + c] = f;
                }
            }
        return lmoe::Tensor::from_data({n, dv}, std::move(out), dt);
    }
    lmoe::MemoryState state(const lmoe::LsmSpec& spec, lmoe::DType dt) const {
        std::vector<float> Mh((size_t)pl.D * pl.D), zh(pl.D);
        d2h(Mh.data(), M.p, Mh.size() * 4);
        lmoe::MemoryState st;
        std::vector<double> m((size_t)spec.d_k * spec.d_v);
        for (int i = 0; i < spec.d_k; ++i)
            for (int j = 0; j < spec.d_v; ++j) m[(size_t)i * spec.d_v + j] = Mh[(size_t)i * pl.D + j];
        st.M = lmoe::Tensor::from_data({spec.d_k, spec.d_v}, std::move(m), dt);
        if (spec.use_normalizer) {
            d2h(zh.data(), z.p, zh.size() * 4);
            std::vector<double> zz(spec.d_k);
            for (int i = 0; i < spec.d_k; ++i) zz[i] = zh[i];
            st.z = lmoe::Tensor::from_data({spec.d_k}, std::move(zz), dt);
        }
        st.step = n;
        return st;
    }
};

}  // namespace bridge

// lsm_forward_chunked (lsm.hpp:668-708) for one (N x d) head on the device.
inline lmoe::Tensor lsm_forward_chunked(const lmoe::Tensor& q_mat, const lmoe::Tensor& k_mat, const lmoe::Tensor& v_mat,
                                  const lmoe::LsmGates& gates, const lmoe::LsmSpec& spec, int chunk_size,
                                  lmoe::MemoryState* final_state = nullptr) {
    spec.validate();  // the reference's own checks and texts ("LsmSpec: normalizer unsupported ...")
    if (chunk_size < 1) throw std::runtime_error("lsm_forward_chunked: chunk_size must be >= 1");
    bridge::LsmDev x(q_mat, k_mat, v_mat, gates, spec);
    lmoe_lsm_desc d = bridge::desc_for(spec, chunk_size);
    if (x.host_fmap) d.feature_map = 0;
    Workspace ws;
    void* w = ws.get(lmoe_lsm_fwd_workspace_size(&d, 1, x.n, 1, x.pl.D, x.pl.dt));
    check(lmoe_lsm_fwd(&d, 1, x.n, 1, x.pl.D, x.pl.dt, x.q.p, x.k.p, x.v.p, x.a_pre.p, x.b_pre.as<float>(),
                       x.a_raw.as<float>(), nullptr, nullptr, x.o.p, x.M.as<float>(),
                       spec.use_normalizer ? x.z.as<float>() : nullptr, w, ws.size(), nullptr));
    if (cudaDeviceSynchronize() != cudaSuccess) throw Error(LMOE_ERR_CUDA, "lsm_forward_chunked: device error");
    if (final_state) *final_state = x.state(spec, q_mat.dtype());
    return x.output(spec.d_v, q_mat.dtype());
}

// sp_lsm_masked_rank (parallel.hpp:303-376): this rank's slice; `nccl_comm` an ncclComm_t from
// lmoe_nccl_comm_init (a 1-rank communicator runs the multi-rank phase structure on one GPU).
inline lmoe::Tensor sp_lsm_masked_rank(void* nccl_comm, int rank, int world, const lmoe::Tensor& q_loc, const lmoe::Tensor& k_loc,
                                 const lmoe::Tensor& v_loc, const lmoe::LsmGates& g_loc, const lmoe::LsmSpec& spec,
                                 lmoe::MemoryState* final_state = nullptr) {
    spec.validate();
    if (!has_closed_chunk_form(spec.instance))
        throw std::runtime_error("sp_forward_masked: state-dependent instances have no chunk-parallel form");
    bridge::LsmDev x(q_loc, k_loc, v_loc, g_loc, spec);
    lmoe_lsm_desc d = bridge::desc_for(spec, 64);
    if (x.host_fmap) d.feature_map = 0;
    Workspace ws;
    void* w = ws.get(lmoe_sp_lsm_fwd_workspace_size(&d, 1, x.n, 1, x.pl.D, x.pl.dt, world));
    check(lmoe_sp_lsm_fwd(&d, 1, x.n, 1, x.pl.D, x.pl.dt, x.q.p, x.k.p, x.v.p, x.a_pre.p, x.b_pre.as<float>(),
                          x.a_raw.as<float>(), x.o.p, x.M.as<float>(), spec.use_normalizer ? x.z.as<float>() : nullptr,
                          nccl_comm, rank, world, w, ws.size(), nullptr));
    if (cudaDeviceSynchronize() != cudaSuccess) throw Error(LMOE_ERR_CUDA, "sp_lsm_masked_rank: device error");
    if (final_state) *final_state = x.state(spec, q_loc.dtype());
    return x.output(spec.d_v, q_loc.dtype());
}

// route (moe.hpp:58-85): the device top-k over fp32 logits, expanded to the reference's
// RoutingDecision (expert_ids ascending per token; dense (T x E) gates, zero outside the
// selection; dense full_probs).
inline lmoe::RoutingDecision route(const lmoe::Tensor& router_logits, int top_k) {
    if (router_logits.shape().size() != 2) detail::shape_error("route", router_logits.shape(), {});
    const int T = router_logits.shape()[0], E = router_logits.shape()[1];
    if (top_k < 1 || top_k > E) throw std::runtime_error("route: bad top_k");
    std::vector<float> lg((size_t)T * E);
    for (size_t i = 0; i < lg.size(); ++i) lg[i] = (float)router_logits.data()[i];
    bridge::DevBuf dl(lg.size() * 4), ids((size_t)T * top_k * 4), gts((size_t)T * top_k * 4),
        probs((size_t)T * E * 4), counts((size_t)E * 4), aux(4);
    bridge::h2d(dl.p, lg.data(), lg.size() * 4);
    Workspace ws;
    cuda::RoutingDecision o{ids.as<int>(), gts.as<float>(), probs.as<float>(), counts.as<int>(), aux.as<float>()};
    cuda::route(dl.as<float>(), T, E, top_k, o, ws, nullptr);
    std::vector<int> hid((size_t)T * top_k);
    std::vector<float> hg((size_t)T * top_k), hp((size_t)T * E);
    bridge::d2h(hid.data(), ids.p, hid.size() * 4);
    bridge::d2h(hg.data(), gts.p, hg.size() * 4);
    bridge::d2h(hp.data(), probs.p, hp.size() * 4);
    lmoe::RoutingDecision dec;
    dec.expert_ids.resize(T);
    std::vector<double> gd((size_t)T * E, 0.0), pd(hp.begin(), hp.end());
    for (int t = 0; t < T; ++t) {
        for (int j = 0; j < top_k; ++j) {
            const int e = hid[(size_t)t * top_k + j];
            dec.expert_ids[t].push_back(e);
            gd[(size_t)t * E + e] = hg[(size_t)t * top_k + j];
        }
    }
    dec.gates = lmoe::Tensor::from_data({T, E}, std::move(gd), router_logits.dtype());
    dec.full_probs = lmoe::Tensor::from_data({T, E}, std::move(pd), router_logits.dtype());
    return dec;
}

// MoeLayer::forward (moe.hpp:133-149): {y (T x hidden), load_balance_loss} on the device.
inline std::pair<lmoe::Tensor, lmoe::Tensor> moe_forward(const lmoe::MoeLayer& layer, const lmoe::Tensor& x) {
    layer.config.validate();
    const lmoe::MoeConfig& c = layer.config;
    const int T = x.shape()[0];
    if (x.shape().size() != 2 || x.shape()[1] != c.hidden) detail::shape_error("MoeLayer::forward", x.shape(), {});
    const int Hp = (c.hidden + 255) / 256 * 256, Fp = (c.ffn_dim + 127) / 128 * 128, E = c.num_experts;
    auto up = [](const lmoe::Tensor& t, int rows, int cols, int prow, int pcol, bridge::DevBuf& dst, size_t off) {
        std::vector<uint16_t> img((size_t)prow * pcol, 0);
        for (int r = 0; r < rows; ++r)
            for (int cc = 0; cc < cols; ++cc) img[(size_t)r * pcol + cc] = bridge::to_bf16((float)t.at(r, cc));
        bridge::h2d(static_cast<uint8_t*>(dst.p) + off, img.data(), img.size() * 2);
    };
    bridge::DevBuf dx((size_t)T * Hp * 2), dr((size_t)Hp * E * 2), dg((size_t)E * Hp * Fp * 2),
        du((size_t)E * Hp * Fp * 2), dd((size_t)E * Fp * Hp * 2), dy((size_t)T * Hp * 4), daux(4);
    up(x, T, c.hidden, T, Hp, dx, 0);
    up(layer.router, c.hidden, E, Hp, E, dr, 0);
    for (int e = 0; e < E; ++e) {
        const lmoe::Expert& ex = layer.experts[e];
        up(ex.w_gate, c.hidden, c.ffn_dim, Hp, Fp, dg, (size_t)e * Hp * Fp * 2);
        up(ex.w_up, c.hidden, c.ffn_dim, Hp, Fp, du, (size_t)e * Hp * Fp * 2);
        up(ex.w_down, c.ffn_dim, c.hidden, Fp, Hp, dd, (size_t)e * Fp * Hp * 2);
    }
    cuda::MoeLayer dl;
    dl.config = cuda::MoeConfig{E, c.top_k, Hp, Fp};
    dl.router = dr.p;
    dl.w_gate = dg.p;
    dl.w_up = du.p;
    dl.w_down = dd.p;
    Workspace ws;
    dl.forward(dx.p, T, dy.p, daux.as<float>(), ws, true, nullptr);
    std::vector<float> hy((size_t)T * Hp);
    float haux = 0.f;
    bridge::d2h(hy.data(), dy.p, hy.size() * 4);
    bridge::d2h(&haux, daux.p, 4);
    std::vector<double> y((size_t)T * c.hidden);
    for (int t = 0; t < T; ++t)
        for (int j = 0; j < c.hidden; ++j) y[(size_t)t * c.hidden + j] = hy[(size_t)t * Hp + j];
    return {lmoe::Tensor::from_data({T, c.hidden}, std::move(y), x.dtype()), lmoe::Tensor::from_data({1}, {haux}, x.dtype())};
}

}  // namespace cuda
}  // namespace lmoe
