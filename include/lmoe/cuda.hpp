// lmoe/cuda.hpp -- C++ drop-in layer over the C ABI (lmoe_cuda.h) that keeps the names,
// argument meaning and error texts of the reference's hot path
// (/root/reference/proj/include/lmoe/{lsm,moe,parallel}.hpp), for callers that hold
// device buffers.  Header-only; link liblmoe_cuda.so.
//
//   reference (CPU, lmoe::)                    this header (B200, lmoe::cuda::)
//   lsm_forward_chunked   lsm.hpp:668          lsm_forward_chunked(view, gates, spec, chunk, &fs)
//   sp_lsm_masked_rank    parallel.hpp:303     sp_lsm_masked_rank(comm, view, gates, spec, &fs)
//   (its tape VJP)                             sp_lsm_masked_rank_backward(comm, ..., dO, grads)
//   route                 moe.hpp:58           route(logits, T, E, top_k)
//   MoeLayer::forward     moe.hpp:133          MoeLayer::forward(x, T, y)
//   std::runtime_error(msg)                    lmoe::cuda::Error (a std::runtime_error) with the
//                                              same message text
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../lmoe_cuda.h"

namespace lmoe {
namespace cuda {

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check(int rc) {
    if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
}

// RAII device scratch buffer (grows, never shrinks).
class Workspace {
public:
    Workspace() = default;
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;
    ~Workspace() { if (p_) cudaFree(p_); }
    void* get(size_t bytes) {
        if (bytes > n_) {
            if (p_) cudaFree(p_);
            p_ = nullptr;
            if (cudaMalloc(&p_, bytes) != cudaSuccess) throw Error(LMOE_ERR_CUDA, "workspace allocation failed");
            n_ = bytes;
        }
        return p_;
    }
    size_t size() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

// lmoe::LsmSpec (lsm.hpp:126-204), separable kinds.  LsmSpec::make applies the reference
// defaults (BLA: elu+1 + normaliser, Rebased: x^2 + normaliser, Lightning a = 0.95,
// RetNet a = 1 - 1/32).
struct LsmSpec {
    int instance = LMOE_BLA;
    int feature_map = LMOE_FM_IDENTITY;
    bool use_normalizer = false;
    float scalar_decay = 1.f;
    const float* mamba2_a_raw = nullptr;  // device [H]

    static LsmSpec make(int instance) {
        LsmSpec s;
        s.instance = instance;
        if (instance == LMOE_BLA) { s.feature_map = LMOE_FM_ELU1; s.use_normalizer = true; }
        if (instance == LMOE_REBASED) { s.feature_map = LMOE_FM_SQUARED; s.use_normalizer = true; }
        if (instance == LMOE_LIGHTNING) s.scalar_decay = 0.95f;
        if (instance == LMOE_RETNET) s.scalar_decay = 1.f - 1.f / 32.f;
        return s;
    }
};

// lmoe::LsmGates (lsm.hpp:216-261): device pointers in the [B, N, H(, D)] layout.
struct LsmGates {
    const void* a_pre = nullptr;   // TokenVector kinds, same dtype as q
    const float* b_pre = nullptr;  // Mamba2, fp32 [B, N, H]
};

// lmoe::MemoryState (lsm.hpp:264-281): device fp32 [B, H, D, D] and [B, H, D].
struct MemoryState {
    float* M = nullptr;
    float* z = nullptr;
};

// A batched head view: q, k, v, o are [B, N, H, D] device buffers.
struct LsmView {
    int B = 1, N = 0, H = 1, D = 0;
    lmoe_dtype dtype = LMOE_BF16;
    const void *q = nullptr, *k = nullptr, *v = nullptr;
    void* o = nullptr;
};

inline lmoe_lsm_desc to_desc(const LsmSpec& s, int chunk_size, bool check_device) {
    lmoe_lsm_desc d{};
    d.instance = s.instance;
    d.feature_map = s.feature_map;
    d.use_normalizer = s.use_normalizer ? 1 : 0;
    d.scalar_decay = s.scalar_decay;
    d.chunk_size = chunk_size;
    d.flags = check_device ? LMOE_FLAG_CHECK : 0;
    return d;
}

// lsm_forward_chunked (lsm.hpp:668-708) for all heads at once.  final_state receives the
// reference's final_state out-parameter when non-null; initial_state is the SP carried-in
// state (parallel.hpp:366-373) or nullptr for MemoryState::fresh.
inline void lsm_forward_chunked(const LsmView& x, const LsmGates& gates, const LsmSpec& spec,
                                int chunk_size, MemoryState* final_state = nullptr,
                                const MemoryState* initial_state = nullptr, Workspace* ws = nullptr,
                                cudaStream_t stream = nullptr, bool check_device = true) {
    Workspace local;
    Workspace& w = ws ? *ws : local;
    const lmoe_lsm_desc d = to_desc(spec, chunk_size, check_device);
    const size_t need = lmoe_lsm_fwd_workspace_size(&d, x.B, x.N, x.H, x.D, x.dtype);
    void* wsp = w.get(need);
    check(lmoe_lsm_fwd(&d, x.B, x.N, x.H, x.D, x.dtype, x.q, x.k, x.v, gates.a_pre, gates.b_pre,
                       spec.mamba2_a_raw, initial_state ? initial_state->M : nullptr,
                       initial_state ? initial_state->z : nullptr, x.o,
                       final_state ? final_state->M : nullptr, final_state ? final_state->z : nullptr,
                       wsp, w.size(), reinterpret_cast<lmoe_stream_t>(stream)));
}

// sp_lsm_masked_rank (parallel.hpp:303-376): this rank's slice (chunk_range), one NCCL
// all-gather of the per-rank state payload.  `nccl_comm` is an ncclComm_t created with
// lmoe_nccl_comm_init (one process / thread per GPU).
inline void sp_lsm_masked_rank(void* nccl_comm, int rank, int world, const LsmView& x_loc,
                               const LsmGates& g_loc, const LsmSpec& spec,
                               MemoryState* final_state = nullptr, Workspace* ws = nullptr,
                               cudaStream_t stream = nullptr, bool check_device = true) {
    Workspace local;
    Workspace& w = ws ? *ws : local;
    const lmoe_lsm_desc d = to_desc(spec, 64, check_device);
    const size_t need = lmoe_sp_lsm_fwd_workspace_size(&d, x_loc.B, x_loc.N, x_loc.H, x_loc.D, x_loc.dtype, world);
    void* wsp = w.get(need);
    check(lmoe_sp_lsm_fwd(&d, x_loc.B, x_loc.N, x_loc.H, x_loc.D, x_loc.dtype, x_loc.q, x_loc.k, x_loc.v,
                          g_loc.a_pre, g_loc.b_pre, spec.mamba2_a_raw, x_loc.o,
                          final_state ? final_state->M : nullptr, final_state ? final_state->z : nullptr,
                          nccl_comm, rank, world, wsp, w.size(),
                          reinterpret_cast<lmoe_stream_t>(stream)));
}

// sp_lsm_nomask_rank (parallel.hpp:282-297): O = phiQ . sum over ranks of phiK^T V, one gather.
inline void sp_lsm_nomask_rank(void* nccl_comm, int rank, int world, const LsmView& x_loc, const LsmSpec& spec,
                               Workspace* ws = nullptr, cudaStream_t stream = nullptr, bool check_device = true) {
    Workspace local;
    Workspace& w = ws ? *ws : local;
    const lmoe_lsm_desc d = to_desc(spec, 64, check_device);
    const size_t need = lmoe_sp_lsm_nomask_workspace_size(&d, x_loc.B, x_loc.N, x_loc.H, x_loc.D, x_loc.dtype, world);
    void* wsp = w.get(need);
    check(lmoe_sp_lsm_nomask_fwd(&d, x_loc.B, x_loc.N, x_loc.H, x_loc.D, x_loc.dtype, x_loc.q, x_loc.k, x_loc.v,
                                 x_loc.o, nccl_comm, rank, world, wsp, w.size(),
                                 reinterpret_cast<lmoe_stream_t>(stream)));
}

// Gradients of lsm_forward_chunked (the reference tape, tensor.hpp:1178-1215): device
// buffers in the layouts of lmoe_lsm_bwd.
struct LsmGrads {
    void *dq = nullptr, *dk = nullptr, *dv = nullptr, *da_pre = nullptr;
    float* db_pre = nullptr;  // [B, N, H]   Mamba2
    float* da_raw = nullptr;  // [H]         Mamba2
    float* dM0 = nullptr;     // [B, H, D, D]
};
inline void lsm_backward_chunked(const LsmView& x, const LsmGates& gates, const LsmSpec& spec, const void* dO,
                                 const LsmGrads& g, const MemoryState* initial_state = nullptr,
                                 const float* dM_final = nullptr, Workspace* ws = nullptr,
                                 cudaStream_t stream = nullptr, bool check_device = true) {
    Workspace local;
    Workspace& w = ws ? *ws : local;
    const lmoe_lsm_desc d = to_desc(spec, 64, check_device);
    const size_t need = lmoe_lsm_bwd_workspace_size(&d, x.B, x.N, x.H, x.D, x.dtype);
    void* wsp = w.get(need);
    check(lmoe_lsm_bwd(&d, x.B, x.N, x.H, x.D, x.dtype, x.q, x.k, x.v, gates.a_pre, gates.b_pre, spec.mamba2_a_raw,
                       initial_state ? initial_state->M : nullptr, dO, dM_final, g.dq, g.dk, g.dv, g.da_pre,
                       g.db_pre, g.da_raw, g.dM0, wsp, w.size(), reinterpret_cast<lmoe_stream_t>(stream)));
}

// Backward of sp_lsm_masked_rank for this rank's slice: two all-gathers (forward and
// reverse-time payloads), suffix combine over later ranks, exact local backward.  da_raw is
// this rank's contribution; dM0 is meaningful on rank 0.
inline void sp_lsm_masked_rank_backward(void* nccl_comm, int rank, int world, const LsmView& x_loc,
                                        const LsmGates& g_loc, const LsmSpec& spec, const void* dO_loc,
                                        const LsmGrads& g, Workspace* ws = nullptr, cudaStream_t stream = nullptr,
                                        bool check_device = true) {
    Workspace local;
    Workspace& w = ws ? *ws : local;
    const lmoe_lsm_desc d = to_desc(spec, 64, check_device);
    const size_t need = lmoe_sp_lsm_bwd_workspace_size(&d, x_loc.B, x_loc.N, x_loc.H, x_loc.D, x_loc.dtype, world);
    void* wsp = w.get(need);
    check(lmoe_sp_lsm_bwd(&d, x_loc.B, x_loc.N, x_loc.H, x_loc.D, x_loc.dtype, x_loc.q, x_loc.k, x_loc.v,
                          g_loc.a_pre, g_loc.b_pre, spec.mamba2_a_raw, dO_loc, g.dq, g.dk, g.dv, g.da_pre, g.db_pre,
                          g.da_raw, g.dM0, nccl_comm, rank, world, wsp, w.size(),
                          reinterpret_cast<lmoe_stream_t>(stream)));
}

// chunk_range (parallel.hpp:192-197)
inline std::pair<int, int> chunk_range(int n, int t, int rank) {
    if (n < t) throw Error(LMOE_ERR_ARG, "chunk_range: need at least one row per rank");
    const int base = n / t, rem = n % t;
    const int r0 = rank * base + (rank < rem ? rank : rem);
    return {r0, r0 + base + (rank < rem ? 1 : 0)};
}

// RoutingDecision (moe.hpp:52-56) in compact device form: ids [T, k] ascending per token,
// gates [T, k] renormalised over the selection, full_probs [T, E].
struct RoutingDecision {
    int* expert_ids = nullptr;
    float* gates = nullptr;
    float* full_probs = nullptr;
    int* counts = nullptr;  // [E]
    float* aux = nullptr;   // load_balance_loss (moe.hpp:90-103), device scalar
};

// route (moe.hpp:58-85) on device fp32 logits [T, E]; "route: bad top_k" as the reference.
inline void route(const float* logits, int T, int E, int top_k, const RoutingDecision& out,
                  Workspace& ws, cudaStream_t stream = nullptr) {
    const size_t need = lmoe_moe_workspace_size(T, 64, 64, E, top_k > 0 ? top_k : 1);
    void* wsp = ws.get(need);
    check(lmoe_moe_route(logits, T, E, top_k, out.expert_ids, out.gates, out.full_probs, out.counts,
                         out.aux, wsp, ws.size(), reinterpret_cast<lmoe_stream_t>(stream)));
}

// MoeConfig / MoeLayer (moe.hpp:15-27, 106-149) with bf16 device weights in the reference
// layouts: router (hidden, E); w_gate, w_up (E, hidden, ffn); w_down (E, ffn, hidden).
struct MoeConfig {
    int num_experts = 1, top_k = 1, hidden = 0, ffn_dim = 0;
    void validate() const {
        if (num_experts < 1 || top_k < 1 || top_k > num_experts)
            throw Error(LMOE_ERR_ARG, "MoeConfig: need 1 <= top_k <= num_experts");
        if (hidden <= 0 || ffn_dim <= 0) throw Error(LMOE_ERR_ARG, "MoeConfig: nonpositive dims");
    }
};

struct MoeLayer {
    MoeConfig config;
    const void* router = nullptr;
    const void* w_gate = nullptr;
    const void* w_up = nullptr;
    const void* w_down = nullptr;

    // y (T, hidden) bf16 (or fp32 with y_f32) and the aux loss (device scalar).
    void forward(const void* x, int T, void* y, float* aux, Workspace& ws, bool y_f32 = false,
                 cudaStream_t stream = nullptr) const {
        config.validate();
        const MoeConfig& c = config;
        const size_t need = lmoe_moe_workspace_size(T, c.hidden, c.ffn_dim, c.num_experts, c.top_k);
        void* wsp = ws.get(need);
        check(lmoe_moe_forward(T, c.hidden, c.ffn_dim, c.num_experts, c.top_k, x, router, w_gate, w_up,
                               w_down, y, y_f32 ? 1 : 0, aux, nullptr, nullptr, nullptr, wsp,
                               ws.size(), reinterpret_cast<lmoe_stream_t>(stream)));
    }
};

}  // namespace cuda
}  // namespace lmoe
