// ref_driver.cpp -- runs the UNMODIFIED reference (/root/reference/proj/include/lmoe,
// header-only C++20) to (1) emit golden vectors that pin oracle/lmoe_oracle.c and the
// CUDA path, and (2) time the reference CPU path for bench.py's cpu_baseline /
// --impl reference arm.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ (git-ignored,
// travels to the GPU box with gpurun).  This file contains no reference source; it
// only #includes the reference headers from their read-only location.
//
//   ref_driver golden <out.bin>
//   ref_driver bench-lsm <instance> <B> <N> <H> <d> <chunk> <threads> <budget_s> [gate_mean]
//   ref_driver bench-moe <T> <hidden> <ffn> <E> <k> <threads> <budget_s>
//   ref_driver bench-block <instance> <kind L|N> <doc_len> <hidden> <heads> <ffn> <E> <k>
//                          <threads> <budget_s>
//
// Golden stream format: records of
//   u32 name_len, name bytes, u32 ndim, u32 shape[ndim], f64 data[prod(shape)]

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lmoe/attention.hpp"
#include "lmoe/lsm.hpp"
#include "lmoe/model.hpp"
#include "lmoe/moe.hpp"
#include "lmoe/parallel.hpp"

using namespace lmoe;

namespace {

FILE* g_out = nullptr;

void emit(const std::string& name, const std::vector<int>& shape, const std::vector<double>& d) {
    uint32_t nl = (uint32_t)name.size();
    fwrite(&nl, 4, 1, g_out);
    fwrite(name.data(), 1, nl, g_out);
    uint32_t nd = (uint32_t)shape.size();
    fwrite(&nd, 4, 1, g_out);
    for (int s : shape) {
        uint32_t u = (uint32_t)s;
        fwrite(&u, 4, 1, g_out);
    }
    fwrite(d.data(), 8, d.size(), g_out);
}
void emit(const std::string& name, const Tensor& t) {
    if (!t.defined()) return;
    emit(name, t.shape(), t.data());
}
void emit_scalar(const std::string& name, double v) { emit(name, {1}, {v}); }

// bf16 round-to-nearest-even, as the device sees bf16 inputs
double to_bf16(double x) {
    float f = (float)x;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
    std::memcpy(&f, &u, 4);
    return (double)f;
}
Tensor round_bf16(const Tensor& t) {
    std::vector<double> d = t.data();
    for (auto& x : d) x = to_bf16(x);
    return Tensor::from_data(t.shape(), d);
}

struct Variant {
    const char* tag;
    LsmInstance inst;
    int fm;    // -1: reference default
    int norm;  // -1: reference default
};

LsmSpec make_spec(const Variant& v, int d, Rng& rng) {
    LsmSpec s = LsmSpec::make(v.inst, d, d, &rng);
    if (v.fm >= 0) s.feature_map = (FeatureMap)v.fm;
    if (v.norm >= 0) s.use_normalizer = v.norm != 0;
    return s;
}

void emit_spec(const std::string& p, const LsmSpec& s) {
    emit_scalar(p + "/instance", (double)(int)s.instance);
    emit_scalar(p + "/feature_map", (double)(int)s.feature_map);
    emit_scalar(p + "/use_normalizer", s.use_normalizer ? 1.0 : 0.0);
    emit_scalar(p + "/scalar_decay", s.scalar_decay);
    emit_scalar(p + "/mamba2_a_raw", s.mamba2_a_raw.defined() ? s.mamba2_a_raw.item() : 0.0);
}

const Variant kVariants[] = {
    {"bla", LsmInstance::BLA, -1, -1},
    {"bla_plain", LsmInstance::BLA, 0, 0},
    {"rebased", LsmInstance::Rebased, -1, -1},
    {"rebased_plain", LsmInstance::Rebased, -1, 0},
    {"lightning", LsmInstance::Lightning, -1, -1},
    {"retnet", LsmInstance::RetNet, -1, -1},
    {"retnet_norm", LsmInstance::RetNet, 1, 1},
    {"gla", LsmInstance::GLA, -1, -1},
    {"gla_norm", LsmInstance::GLA, 1, 1},
    {"hgrn2", LsmInstance::HGRN2, -1, -1},
    {"rwkv6", LsmInstance::RWKV6, -1, -1},
    {"mamba2", LsmInstance::Mamba2, -1, -1},
};

// ---- LSM: chunked vs sequential, tiny head dims (acceptance.cpp:44-69 style) ----
void golden_lsm_small() {
    int vi = 0;
    for (const Variant& var : kVariants) {
        for (int n : {7, 33}) {
            const int d = 4;
            Rng rng(1000 + 17 * vi + n);
            LsmSpec spec = make_spec(var, d, rng);
            const Tensor q = Tensor::randn({n, d}, rng, 0.5);
            const Tensor k = Tensor::randn({n, d}, rng, 0.5);
            const Tensor v = Tensor::randn({n, d}, rng, 0.5);
            const LsmGates g = LsmGates::random_for(spec, n, rng);
            const std::string p = std::string("lsm_small/") + var.tag + "_n" + std::to_string(n);
            emit_spec(p, spec);
            emit(p + "/q", q);
            emit(p + "/k", k);
            emit(p + "/v", v);
            emit(p + "/a_pre", g.a_pre);
            emit(p + "/b_pre", g.b_pre);
            MemoryState fs;
            emit(p + "/o_seq", lsm_forward_sequential(q, k, v, g, spec, &fs));
            emit(p + "/M_seq", fs.M);
            emit(p + "/z_seq", fs.z);
            for (int c : {1, 3, 8, n}) {
                MemoryState fc;
                emit(p + "/o_c" + std::to_string(c), lsm_forward_chunked(q, k, v, g, spec, c, &fc));
                emit(p + "/M_c" + std::to_string(c), fc.M);
                emit(p + "/z_c" + std::to_string(c), fc.z);
            }
        }
        ++vi;
    }
}

// ---- LSM at device head dims, bf16-exact inputs (GPU golden) ----
void golden_lsm_device() {
    struct Case { const char* var; int n; int d; int chunk; double gate_mean; double gate_std; };
    const Case cases[] = {
        {"bla_plain", 300, 64, 64, 0, 1},  {"bla", 300, 64, 64, 0, 1},
        {"lightning", 300, 64, 64, 0, 1},  {"retnet", 257, 128, 64, 0, 1},
        {"mamba2", 300, 64, 64, 0, 1},     {"mamba2", 260, 128, 64, -3, 0.5},
        {"gla", 300, 64, 64, 0, 1},        {"gla", 260, 128, 64, 4, 0.5},
        {"hgrn2", 300, 64, 64, 0, 1},      {"rwkv6", 200, 64, 64, 0, 1},
        {"rebased", 200, 64, 64, 0, 1},    {"gla_norm", 200, 64, 64, 0, 1},
    };
    int ci = 0;
    for (const Case& c : cases) {
        const Variant* var = nullptr;
        for (const Variant& v : kVariants) if (std::string(v.tag) == c.var) var = &v;
        Rng rng(5000 + ci);
        LsmSpec spec = make_spec(*var, c.d, rng);
        if (spec.mamba2_a_raw.defined())
            spec.mamba2_a_raw = Tensor::from_data({1}, {to_bf16(spec.mamba2_a_raw.item())});
        const Tensor q = round_bf16(Tensor::randn({c.n, c.d}, rng, 0.5));
        const Tensor k = round_bf16(Tensor::randn({c.n, c.d}, rng, 0.5));
        const Tensor v = round_bf16(Tensor::randn({c.n, c.d}, rng, 0.5));
        LsmGates g = LsmGates::random_for(spec, c.n, rng, c.gate_std);
        if (g.a_pre.defined()) {
            std::vector<double> a = g.a_pre.data();
            for (auto& x : a) x = to_bf16(x + c.gate_mean);
            g.a_pre = Tensor::from_data(g.a_pre.shape(), a);
        }
        if (g.b_pre.defined()) {
            std::vector<double> b = g.b_pre.data();
            for (auto& x : b) x = (double)(float)(x + c.gate_mean);
            g.b_pre = Tensor::from_data(g.b_pre.shape(), b);
        }
        const std::string p = std::string("lsm_dev/") + c.var + "_n" + std::to_string(c.n) +
                              "_d" + std::to_string(c.d) + (c.gate_mean != 0 ? "_long" : "");
        emit_spec(p, spec);
        emit_scalar(p + "/chunk", c.chunk);
        emit(p + "/q", q);
        emit(p + "/k", k);
        emit(p + "/v", v);
        emit(p + "/a_pre", g.a_pre);
        emit(p + "/b_pre", g.b_pre);
        MemoryState fs;
        emit(p + "/o", lsm_forward_chunked(q, k, v, g, spec, c.chunk, &fs));
        emit(p + "/M", fs.M);
        emit(p + "/z", fs.z);
        ++ci;
    }
}

// ---- non-separable kinds (DecayKind TokenOuter / FullElementwise / StateLinear / Gradient):
// recurrent_step (lsm.hpp:335-441) token by token, and lsm_forward_chunked (sequential inside
// each chunk, lsm.hpp:604-637) ----
void golden_lsm_seq() {
    struct SV { const char* tag; LsmInstance inst; };
    const SV kinds[] = {{"deltanet", LsmInstance::DeltaNet}, {"gated_deltanet", LsmInstance::GatedDeltaNet},
                        {"gfw", LsmInstance::GFW}, {"gateloop", LsmInstance::GateLoop}, {"ttt", LsmInstance::TTT},
                        {"titans", LsmInstance::Titans}, {"rwkv7", LsmInstance::RWKV7}, {"s4", LsmInstance::S4},
                        {"mamba", LsmInstance::Mamba}};
    int vi = 0;
    for (const SV& sv : kinds) {
        for (int n : {7, 40}) {
            const int d = 8;
            Rng rng(21000 + 31 * vi + n);
            LsmSpec spec = LsmSpec::make(sv.inst, d, d, &rng);
            const Tensor q = Tensor::randn({n, d}, rng, 0.5);
            const Tensor k = Tensor::randn({n, d}, rng, 0.5);
            const Tensor v = Tensor::randn({n, d}, rng, 0.5);
            const LsmGates g = LsmGates::random_for(spec, n, rng);
            const std::string p = std::string("lsm_seq/") + sv.tag + "_n" + std::to_string(n);
            emit_spec(p, spec);
            emit(p + "/q", q);
            emit(p + "/k", k);
            emit(p + "/v", v);
            emit(p + "/a_pre", g.a_pre);
            emit(p + "/b_pre", g.b_pre);
            emit(p + "/alpha_pre", g.alpha_pre);
            emit(p + "/beta_pre", g.beta_pre);
            emit(p + "/s4_delta_raw", spec.s4_delta_raw);
            emit(p + "/s4_b", spec.s4_b);
            emit(p + "/s4_A_raw", spec.s4_A_raw);
            emit(p + "/mamba_A_raw", spec.mamba_A_raw);
            MemoryState fs;
            emit(p + "/o_seq", lsm_forward_sequential(q, k, v, g, spec, &fs));
            emit(p + "/M_seq", fs.M);
            MemoryState fc;
            emit(p + "/o_c8", lsm_forward_chunked(q, k, v, g, spec, 8, &fc));
            emit(p + "/M_c8", fc.M);
        }
        ++vi;
    }
}

// ---- LSM gradients from the reference tape (tensor.hpp:1178) ----
void golden_lsm_grad() {
    // appended tags keep the seeds of the earlier ones: the normalised reference defaults
    const char* tags[] = {"bla_plain", "lightning", "retnet", "gla", "hgrn2", "rwkv6", "mamba2",
                          "rebased_plain", "bla", "rebased", "retnet_norm", "gla_norm"};
    int ci = 0;
    for (const char* tag : tags) {
        const Variant* var = nullptr;
        for (const Variant& v : kVariants) if (std::string(v.tag) == tag) var = &v;
        const int n = 20, d = 4;
        Rng rng(7000 + ci);
        LsmSpec spec = make_spec(*var, d, rng);
        if (spec.mamba2_a_raw.defined()) spec.mamba2_a_raw.set_requires_grad(true);
        Tensor q = Tensor::randn({n, d}, rng, 0.5, DType::f64, true);
        Tensor k = Tensor::randn({n, d}, rng, 0.5, DType::f64, true);
        Tensor v = Tensor::randn({n, d}, rng, 0.5, DType::f64, true);
        LsmGates g = LsmGates::random_for(spec, n, rng);
        if (g.a_pre.defined()) g.a_pre.set_requires_grad(true);
        if (g.b_pre.defined()) g.b_pre.set_requires_grad(true);
        const Tensor w = Tensor::randn({n, d}, rng, 1.0);
        const Tensor o = lsm_forward_chunked(q, k, v, g, spec, 8);
        backward(sum(mul(o, w)));
        const std::string p = std::string("lsm_grad/") + tag;
        emit_spec(p, spec);
        emit(p + "/q", q);
        emit(p + "/k", k);
        emit(p + "/v", v);
        emit(p + "/a_pre", g.a_pre);
        emit(p + "/b_pre", g.b_pre);
        emit(p + "/dO", w);
        emit(p + "/o", o);
        emit(p + "/dq", {n, d}, q.grad());
        emit(p + "/dk", {n, d}, k.has_grad() ? k.grad() : std::vector<double>(n * d, 0.0));
        emit(p + "/dv", {n, d}, v.grad());
        if (g.a_pre.defined()) emit(p + "/da_pre", g.a_pre.shape(), g.a_pre.grad());
        if (g.b_pre.defined()) emit(p + "/db_pre", g.b_pre.shape(), g.b_pre.grad());
        if (spec.mamba2_a_raw.defined()) emit(p + "/da_raw", {1}, spec.mamba2_a_raw.grad());
        ++ci;
    }
}

// ---- gradients of the recurrent kinds from the reference tape (tensor.hpp:1178) over
// recurrent_step (lsm.hpp:335-441): every input and static parameter requires grad ----
void golden_lsm_rec_grad() {
    struct SV { const char* tag; LsmInstance inst; };
    const SV kinds[] = {{"deltanet", LsmInstance::DeltaNet}, {"gated_deltanet", LsmInstance::GatedDeltaNet},
                        {"gfw", LsmInstance::GFW}, {"gateloop", LsmInstance::GateLoop}, {"ttt", LsmInstance::TTT},
                        {"titans", LsmInstance::Titans}, {"rwkv7", LsmInstance::RWKV7}, {"s4", LsmInstance::S4},
                        {"mamba", LsmInstance::Mamba}};
    int vi = 0;
    for (const SV& sv : kinds) {
        const int n = 37, d = 4;
        Rng rng(31000 + 17 * vi);
        LsmSpec spec = LsmSpec::make(sv.inst, d, d, &rng);
        for (Tensor* t : {&spec.s4_delta_raw, &spec.s4_b, &spec.s4_A_raw, &spec.mamba_A_raw})
            if (t->defined()) t->set_requires_grad(true);
        Tensor q = Tensor::randn({n, d}, rng, 0.5, DType::f64, true);
        Tensor k = Tensor::randn({n, d}, rng, 0.5, DType::f64, true);
        Tensor v = Tensor::randn({n, d}, rng, 0.5, DType::f64, true);
        LsmGates g = LsmGates::random_for(spec, n, rng);
        for (Tensor* t : {&g.a_pre, &g.b_pre, &g.alpha_pre, &g.beta_pre})
            if (t->defined()) t->set_requires_grad(true);
        const Tensor w = Tensor::randn({n, d}, rng, 1.0);
        const Tensor o = lsm_forward_chunked(q, k, v, g, spec, 8);
        backward(sum(mul(o, w)));
        const std::string p = std::string("lsm_rec_grad/") + sv.tag;
        emit_spec(p, spec);
        emit(p + "/q", q);
        emit(p + "/k", k);
        emit(p + "/v", v);
        emit(p + "/dO", w);
        emit(p + "/o", o);
        auto grad_of = [&](const Tensor& t) {
            return t.has_grad() ? t.grad() : std::vector<double>(t.size(), 0.0);
        };
        emit(p + "/dq", {n, d}, grad_of(q));
        emit(p + "/dk", {n, d}, grad_of(k));
        emit(p + "/dv", {n, d}, grad_of(v));
        const char* names[] = {"a_pre", "b_pre", "alpha_pre", "beta_pre", "s4_delta_raw", "s4_b", "s4_A_raw",
                               "mamba_A_raw"};
        const Tensor* ts[] = {&g.a_pre, &g.b_pre, &g.alpha_pre, &g.beta_pre, &spec.s4_delta_raw, &spec.s4_b,
                              &spec.s4_A_raw, &spec.mamba_A_raw};
        for (int i = 0; i < 8; ++i) {
            if (!ts[i]->defined()) continue;
            emit(p + "/" + names[i], *ts[i]);
            emit(p + "/d" + names[i], ts[i]->shape(), grad_of(*ts[i]));
        }
        ++vi;
    }
}

// ---- routing (moe.hpp:58-103), KATs of test_moe.cpp:9-62 plus random ----
void golden_route() {
    NoGradGuard ng;
    struct RC { const char* tag; int t; int e; int k; int kind; };
    const RC cases[] = {{"tie", 2, 4, 2, 0}, {"rand_k1", 64, 8, 1, 1}, {"rand_k2", 64, 8, 2, 1},
                        {"rand_k3", 64, 8, 3, 1}, {"rand_k8", 64, 8, 8, 1},
                        {"e64_k8", 256, 64, 8, 1}, {"e64_k8_ties", 128, 64, 8, 2}};
    int ci = 0;
    for (const RC& c : cases) {
        Rng rng(9000 + ci);
        Tensor logits;
        if (c.kind == 0) {
            logits = Tensor::from_data({2, 4}, {0.1, 0.9, 0.9, 0.2, -1.0, -1.0, -1.0, -1.0});
        } else if (c.kind == 1) {
            logits = round_bf16(Tensor::randn({c.t, c.e}, rng, 1.0));
            std::vector<double> d = logits.data();
            for (auto& x : d) x = (double)(float)x;
            logits = Tensor::from_data({c.t, c.e}, d);
        } else {  // heavy ties: small integer grid
            std::vector<double> d((size_t)c.t * c.e);
            for (auto& x : d) x = (double)(int)rng.randint(5) * 0.25;
            logits = Tensor::from_data({c.t, c.e}, d);
        }
        const RoutingDecision dec = route(logits, c.k);
        const std::string p = std::string("route/") + c.tag;
        emit(p + "/logits", logits);
        emit_scalar(p + "/top_k", c.k);
        std::vector<double> ids;
        for (const auto& row : dec.expert_ids) for (int id : row) ids.push_back(id);
        emit(p + "/ids", {c.t, c.k}, ids);
        emit(p + "/gates", dec.gates);
        emit(p + "/probs", dec.full_probs);
        emit_scalar(p + "/aux", load_balance_loss(dec).item());
        ++ci;
    }
}

// ---- MoE layer forward (moe.hpp:133-149) ----
void golden_moe() {
    NoGradGuard ng;
    struct MC { const char* tag; int t; int hidden; int ffn; int e; int k; };
    const MC cases[] = {{"small", 10, 6, 8, 4, 2}, {"mid", 40, 16, 12, 8, 2}, {"dense", 16, 8, 8, 4, 4}};
    int ci = 0;
    for (const MC& c : cases) {
        Rng rng(11000 + ci);
        const MoeConfig cfg{c.e, c.k, c.hidden, c.ffn, 0.01};
        const MoeLayer layer = MoeLayer::init(cfg, rng, DType::f64);
        const Tensor x = Tensor::randn({c.t, c.hidden}, rng, 0.5);
        auto [y, aux] = layer.forward(x);
        const std::string p = std::string("moe/") + c.tag;
        emit_scalar(p + "/top_k", c.k);
        emit(p + "/x", x);
        emit(p + "/router", layer.router);
        std::vector<double> wg, wu, wd;
        for (const auto& ex : layer.experts) {
            wg.insert(wg.end(), ex.w_gate.data().begin(), ex.w_gate.data().end());
            wu.insert(wu.end(), ex.w_up.data().begin(), ex.w_up.data().end());
            wd.insert(wd.end(), ex.w_down.data().begin(), ex.w_down.data().end());
        }
        emit(p + "/w_gate", {c.e, c.hidden, c.ffn}, wg);
        emit(p + "/w_up", {c.e, c.hidden, c.ffn}, wu);
        emit(p + "/w_down", {c.e, c.ffn, c.hidden}, wd);
        emit(p + "/y", y);
        emit_scalar(p + "/aux", aux.item());
        ++ci;
    }
}

// ---- sequence parallelism (parallel.hpp:282-418) ----
void golden_sp() {
    NoGradGuard ng;
    const int n = 32, d = 4;
    int ci = 0;
    for (const char* tag : {"bla", "bla_plain", "lightning", "gla", "mamba2", "hgrn2", "gla_norm"}) {
        const Variant* var = nullptr;
        for (const Variant& v : kVariants) if (std::string(v.tag) == tag) var = &v;
        Rng rng(13000 + ci);
        LsmSpec spec = make_spec(*var, d, rng);
        const Tensor q = Tensor::randn({n, d}, rng, 0.5);
        const Tensor k = Tensor::randn({n, d}, rng, 0.5);
        const Tensor v = Tensor::randn({n, d}, rng, 0.5);
        const LsmGates g = LsmGates::random_for(spec, n, rng);
        const std::string p = std::string("sp/") + tag;
        emit_spec(p, spec);
        emit(p + "/q", q);
        emit(p + "/k", k);
        emit(p + "/v", v);
        emit(p + "/a_pre", g.a_pre);
        emit(p + "/b_pre", g.b_pre);
        emit(p + "/o_seq", lsm_forward_sequential(q, k, v, g, spec));
        for (int t : {1, 2, 4, 8}) {
            RankGroup grp(t);
            emit(p + "/o_t" + std::to_string(t), sp_forward_masked(grp, q, k, v, g, spec));
            emit_scalar(p + "/comm_elems_t" + std::to_string(t),
                        (double)(grp.comm_log().empty() ? 0 : grp.comm_log()[0].elements));
        }
        ++ci;
    }
    // unmasked SP, Alg. 1 (parallel.hpp:282-297, 391-403)
    for (const char* tag : {"bla_plain", "rebased_plain"}) {
        const Variant* var = nullptr;
        for (const Variant& v : kVariants) if (std::string(v.tag) == tag) var = &v;
        Rng rng(13500 + ci);
        LsmSpec spec = make_spec(*var, d, rng);
        const Tensor q = Tensor::randn({n, d}, rng, 0.5);
        const Tensor k = Tensor::randn({n, d}, rng, 0.5);
        const Tensor v = Tensor::randn({n, d}, rng, 0.5);
        const std::string p = std::string("spn/") + tag;
        emit_spec(p, spec);
        emit(p + "/q", q);
        emit(p + "/k", k);
        emit(p + "/v", v);
        for (int t : {1, 2, 4, 8}) {
            RankGroup grp(t);
            emit(p + "/o_t" + std::to_string(t), sp_forward_nomask(grp, q, k, v, spec));
            emit_scalar(p + "/comm_elems_t" + std::to_string(t),
                        (double)(grp.comm_log().empty() ? 0 : grp.comm_log()[0].elements));
        }
        ++ci;
    }
    // attention with row offset + KV all-gather SP (attention.hpp:18-38, parallel.hpp:380-387)
    Rng rng(14000);
    const int na = 24;
    const Tensor q = Tensor::randn({na, 8}, rng, 0.5);
    const Tensor k = Tensor::randn({na, 8}, rng, 0.5);
    const Tensor v = Tensor::randn({na, 8}, rng, 0.5);
    emit("attn/q", q);
    emit("attn/k", k);
    emit("attn/v", v);
    emit("attn/o_full", softmax_attention_parallel(q, k, v, true));
    emit("attn/o_off", softmax_attention_parallel(slice_rows(q, 16, 24), k, v, true, 16));
    for (int t : {2, 4}) {
        RankGroup grp(t);
        emit("attn/o_sp_t" + std::to_string(t), sp_attention_allgather(grp, q, k, v));
        long el = 0;
        for (const auto& r : grp.comm_log()) el += r.elements;
        emit_scalar("attn/comm_elems_t" + std::to_string(t), (double)el);
    }
}

// ---- hybrid model (model.hpp:284-405, parallel.hpp:477-506): tiny stacks whose weights are
// rounded to bf16 IN PLACE before the run, so the device sees the identical parameters ----
void golden_model() {
    NoGradGuard ng;
    struct MC { const char* tag; LsmInstance inst; const char* pattern; };
    const MC cases[] = {{"mamba2_hybrid", LsmInstance::Mamba2, "LNL"}, {"gla", LsmInstance::GLA, "L"}};
    int ci = 0;
    for (const MC& c : cases) {
        ModelConfig cfg;
        cfg.hidden = 256;
        cfg.ffn_dim = 128;
        cfg.num_heads = 2;
        cfg.num_layers = (int)std::string(c.pattern).size();
        cfg.num_experts = 2;
        cfg.num_active = 2;
        cfg.vocab_size = 64;
        cfg.instance = c.inst;
        cfg.pattern = c.pattern;
        cfg.max_seq_len = 256;
        Rng rng(15000 + ci);
        Model m = build_model(cfg, rng);
        for (const Tensor& t : m.params()) {
            auto& d = const_cast<std::vector<double>&>(t.data());
            for (double& x : d) x = to_bf16(x);
        }
        const int n = 256;
        std::vector<int> toks(n);
        for (int i = 0; i < n; ++i) toks[i] = (int)(rng.uniform() * cfg.vocab_size) % cfg.vocab_size;
        const PackedBatch batch = pack_sequences({toks});
        const std::string p = std::string("model/") + c.tag;
        emit_scalar(p + "/instance", (double)(int)c.inst);
        emit_scalar(p + "/hidden", cfg.hidden);
        emit_scalar(p + "/heads", cfg.num_heads);
        emit_scalar(p + "/ffn", cfg.ffn_dim);
        emit_scalar(p + "/experts", cfg.num_experts);
        emit_scalar(p + "/top_k", cfg.num_active);
        emit_scalar(p + "/eps", cfg.norm_eps);
        emit_scalar(p + "/scalar_decay", m.blocks[0].kind == 'L' ? m.blocks[0].lsm.head_specs[0].scalar_decay : 1.0);
        std::vector<double> kinds;
        for (char k : std::string(c.pattern)) kinds.push_back(k == 'L' ? 1.0 : 0.0);
        emit(p + "/is_lsm", {(int)kinds.size()}, kinds);
        std::vector<double> tk(toks.begin(), toks.end());
        emit(p + "/tokens", {n}, tk);
        emit(p + "/embedding", m.embedding);
        emit(p + "/pos_embedding", m.pos_embedding);
        for (size_t b = 0; b < m.blocks.size(); ++b) {
            const Block& blk = m.blocks[b];
            const std::string q = p + "/b" + std::to_string(b);
            emit(q + "/norm_mixer", blk.norm_mixer);
            emit(q + "/norm_moe", blk.norm_moe);
            if (blk.kind == 'L') {
                emit(q + "/wq", blk.lsm.wq); emit(q + "/wk", blk.lsm.wk);
                emit(q + "/wv", blk.lsm.wv); emit(q + "/wo", blk.lsm.wo);
                emit(q + "/w_gate_a", blk.lsm.w_gate_a);
                emit(q + "/w_gate_b", blk.lsm.w_gate_b);
                std::vector<double> ar;
                for (const auto& hs : blk.lsm.head_specs)
                    ar.push_back(hs.mamba2_a_raw.defined() ? hs.mamba2_a_raw.item() : 0.0);
                emit(q + "/a_raw", {(int)ar.size()}, ar);
            } else {
                emit(q + "/wq", blk.attn.wq); emit(q + "/wk", blk.attn.wk);
                emit(q + "/wv", blk.attn.wv); emit(q + "/wo", blk.attn.wo);
            }
            emit(q + "/router", blk.moe.router);
            std::vector<double> wg, wu, wd;
            for (const auto& ex : blk.moe.experts) {
                wg.insert(wg.end(), ex.w_gate.data().begin(), ex.w_gate.data().end());
                wu.insert(wu.end(), ex.w_up.data().begin(), ex.w_up.data().end());
                wd.insert(wd.end(), ex.w_down.data().begin(), ex.w_down.data().end());
            }
            emit(q + "/w_gate", {cfg.num_experts, cfg.hidden, cfg.ffn_dim}, wg);
            emit(q + "/w_up", {cfg.num_experts, cfg.hidden, cfg.ffn_dim}, wu);
            emit(q + "/w_down", {cfg.num_experts, cfg.ffn_dim, cfg.hidden}, wd);
        }
        emit(p + "/final_norm", m.final_norm);
        emit(p + "/lm_head", m.lm_head);
        const ForwardOut fo = model_forward(m, batch);
        emit(p + "/logits", fo.logits);
        emit_scalar(p + "/aux", fo.aux_loss.item());
        RankGroup g2(2);
        emit(p + "/logits_sp2", hybrid_sp_forward(g2, m, batch));
        // packed documents (model.hpp:86-121, 374-405): the mixer runs per document, positions
        // restart at each boundary; the MoE sees all tokens
        const std::vector<int> d0(toks.begin(), toks.begin() + 100), d1(toks.begin() + 100, toks.begin() + 137),
            d2(toks.begin() + 137, toks.end());
        const PackedBatch packed = pack_sequences({d0, d1, d2});
        std::vector<double> bounds(packed.boundaries.begin(), packed.boundaries.end());
        emit(p + "/packed_bounds", {(int)bounds.size()}, bounds);
        const ForwardOut fp = model_forward(m, packed);
        emit(p + "/packed_logits", fp.logits);
        emit_scalar(p + "/packed_aux", fp.aux_loss.item());
        ++ci;
    }
}

int cmd_golden(const char* path) {
    g_out = fopen(path, "wb");
    if (!g_out) return 2;
    golden_lsm_small();
    golden_lsm_seq();
    golden_lsm_device();
    golden_lsm_grad();
    golden_lsm_rec_grad();
    golden_route();
    golden_moe();
    golden_sp();
    golden_model();
    fclose(g_out);
    return 0;
}

// ---- CPU baseline timers (SURVEY 8d "CPU baseline timing") ----
int cmd_bench_lsm(int argc, char** argv) {
    if (argc < 10) return 2;
    auto inst = instance_from_name(argv[2]);
    if (!inst) return 3;
    const int B = atoi(argv[3]), N = atoi(argv[4]), H = atoi(argv[5]), d = atoi(argv[6]);
    const int chunk = atoi(argv[7]);
    int threads = atoi(argv[8]);
    const double budget = atof(argv[9]);
    const double gate_mean = argc > 10 ? atof(argv[10]) : 0.0;
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    NoGradGuard ng;
    // f32 mode everywhere, gates included (BASELINE.md CPU-baseline plan step 4)
    const int heads = B * H;
    std::vector<std::thread> pool;
    std::vector<int> done(threads, 0);
    auto t0 = std::chrono::steady_clock::now();
    std::atomic<int> next{0};
    std::atomic<int> failed{0};
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w]() {
            Rng rng(100 + w);
            LsmSpec spec = LsmSpec::make(*inst, d, d, &rng, DType::f32);
            const Tensor q = Tensor::randn({N, d}, rng, 0.5, DType::f32);
            const Tensor k = Tensor::randn({N, d}, rng, 0.5, DType::f32);
            const Tensor v = Tensor::randn({N, d}, rng, 0.5, DType::f32);
            LsmGates g = LsmGates::random_for(spec, N, rng);
            for (Tensor* t : {&g.a_pre, &g.b_pre}) {
                if (!t->defined()) continue;
                std::vector<double> x = t->data();
                for (auto& e : x) e += gate_mean;
                *t = Tensor::from_data(t->shape(), x, DType::f32);
            }
            while (true) {
                const int h = next.fetch_add(1);
                if (h >= heads) break;
                double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (el > budget) break;
                try {
                    (void)lsm_forward_chunked(q, k, v, g, spec, chunk);
                } catch (const std::exception& e) {
                    fprintf(stderr, "reference error: %s\n", e.what());
                    failed = 1;
                    break;
                }
                done[w]++;
            }
        });
    for (auto& th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    int total = 0;
    for (int x : done) total += x;
    // heads_done sequences of N tokens each; tokens/s counts (token, all H heads) units
    const double tok_s = (double)total * N / (double)H / secs;
    printf("{\"heads_done\": %d, \"heads_total\": %d, \"seconds\": %.6f, \"threads\": %d, "
           "\"tokens_per_sec\": %.3f, \"failed\": %d}\n", total, heads, secs, threads, tok_s,
           failed.load());
    return failed.load() ? 1 : 0;
}

int cmd_bench_moe(int argc, char** argv) {
    if (argc < 9) return 2;
    const int T = atoi(argv[2]), hidden = atoi(argv[3]), ffn = atoi(argv[4]), E = atoi(argv[5]);
    const int K = atoi(argv[6]);
    int threads = atoi(argv[7]);
    const double budget = atof(argv[8]);
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    NoGradGuard ng;
    Rng rng(3);
    const MoeConfig cfg{E, K, hidden, ffn, 0.01};
    const MoeLayer layer = MoeLayer::init(cfg, rng, DType::f32);
    const int shard = 64;
    std::atomic<int> next{0};
    std::vector<int> done(threads, 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w]() {
            Rng r2(50 + w);
            const Tensor x = Tensor::randn({shard, hidden}, r2, 1.0, DType::f32);
            while (true) {
                const int s = next.fetch_add(1);
                if (s * shard >= T) break;
                double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (el > budget) break;
                (void)layer.forward(x);
                done[w] += shard;
            }
        });
    for (auto& th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    int total = 0;
    for (int x : done) total += x;
    printf("{\"tokens_done\": %d, \"tokens_total\": %d, \"seconds\": %.6f, \"threads\": %d, "
           "\"tokens_per_sec\": %.3f}\n", total, T, secs, threads, total / secs);
    return 0;
}

// One Linear-MoE block of the reference model (the loop body of model_forward, model.hpp:387-397:
// rms_norm -> mixer per document -> residual -> rms_norm -> MoeLayer -> residual), f32 mode, no
// tape, documents of doc_len tokens processed independently by `threads` workers.  Prints
// tokens/s over the documents finished within the budget.
int cmd_bench_block(int argc, char** argv) {
    if (argc < 12) return 2;
    auto inst = instance_from_name(argv[2]);
    if (!inst) return 3;
    const char kind = argv[3][0];
    const int len = atoi(argv[4]), hidden = atoi(argv[5]), heads = atoi(argv[6]), ffn = atoi(argv[7]);
    const int E = atoi(argv[8]), K = atoi(argv[9]);
    int threads = atoi(argv[10]);
    const double budget = atof(argv[11]);
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    NoGradGuard ng;
    ModelConfig cfg;
    cfg.hidden = hidden;
    cfg.ffn_dim = ffn;
    cfg.num_heads = heads;
    cfg.num_layers = 1;
    cfg.num_experts = E;
    cfg.num_active = K;
    cfg.vocab_size = 256;
    cfg.instance = *inst;
    cfg.pattern = std::string(1, kind);
    cfg.max_seq_len = len;
    cfg.dtype = DType::f32;
    Rng rng(5);
    const Model m = build_model(cfg, rng);
    const Block& b = m.blocks[0];
    std::vector<int> done(threads, 0);
    std::atomic<int> failed{0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w]() {
            Rng r2(70 + w);
            Tensor x = Tensor::randn({len, hidden}, r2, 1.0, DType::f32);
            try {
                while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < budget) {
                    const Tensor h = rms_norm(x, b.norm_mixer, cfg.norm_eps);
                    Tensor y = add(x, b.mixer_forward(h));
                    const Tensor h2 = rms_norm(y, b.norm_moe, cfg.norm_eps);
                    auto out = b.moe.forward(h2);
                    y = add(y, out.first);
                    done[w] += len;
                }
            } catch (const std::exception&) {
                failed.fetch_add(1);
            }
        });
    for (auto& th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    int total = 0;
    for (int x : done) total += x;
    printf("{\"tokens_done\": %d, \"seconds\": %.6f, \"threads\": %d, \"failed\": %d, "
           "\"tokens_per_sec\": %.3f}\n", total, secs, threads, failed.load(), total / secs);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: ref_driver golden <out> | bench-lsm ... | bench-moe ...\n");
        return 2;
    }
    try {
        if (!strcmp(argv[1], "golden") && argc >= 3) return cmd_golden(argv[2]);
        if (!strcmp(argv[1], "bench-lsm")) return cmd_bench_lsm(argc, argv);
        if (!strcmp(argv[1], "bench-moe")) return cmd_bench_moe(argc, argv);
        if (!strcmp(argv[1], "bench-block")) return cmd_bench_block(argc, argv);
    } catch (const std::exception& e) {
        fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 2;
}
