// tensor_bridge_test.cpp -- calls the reference implementation (the read-only reference headers,
// /root/reference/proj/include/lmoe) and the Tensor-level drop-in (include/lmoe/cuda_tensor.hpp,
// B200 through liblmoe_cuda.so) on the SAME lmoe::Tensor inputs and compares results and error
// texts.  Test infrastructure only: built by oracle/Makefile into oracle/_ref/ (it needs the
// reference headers, which exist only in the build container), run on the GPU box by
// tests/test_tensor_bridge_gpu.py.  Exit code 0 = every check passed.
//
// Checks (reference test each one restates):
//   lsm_forward_chunked outputs + final state, 7 instances   test_lsm.cpp:200-219 (chunked == sequential)
//   chunk_size / normaliser error texts                      lsm.hpp:672, 199-201; test_lsm.cpp:237-259
//   route KAT ties + random ids / gates / probs              test_moe.cpp:9-47
//   "route: bad top_k"                                       moe.hpp:63
//   MoeLayer::forward y and aux                              test_moe.cpp:64-82, acceptance.cpp:254-290
//   sp_lsm_masked_rank over a 1-rank NCCL communicator       parallel.hpp:303-376, test_parallel.cpp:150-176
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "lmoe/lsm.hpp"
#include "lmoe/moe.hpp"
#include "lmoe/parallel.hpp"
#include "lmoe/cuda_tensor.hpp"

namespace {

int g_fail = 0;

void report(const std::string& name, bool ok, double err = 0.0, double tol = 0.0) {
    std::printf("%s %s err=%.3e tol=%.1e\n", ok ? "PASS" : "FAIL", name.c_str(), err, tol);
    if (!ok) ++g_fail;
}

double norm_rel(const lmoe::Tensor& got, const lmoe::Tensor& want) {
    const auto& a = got.data();
    const auto& b = want.data();
    if (a.size() != b.size()) return INFINITY;
    double num = 0.0, den = 1e-300;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, std::fabs(a[i] - b[i]));
        den = std::max(den, std::fabs(b[i]));
    }
    return num / den;
}

template <typename F>
std::string error_text(F&& f) {
    try {
        f();
    } catch (const std::exception& e) {
        return e.what();
    }
    return "<no error>";
}

// round every element to the nearest bf16 value (the MoE test feeds both sides bf16-exact
// operands so routing decisions do not depend on operand rounding)
lmoe::Tensor bf16_exact(const lmoe::Tensor& t) {
    std::vector<double> d(t.data());
    for (auto& x : d) x = lmoe::cuda::bridge::from_bf16(lmoe::cuda::bridge::to_bf16((float)x));
    return lmoe::Tensor::from_data(t.shape(), std::move(d), t.dtype());
}

void test_lsm() {
    struct Case {
        const char* name;
        double tol;
    };
    const Case cases[] = {{"bla", 1e-3},   {"rebased", 1e-3}, {"lightning", 1e-3}, {"retnet", 1e-3},
                          {"mamba2", 1e-3}, {"gla", 2e-2},     {"hgrn2", 2e-2}};
    const int N = 300, d = 8;
    for (const Case& c : cases) {
        lmoe::Rng rng(11);
        const lmoe::LsmInstance inst = *lmoe::instance_from_name(c.name);
        const lmoe::LsmSpec spec = lmoe::LsmSpec::make(inst, d, d, &rng);
        const lmoe::Tensor q = lmoe::Tensor::randn({N, d}, rng, 0.5);
        const lmoe::Tensor k = lmoe::Tensor::randn({N, d}, rng, 0.5);
        const lmoe::Tensor v = lmoe::Tensor::randn({N, d}, rng, 0.5);
        const lmoe::LsmGates g = lmoe::LsmGates::random_for(spec, N, rng);
        lmoe::MemoryState fs_ref, fs;
        const lmoe::Tensor want = lmoe::lsm_forward_chunked(q, k, v, g, spec, 16, &fs_ref);
        const lmoe::Tensor got = lmoe::cuda::lsm_forward_chunked(q, k, v, g, spec, 16, &fs);
        const double e = norm_rel(got, want), eM = norm_rel(fs.M, fs_ref.M);
        report(std::string("lsm_forward_chunked/") + c.name, e < c.tol, e, c.tol);
        report(std::string("final_state.M/") + c.name, eM < c.tol, eM, c.tol);
        report(std::string("final_state.step/") + c.name, fs.step == fs_ref.step, 0, 0);
        if (spec.use_normalizer) {
            const double ez = norm_rel(fs.z, fs_ref.z);
            report(std::string("final_state.z/") + c.name, ez < c.tol, ez, c.tol);
        }
        if (inst == lmoe::LsmInstance::Lightning) {
            const std::string a = error_text([&] { lmoe::lsm_forward_chunked(q, k, v, g, spec, 0); });
            const std::string b = error_text([&] { lmoe::cuda::lsm_forward_chunked(q, k, v, g, spec, 0); });
            report("error_text/chunk_size: " + b, a == b && a == "lsm_forward_chunked: chunk_size must be >= 1");
        }
        if (inst == lmoe::LsmInstance::Mamba2) {
            lmoe::LsmSpec bad = spec;
            bad.use_normalizer = true;
            const std::string a = error_text([&] { lmoe::lsm_forward_chunked(q, k, v, g, bad, 16); });
            const std::string b = error_text([&] { lmoe::cuda::lsm_forward_chunked(q, k, v, g, bad, 16); });
            report("error_text/normalizer: " + b, a == b && a == "LsmSpec: normalizer unsupported for instance mamba2");
        }
    }
}

void test_route() {
    // test_moe.cpp:9-20: ties go to the lower id, ids ascending
    const lmoe::Tensor kat = lmoe::Tensor::from_data({2, 4}, {0.1, 0.9, 0.9, 0.2, 0.5, 0.5, 0.5, 0.5});
    const lmoe::RoutingDecision a = lmoe::route(kat, 2), b = lmoe::cuda::route(kat, 2);
    report("route/kat_ids", a.expert_ids == b.expert_ids && b.expert_ids[0] == std::vector<int>{1, 2} &&
                                b.expert_ids[1] == std::vector<int>{0, 1});
    const double eg = norm_rel(b.gates, a.gates);
    report("route/kat_gates", eg < 1e-6, eg, 1e-6);
    // random logits, fp32-representable so both sides rank identical values
    lmoe::Rng rng(3);
    const int T = 257, E = 16, K = 4;
    std::vector<double> lg((size_t)T * E);
    for (auto& x : lg) x = (double)(float)(rng.uniform() * 4.0 - 2.0);
    const lmoe::Tensor logits = lmoe::Tensor::from_data({T, E}, lg);
    const lmoe::RoutingDecision r = lmoe::route(logits, K), c = lmoe::cuda::route(logits, K);
    report("route/random_ids_bit_exact", r.expert_ids == c.expert_ids);
    const double e1 = norm_rel(c.gates, r.gates), e2 = norm_rel(c.full_probs, r.full_probs);
    report("route/random_gates", e1 < 1e-5, e1, 1e-5);
    report("route/random_full_probs", e2 < 1e-5, e2, 1e-5);
    const double aux_ref = lmoe::load_balance_loss(r).item(), aux = lmoe::load_balance_loss(c).item();
    report("route/load_balance_loss", std::fabs(aux - aux_ref) < 1e-5 * aux_ref, std::fabs(aux - aux_ref), 1e-5);
    const std::string ta = error_text([&] { lmoe::route(logits, 0); });
    const std::string tb = error_text([&] { lmoe::cuda::route(logits, 0); });
    report("error_text/route: " + tb, ta == tb && ta == "route: bad top_k");
}

void test_moe() {
    lmoe::Rng rng(21);
    const lmoe::MoeConfig cfg{8, 2, 16, 24, 0.01};
    lmoe::MoeLayer layer = lmoe::MoeLayer::init(cfg, rng, lmoe::DType::f64);
    layer.router = bf16_exact(layer.router);
    for (auto& e : layer.experts) {
        e.w_gate = bf16_exact(e.w_gate);
        e.w_up = bf16_exact(e.w_up);
        e.w_down = bf16_exact(e.w_down);
    }
    const lmoe::Tensor x = bf16_exact(lmoe::Tensor::randn({96, 16}, rng, 1.0));
    const auto [y_ref, aux_ref] = layer.forward(x);
    const auto [y, aux] = lmoe::cuda::moe_forward(layer, x);
    const double e = norm_rel(y, y_ref);
    report("MoeLayer::forward/y", e < 2e-2, e, 2e-2);
    const double ea = std::fabs(aux.item() - aux_ref.item()) / std::fabs(aux_ref.item());
    report("MoeLayer::forward/aux", ea < 1e-4, ea, 1e-4);
}

void test_sp() {
    char id[128];
    void* comm = nullptr;
    if (lmoe_nccl_unique_id(id) != LMOE_OK || lmoe_nccl_comm_init(&comm, 1, 0, id) != LMOE_OK) {
        report("sp/nccl_comm_init", false);
        return;
    }
    for (const char* name : {"retnet", "mamba2"}) {
        lmoe::Rng rng(5);
        const lmoe::LsmSpec spec = lmoe::LsmSpec::make(*lmoe::instance_from_name(name), 8, 8, &rng);
        const int N = 200;
        const lmoe::Tensor q = lmoe::Tensor::randn({N, 8}, rng, 0.5);
        const lmoe::Tensor k = lmoe::Tensor::randn({N, 8}, rng, 0.5);
        const lmoe::Tensor v = lmoe::Tensor::randn({N, 8}, rng, 0.5);
        const lmoe::LsmGates g = lmoe::LsmGates::random_for(spec, N, rng);
        lmoe::RankGroup group(1);
        const lmoe::Tensor want = lmoe::sp_forward_masked(group, q, k, v, g, spec);
        const lmoe::Tensor got = lmoe::cuda::sp_lsm_masked_rank(comm, 0, 1, q, k, v, g, spec);
        const double e = norm_rel(got, want);
        report(std::string("sp_lsm_masked_rank(nccl 1 rank)/") + name, e < 1e-3, e, 1e-3);
    }
    lmoe_nccl_comm_destroy(comm);
}

}  // namespace

int main() {
    lmoe::NoGradGuard ng;
    test_lsm();
    test_route();
    test_moe();
    test_sp();
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
