// lsm_cpp_api.cpp -- exercises the C++ drop-in header (include/lmoe/cuda.hpp) the way a
// reference caller would: lsm_forward_chunked with device buffers, compared against the
// token recurrence of lsm.hpp:335-441 evaluated in double on the host.  Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "lmoe/cuda.hpp"

int main() {
    using namespace lmoe::cuda;
    const int N = 700, H = 2, D = 64;  // fp32 path (tf32 tensor cores), ragged last chunk
    std::mt19937 gen(7);
    std::normal_distribution<float> nd(0.f, 0.5f);
    std::vector<float> q(N * H * D), k(N * H * D), v(N * H * D), o(N * H * D);
    for (auto* a : {&q, &k, &v})
        for (auto& x : *a) x = nd(gen);
    float *dq, *dk, *dv, *dout, *dM;
    const size_t bytes = q.size() * 4;
    cudaMalloc(&dq, bytes); cudaMalloc(&dk, bytes); cudaMalloc(&dv, bytes); cudaMalloc(&dout, bytes);
    cudaMalloc(&dM, H * D * D * 4);
    cudaMemcpy(dq, q.data(), bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, k.data(), bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), bytes, cudaMemcpyHostToDevice);

    LsmView x;
    x.B = 1; x.N = N; x.H = H; x.D = D; x.dtype = LMOE_F32;
    x.q = dq; x.k = dk; x.v = dv; x.o = dout;
    const LsmSpec spec = LsmSpec::make(LMOE_RETNET);
    MemoryState fs;
    fs.M = dM;
    try {
        lsm_forward_chunked(x, LsmGates{}, spec, 16, &fs);
    } catch (const Error& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
    cudaMemcpy(o.data(), dout, bytes, cudaMemcpyDeviceToHost);

    // reference recurrence: M_s = a M_{s-1} + k_s v_s^T, o_s = q_s M_s
    double worst = 0.0;
    for (int h = 0; h < H; ++h) {
        std::vector<double> M(D * D, 0.0);
        double maxref = 0.0, maxerr = 0.0;
        for (int t = 0; t < N; ++t) {
            const float* qt = &q[(t * H + h) * D];
            const float* kt = &k[(t * H + h) * D];
            const float* vt = &v[(t * H + h) * D];
            for (int i = 0; i < D; ++i)
                for (int j = 0; j < D; ++j) M[i * D + j] = spec.scalar_decay * M[i * D + j] + (double)kt[i] * vt[j];
            for (int j = 0; j < D; ++j) {
                double acc = 0.0;
                for (int i = 0; i < D; ++i) acc += (double)qt[i] * M[i * D + j];
                maxref = std::fmax(maxref, std::fabs(acc));
                maxerr = std::fmax(maxerr, std::fabs(acc - o[(t * H + h) * D + j]));
            }
        }
        worst = std::fmax(worst, maxerr / maxref);
    }
    // the reference's error text survives the boundary
    bool text_ok = false;
    try {
        LsmSpec bad = LsmSpec::make(LMOE_MAMBA2);
        bad.use_normalizer = true;
        lsm_forward_chunked(x, LsmGates{}, bad, 16);
    } catch (const Error& e) {
        text_ok = std::string(e.what()) == "LsmSpec: normalizer unsupported for instance mamba2";
    }
    // backward through the drop-in API: lsm_backward_chunked (the tape's VJP) with dO = 1 /
    // N-scaled random, dv checked against dv_s = sum_{t >= s} a^{t-s} (q_t . k_s) dO_t, and the
    // SP backward at world 1 (sp_lsm_masked_rank_backward) equal to it
    std::vector<float> gO(N * H * D);
    for (auto& x : gO) x = nd(gen);
    float *ddO, *gq, *gk, *gv, *sq, *sk, *sv;
    for (float** p : {&ddO, &gq, &gk, &gv, &sq, &sk, &sv}) cudaMalloc(p, bytes);
    cudaMemcpy(ddO, gO.data(), bytes, cudaMemcpyHostToDevice);
    double worst_bwd = 1.0, worst_sp = 1.0;
    try {
        LsmGrads g;
        g.dq = gq; g.dk = gk; g.dv = gv;
        lsm_backward_chunked(x, LsmGates{}, spec, ddO, g);
        LsmGrads gs;
        gs.dq = sq; gs.dk = sk; gs.dv = sv;
        sp_lsm_masked_rank_backward(nullptr, 0, 1, x, LsmGates{}, spec, ddO, gs);
        std::vector<float> hv(N * H * D), hs(N * H * D);
        cudaMemcpy(hv.data(), gv, bytes, cudaMemcpyDeviceToHost);
        cudaMemcpy(hs.data(), sv, bytes, cudaMemcpyDeviceToHost);
        worst_bwd = worst_sp = 0.0;
        for (int h = 0; h < H; ++h) {
            double maxref = 0.0, maxerr = 0.0, maxsp = 0.0;
            for (int s0 = 0; s0 < N; s0 += 7) {  // every 7th row keeps the host reference cheap
                std::vector<double> acc(D, 0.0);
                double w = 1.0;
                for (int t = s0; t < N; ++t, w *= spec.scalar_decay) {
                    double qk = 0.0;
                    for (int i = 0; i < D; ++i) qk += (double)q[(t * H + h) * D + i] * k[(s0 * H + h) * D + i];
                    for (int j = 0; j < D; ++j) acc[j] += w * qk * gO[(t * H + h) * D + j];
                }
                for (int j = 0; j < D; ++j) {
                    const size_t e = (size_t)(s0 * H + h) * D + j;
                    maxref = std::fmax(maxref, std::fabs(acc[j]));
                    maxerr = std::fmax(maxerr, std::fabs(acc[j] - hv[e]));
                    maxsp = std::fmax(maxsp, std::fabs((double)hs[e] - hv[e]));
                }
            }
            worst_bwd = std::fmax(worst_bwd, maxerr / maxref);
            worst_sp = std::fmax(worst_sp, maxsp / maxref);
        }
    } catch (const Error& e) {
        std::printf("backward error: %s\n", e.what());
    }
    std::printf("cpp api: norm-rel err %.3e (tol 1e-3), error text %s, backward dv %.3e (tol 2e-3), "
                "SP world-1 vs local %.3e\n", worst, text_ok ? "ok" : "MISMATCH", worst_bwd, worst_sp);
    cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(dM);
    for (float* p : {ddO, gq, gk, gv, sq, sk, sv}) cudaFree(p);
    return (worst < 1e-3 && text_ok && worst_bwd < 2e-3 && worst_sp < 1e-5) ? 0 : 1;
}
