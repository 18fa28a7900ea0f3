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
    std::printf("cpp api: norm-rel err %.3e (tol 1e-3), error text %s\n", worst, text_ok ? "ok" : "MISMATCH");
    cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(dM);
    return (worst < 1e-3 && text_ok) ? 0 : 1;
}
