// tc_probe.cu -- single-tile tcgen05 probes (debug tool): D[128 x N] = A[128 x K] * B[K x N]
// with TMA-loaded SW128 operands, for bf16/tf32 and K-/MN-major operands.  Prints max error
// vs a host fp64 reference.   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2
//   -I paper_2503_05447_b200/csrc tools/tc_probe.cu -o /tmp/tc_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>

#include "ptx.cuh"
using namespace lmoe_dev;

// A: 128 x K (K-major: rows of K; MN-major: stored K rows of 128 M)   B: K x N
// Operands are plain SW128 images written by the host into smem-layout buffers (no TMA), so
// the probe isolates descriptors + MMA.
template <bool kTF32>
__global__ void probe(const uint8_t* a_img, const uint8_t* b_img, int a_bytes, int b_bytes,
                      int K, int N, int a_major, int b_major, uint32_t lbo_a, uint32_t lbo_b,
                      float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    uint8_t* sa = smem;
    uint8_t* sb = smem + ((a_bytes + 1023) / 1024) * 1024;
    for (int i = threadIdx.x * 16; i < a_bytes; i += blockDim.x * 16) *(uint4*)(sa + i) = *(const uint4*)(a_img + i);
    for (int i = threadIdx.x * 16; i < b_bytes; i += blockDim.x * 16) *(uint4*)(sb + i) = *(const uint4*)(b_img + i);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp_id() == 0) tmem_alloc<256>(&tm);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int esz = kTF32 ? 4 : 2;
    const int kstep = 32 / esz;  // elements per MMA K
    if (threadIdx.x == 0) {
        uint32_t idesc = umma_idesc(kTF32 ? 2 : 1, a_major, b_major, 128, N);
        for (int kk = 0; kk < K / kstep; ++kk) {
            uint32_t aoff, boff;
            if (a_major == 0) aoff = (kk * 32 / 128) * (128 * 128) + (kk * 32 % 128);  // K-major: 128 rows per block
            else aoff = kk * kstep * 128;
            if (b_major == 0) boff = (kk * 32 / 128) * (N * 128) + (kk * 32 % 128);
            else boff = kk * kstep * 128;
            uint64_t ad = umma_desc_sw128(smem_u32(sa) + aoff, a_major ? lbo_a : 16, 1024);
            uint64_t bd = umma_desc_sw128(smem_u32(sb) + boff, b_major ? lbo_b : 16, 1024);
            if (kTF32) mma_ss_tf32(tm, ad, bd, idesc, kk > 0);
            else mma_ss_f16(tm, ad, bd, idesc, kk > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (warp_id() < 4) {
        int row = warp_id() * 32 + lane_id();
        for (int c = 0; c < N; c += 32) {
            uint32_t r[32];
            tmem_ld32(tm + ((uint32_t)(warp_id() * 32) << 16) + c, r);
            tmem_wait_ld();
            for (int j = 0; j < 32; ++j) out[row * N + c + j] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp_id() == 0) tmem_dealloc<256>(tm);
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7FFF + ((u >> 16) & 1); return u >> 16; }
static float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

// write element (r, c) of a [rows x cols] matrix, "cols" contiguous, into SW128 blocks of 128 B
// rows: block = c / epb; block stride = rows*128
static void put(std::vector<uint8_t>& img, int rows, int esz, int r, int c, float v) {
    int epb = 128 / esz, blk = c / epb, cin = c % epb;
    int chunk = (cin * esz) / 16, within = (cin * esz) % 16;
    size_t off = (size_t)blk * rows * 128 + r * 128 + ((chunk ^ (r & 7)) << 4) + within;
    if (esz == 2) { uint16_t b = f2bf(v); memcpy(&img[off], &b, 2); }
    else memcpy(&img[off], &v, 4);
}

template <bool kTF32>
static void run(int K, int N, int a_major, int b_major) {
    const int M = 128, esz = kTF32 ? 4 : 2;
    std::vector<float> A(M * K), B(K * N);
    srand(1);
    for (auto& x : A) { x = (rand() % 17 - 8) / 8.0f; }
    for (auto& x : B) { x = (rand() % 17 - 8) / 8.0f; }
    // A image
    std::vector<uint8_t> ai, bi;
    int a_bytes, b_bytes;
    uint32_t lbo_a = 0, lbo_b = 0;
    if (a_major == 0) {  // [M rows][K]
        a_bytes = M * K * esz; ai.assign(a_bytes, 0);
        for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) put(ai, M, esz, m, k, A[m * K + k]);
    } else {  // [K rows][M]
        a_bytes = K * M * esz; ai.assign(a_bytes, 0);
        for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) put(ai, K, esz, k, m, A[m * K + k]);
        lbo_a = K * 128;
    }
    if (b_major == 0) {  // [N rows][K]
        b_bytes = N * K * esz; bi.assign(b_bytes, 0);
        for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) put(bi, N, esz, n, k, B[k * N + n]);
    } else {  // [K rows][N]
        b_bytes = K * N * esz; bi.assign(b_bytes, 0);
        for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) put(bi, K, esz, k, n, B[k * N + n]);
        lbo_b = K * 128;
    }
    uint8_t *da, *db; float* dout;
    cudaMalloc(&da, a_bytes); cudaMalloc(&db, b_bytes); cudaMalloc(&dout, M * N * 4);
    cudaMemcpy(da, ai.data(), a_bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(db, bi.data(), b_bytes, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, M * N * 4);
    int smem = ((a_bytes + 1023) / 1024) * 1024 + b_bytes + 1024;
    cudaFuncSetAttribute(probe<kTF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<kTF32><<<1, 128, smem>>>(da, db, a_bytes, b_bytes, K, N, a_major, b_major, lbo_a, lbo_b, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(M * N);
    cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[k * N + n];
        maxerr = std::max(maxerr, std::fabs(ref - out[m * N + n]));
        maxref = std::max(maxref, std::fabs(ref));
    }
    printf("%s K=%3d N=%3d a_major=%d b_major=%d : err=%s maxerr=%.3e maxref=%.3e out[0]=%.3f\n",
           kTF32 ? "tf32" : "bf16", K, N, a_major, b_major, cudaGetErrorString(e), maxerr, maxref, out[0]);
    cudaFree(da); cudaFree(db); cudaFree(dout);
}


template <bool kTF32>
__global__ void probe_ts(const float* A, const uint8_t* b_img, int b_bytes, int K, int N, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x * 16; i < b_bytes; i += blockDim.x * 16) *(uint4*)(smem + i) = *(const uint4*)(b_img + i);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp_id() == 0) tmem_alloc<512>(&tm);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // A -> TMEM columns [256, ...): row = lane of quarter
    const int row = warp_id() * 32 + lane_id();
    const uint32_t ta = tm + 256 + ((uint32_t)(warp_id() * 32) << 16);
    if (kTF32) {
        for (int c0 = 0; c0 < K; c0 += 32) {
            uint32_t r[32];
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(A[row * K + c0 + j]);
            tmem_st32(ta + c0, r);
        }
    } else {
        for (int c0 = 0; c0 < K; c0 += 64) {
            uint32_t r[32];
            for (int j = 0; j < 32; ++j) r[j] = pack_bf16(A[row * K + c0 + 2 * j], A[row * K + c0 + 2 * j + 1]);
            tmem_st32(ta + c0 / 2, r);
        }
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        uint32_t idesc = umma_idesc(kTF32 ? 2 : 1, 0, 0, 128, N);
        const int kstep = kTF32 ? 8 : 16;
        for (int kk = 0; kk < K / kstep; ++kk) {
            uint32_t boff = (kk * 32 / 128) * (N * 128) + (kk * 32 % 128);
            uint64_t bd = umma_desc_sw128(smem_u32(smem) + boff, 16, 1024);
            if (kTF32) mma_ts_tf32(tm, tm + 256 + kk * 8, bd, idesc, kk > 0);
            else mma_ts_f16(tm, tm + 256 + kk * 8, bd, idesc, kk > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        tmem_ld32(tm + ((uint32_t)(warp_id() * 32) << 16) + c, r);
        tmem_wait_ld();
        for (int j = 0; j < 32; ++j) out[row * N + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp_id() == 0) tmem_dealloc<512>(tm);
}

template <bool kTF32>
static void run_ts(int K, int N) {
    const int M = 128, esz = kTF32 ? 4 : 2;
    std::vector<float> A(M * K), B(K * N);
    srand(2);
    for (auto& x : A) x = (rand() % 17 - 8) / 8.0f;
    for (auto& x : B) x = (rand() % 17 - 8) / 8.0f;
    std::vector<uint8_t> bi(N * K * esz, 0);
    for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) put(bi, N, esz, n, k, B[k * N + n]);
    float *dA, *dout; uint8_t* db;
    cudaMalloc(&dA, M * K * 4); cudaMalloc(&db, bi.size()); cudaMalloc(&dout, M * N * 4);
    cudaMemcpy(dA, A.data(), M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice);
    int smem = (int)bi.size() + 1024;
    cudaFuncSetAttribute(probe_ts<kTF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_ts<kTF32><<<1, 128, smem>>>(dA, db, (int)bi.size(), K, N, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(M * N);
    cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[k * N + n];
        maxerr = std::max(maxerr, std::fabs(ref - out[m * N + n]));
        maxref = std::max(maxref, std::fabs(ref));
    }
    printf("TS %s K=%3d N=%3d : err=%s maxerr=%.3e maxref=%.3e\n", kTF32 ? "tf32" : "bf16", K, N,
           cudaGetErrorString(e), maxerr, maxref);
}

int main() {
    run_ts<false>(128, 128);
    run_ts<true>(128, 64);
    run_ts<true>(64, 64);
    return 0;

    for (int am = 0; am < 2; ++am) for (int bm = 0; bm < 2; ++bm) {
        run<false>(128, 128, am, bm);
        run<true>(64, 64, am, bm);
        run<true>(64, 128, am, bm);
    }
    return 0;
}
