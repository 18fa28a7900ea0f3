// common.cu -- C-ABI plumbing: thread-local last error, TMA descriptor encoding, device info.
#include <mutex>
#include <set>
#include <utility>

#include "common.h"

namespace lmoe_host {

static thread_local std::string t_last_error;
std::atomic<long long> g_launch_count{0};

void set_last_error(const std::string& msg) { t_last_error = msg; }

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, []() {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    if (!fn) throw Error(LMOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_tmap_4d(const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
                         uint64_t d1, uint64_t d2, uint64_t d3, uint32_t box0, uint32_t box2,
                         uint64_t d2_stride, uint64_t row_stride) {
    CUtensorMap m;
    if (d2_stride == 0) d2_stride = d2;
    if (row_stride == 0) row_stride = d0 * d1;
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t strides[3] = {d0 * esize, row_stride * esize, row_stride * d2_stride * esize};
    cuuint32_t box[4] = {box0, 1, box2, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, dt, 4, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(LMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
                         uint64_t d1, uint64_t d2, uint32_t box0, uint32_t box1) {
    CUtensorMap m;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * esize, d0 * d1 * esize};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, dt, 3, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(LMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dt, int esize, uint64_t cols,
                         uint64_t rows, uint64_t row_stride_elems, uint32_t box_cols,
                         uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {row_stride_elems * esize};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(LMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<int> cache[64] = {};
    if (dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load();
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev].store(n);
    }
    return n;
}

}  // namespace lmoe_host

namespace lmoe_dev {
cudaError_t ensure_smem(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}
}  // namespace lmoe_dev

extern "C" const char* lmoe_last_error(void) { return lmoe_host::t_last_error.c_str(); }
extern "C" const char* lmoe_version(void) { return "lmoe-b200 0.1 (sm_100a)"; }
extern "C" long long lmoe_launch_count(void) { return lmoe_host::g_launch_count.load(); }
