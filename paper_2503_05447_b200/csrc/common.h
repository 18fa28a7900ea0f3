// common.h -- host-side helpers shared by the C-ABI implementation files.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/lmoe_cuda.h"

namespace lmoe_host {

// Thrown inside the library, converted to (status, thread-local message) at the C boundary.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void set_last_error(const std::string& msg);

#define LMOE_CUDA_CHECK(x)                                                                   \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess)                                                               \
            throw ::lmoe_host::Error(LMOE_ERR_CUDA, std::string("CUDA error: ") +            \
                                                        cudaGetErrorString(e_) + " at " +    \
                                                        __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

// Tensor map for a 4-D row-major tensor [d3][d2][d1][d0] (d0 innermost), SWIZZLE_128B,
// box {box0, 1, box2, 1}.
CUtensorMap make_tmap_4d(const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
                         uint64_t d1, uint64_t d2, uint64_t d3, uint32_t box0, uint32_t box2,
                         uint64_t d2_stride = 0 /* elements of dim 2 per dim-3 step; 0 = d2 */,
                         uint64_t row_stride = 0 /* elements per dim-2 step; 0 = d0 * d1 */);
// 3-D row-major tensor [d2][d1][d0], SWIZZLE_128B, box {box0, box1, 1}.
CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
                         uint64_t d1, uint64_t d2, uint32_t box0, uint32_t box1);
// 2-D row-major tensor [rows][cols], SWIZZLE_128B, box {box_cols, box_rows}.
CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dt, int esize, uint64_t cols,
                         uint64_t rows, uint64_t row_stride_elems, uint32_t box_cols,
                         uint32_t box_rows);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }


int num_sms();

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LMOE_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return LMOE_ERR_ARG;
    }
}

// Launch counters (kernels of this library enqueued since process start).
extern std::atomic<long long> g_launch_count;

}  // namespace lmoe_host

namespace lmoe_dev {
cudaError_t ensure_smem(const void* fn, int bytes);  // common.cu; see lsm_launch.h
}
