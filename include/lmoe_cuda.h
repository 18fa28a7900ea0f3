/*
 * lmoe_cuda.h -- C ABI of the B200 (sm_100a) Linear-MoE hot path.
 *
 * The reference (/root/reference/proj/include/lmoe, header-only C++20) has no FFI layer;
 * its hot path is a set of free functions in namespace lmoe.  Each entry point below
 * replaces one of them (cited per function) with plain pointers and sizes: no C++ or
 * torch types cross this boundary.  include/lmoe/cuda.hpp layers the reference's C++
 * names, argument meaning and std::runtime_error texts on top of it.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers owned by the caller; the library never
 *    allocates inside a hot call.  Scratch comes from a caller-provided workspace whose
 *    size is returned by the matching *_workspace_size query.
 *  - Layouts: per-head activations are [B, N, H, D] row-major (the reference's (N x H*D)
 *    projection per batch row, model.hpp:234-243); states are fp32 [B, H, D, D] and
 *    normaliser states fp32 [B, H, D].
 *  - Work is enqueued on `stream`; calls return LMOE_OK or an error code, and
 *    lmoe_last_error() returns the thread-local message (the reference's error text where
 *    one exists).  With LMOE_FLAG_CHECK the call synchronises the stream and reports
 *    device-detected conditions (degenerate normaliser, non-finite state) the way the
 *    reference throws them; without it the call is fully asynchronous.
 */
#ifndef LMOE_CUDA_H
#define LMOE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lmoe_stream_t; /* == cudaStream_t */

enum lmoe_status {
    LMOE_OK = 0,
    LMOE_ERR_ARG = 1,          /* invalid argument / unsupported shape            */
    LMOE_ERR_SHAPE = 2,        /* "shape mismatch in ..."                          */
    LMOE_ERR_DEGENERATE = 3,   /* "degenerate normalizer in instance <name>"       */
    LMOE_ERR_NONFINITE = 4,    /* "non-finite memory state in instance <name>"     */
    LMOE_ERR_CUDA = 5,
    LMOE_ERR_NCCL = 6,
    LMOE_ERR_UNSUPPORTED = 7   /* instance / kind outside the accelerated scope    */
};

typedef enum lmoe_dtype { LMOE_F32 = 0, LMOE_BF16 = 1 } lmoe_dtype;

/* lmoe::LsmInstance numbering (lsm.hpp:30-48) */
enum lmoe_instance {
    LMOE_BLA = 0, LMOE_LIGHTNING = 1, LMOE_RETNET = 2, LMOE_GLA = 3, LMOE_REBASED = 6,
    LMOE_MAMBA2 = 13, LMOE_HGRN2 = 14, LMOE_RWKV6 = 15
};
enum lmoe_feature_map { LMOE_FM_IDENTITY = 0, LMOE_FM_ELU1 = 1, LMOE_FM_SQUARED = 2 };
enum lmoe_flags { LMOE_FLAG_CHECK = 1, LMOE_FLAG_TIMING = 2 };

/* Mirrors the fields of lmoe::LsmSpec (lsm.hpp:126-140) that the separable kinds use.
 * Static per-head parameters (Mamba2 a_raw) are passed as arrays. */
typedef struct lmoe_lsm_desc {
    int instance;        /* enum lmoe_instance                                      */
    int feature_map;     /* enum lmoe_feature_map                                   */
    int use_normalizer;  /* 0 / 1                                                   */
    float scalar_decay;  /* Lightning / RetNet a                                    */
    int chunk_size;      /* reference chunk_size (>= 1).  The device tile is 128
                            tokens; outputs are chunk-size invariant up to rounding  */
    int flags;           /* LMOE_FLAG_*                                             */
} lmoe_lsm_desc;

const char* lmoe_last_error(void);
const char* lmoe_version(void);

/* ---------------------------------------------------------------------------------------
 * LSM forward.  Replaces lsm_forward_chunked(q, k, v, gates, spec, chunk_size,
 * &final_state) (lsm.hpp:668-708) for every (b, h) at once, including the separable
 * closed form kern::chunk_forward_separable (lsm.hpp:554-598).
 *   q, k, v, o   : [B,N,H,D] dtype (bf16: D = 128; f32: D = 64, tf32 tensor cores)
 *   b_pre        : [B,N,H] fp32, Mamba2 gate pre-activation (LsmGates::b_pre) or NULL
 *   a_pre        : [B,N,H,D] dtype, TokenVector gate pre-activation (LsmGates::a_pre)
 *   a_raw        : [H] fp32, Mamba2 LsmSpec::mamba2_a_raw per head, or NULL
 *   M0, z0       : optional initial state (NULL = MemoryState::fresh)
 *   M_out, z_out : optional final state (the reference's final_state out-parameter)
 * ------------------------------------------------------------------------------------- */
size_t lmoe_lsm_fwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                   lmoe_dtype dtype);
int lmoe_lsm_fwd(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                 const void* q, const void* k, const void* v, const void* a_pre,
                 const float* b_pre, const float* a_raw, const float* M0, const float* z0,
                 void* o, float* M_out, float* z_out, void* workspace, size_t workspace_bytes,
                 lmoe_stream_t stream);

/* Number of kernels one lmoe_lsm_fwd call launches (for launch accounting). */
int lmoe_lsm_fwd_num_launches(const lmoe_lsm_desc* desc);

/* Per-phase device time of calls made with LMOE_FLAG_TIMING since the last read (CUDA
 * events on the caller's stream).  Returns the number of calls, or -status on error. */
int lmoe_timing_read(float* ms_out, int nphase);
/* Kernels of this library enqueued since process start. */
long long lmoe_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LMOE_CUDA_H */
