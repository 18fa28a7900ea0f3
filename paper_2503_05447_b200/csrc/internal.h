// internal.h -- C++ entry points shared between the C-ABI translation units (not exported
// in include/): strided-view LSM / attention cores and the dense tcgen05 GEMM, composed by
// the block executor (block.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "../../include/lmoe_cuda.h"

namespace lmoe_host {

const char* instance_name(int inst);  // lsm_host.cu: the reference's instance names

// LSM mixer over q, k, v (and TokenVector a_pre) [B, N, H, D] views whose token rows are
// `ld` elements apart (0: H * D); o dense.  world == 1: lsm_forward_chunked; world > 1:
// sp_lsm_masked_rank with one NCCL all-gather.
size_t lsm_mixer_ws(const lmoe_lsm_desc* d, int B, int N, int H, int D, int world);
void lsm_mixer_core(const lmoe_lsm_desc* d, int B, int N, int H, int D, lmoe_dtype dt, const void* q,
                    const void* k, const void* v, const void* a_pre, int ld, const float* b_pre,
                    const float* a_raw, void* o, void* comm, int rank, int world, void* ws, size_t ws_bytes,
                    cudaStream_t st);

// Causal attention (bf16, D = 128) over strided q / k / v rows; sp_attn_core gathers K, V.
void attn_core(int B, int Nq, int Nk, int H, int D, const void* q, const void* k, const void* v, int ld,
               void* o, int row_offset, cudaStream_t st);
size_t sp_attn_ws(int B, int N_total, int H, int D, int world);
void sp_attn_core(int B, int N_total, int H, int D, const void* q_loc, const void* k_loc, const void* v_loc,
                  int ld, void* o_loc, void* comm, int rank, int world, void* ws, size_t ws_bytes,
                  cudaStream_t st);

// C[M, N] = A[M, K] (bf16, row stride lda) x W[K, N] (bf16 row-major); C bf16 or fp32 (row
// stride ldc).  K % 64 == 0; N % 128 == 0 (bf16) or N % 64 == 0 (fp32).
size_t dense_gemm_ws(int M);
void dense_gemm(const void* A, int M, int K, int lda, const void* W, int N, void* C, int ldc, bool out_f32,
                void* ws, cudaStream_t st);

}  // namespace lmoe_host
