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
    LMOE_MAMBA2 = 13, LMOE_HGRN2 = 14, LMOE_RWKV6 = 15,
    /* no chunk-parallel form: lmoe_lsm_fwd_recurrent */
    LMOE_DELTANET = 4, LMOE_GATED_DELTANET = 5, LMOE_GFW = 7, LMOE_GATELOOP = 8, LMOE_TTT = 9,
    LMOE_TITANS = 10, LMOE_S4 = 11, LMOE_MAMBA = 12, LMOE_RWKV7 = 16
};
enum lmoe_feature_map { LMOE_FM_IDENTITY = 0, LMOE_FM_ELU1 = 1, LMOE_FM_SQUARED = 2 };
/* LMOE_FLAG_TEST_DECAY_FAULT: TEST ONLY -- the within-chunk cumulative decay of the scalar-decay
 * kernels is shifted by one token (the reference's kern::chunk_decay_fault hook, lsm.hpp:310-317,
 * caught by test_lsm.cpp:221-235); results are then wrong by construction. */
enum lmoe_flags { LMOE_FLAG_CHECK = 1, LMOE_FLAG_TIMING = 2, LMOE_FLAG_TEST_DECAY_FAULT = 4 };

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

/* ---------------------------------------------------------------------------------------
 * Unmasked LSM sequence parallelism (paper Alg. 1).  Replaces sp_lsm_nomask_rank
 * (parallel.hpp:282-297): O_t = phi(Q_t) . sum_i phi(K_i)^T V_i over ALL ranks, with one
 * all-gather of exactly T * d_k * d_v fp32 elements per (b, h).  Undecayed instances only
 * ("sp_forward_nomask: requires an undecayed instance"), no normaliser
 * ("sp_forward_nomask: normalizer unsupported").  The loopback variant runs `world`
 * virtual ranks over a full [B,N,H,D] sequence on one device (chunk_range slices).
 * ------------------------------------------------------------------------------------- */
size_t lmoe_sp_lsm_nomask_workspace_size(const lmoe_lsm_desc* desc, int B, int N_local, int H,
                                         int D, lmoe_dtype dtype, int world);
int lmoe_sp_lsm_nomask_fwd(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D,
                           lmoe_dtype dtype, const void* q, const void* k, const void* v, void* o,
                           void* nccl_comm, int rank, int world, void* workspace,
                           size_t workspace_bytes, lmoe_stream_t stream);
int lmoe_sp_lsm_nomask_fwd_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                    lmoe_dtype dtype, const void* q, const void* k, const void* v,
                                    void* o, int world, void* workspace, size_t workspace_bytes,
                                    lmoe_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Softmax attention (the hybrid model's "N" layers).  lmoe_attn_fwd replaces
 * softmax_attention_parallel(q, k, v, causal = true, row_offset) (attention.hpp:18-38):
 * query row i attends to keys j <= i + row_offset (row_offset >= Nk: no mask).
 *   q [B, Nq, H, D], k / v [B, Nk, H, D], o [B, Nq, H, D]; bf16, D = 128.
 * lmoe_sp_attn_fwd replaces sp_attention_rank (parallel.hpp:380-387): this rank's
 * chunk_range slice of an N_total sequence; K and V are all-gathered (one NCCL group of the
 * two all-gathers) and the local queries attend with row_offset = r0.
 * ------------------------------------------------------------------------------------- */
int lmoe_attn_fwd(int B, int Nq, int Nk, int H, int D, lmoe_dtype dtype, const void* q,
                  const void* k, const void* v, void* o, int row_offset, lmoe_stream_t stream);
size_t lmoe_sp_attn_workspace_size(int B, int N_total, int H, int D, lmoe_dtype dtype, int world);
int lmoe_sp_attn_fwd(int B, int N_total, int H, int D, lmoe_dtype dtype, const void* q_loc,
                     const void* k_loc, const void* v_loc, void* o_loc, void* nccl_comm, int rank,
                     int world, void* workspace, size_t workspace_bytes, lmoe_stream_t stream);
/* Elements moved by the last lmoe_sp_attn_fwd gathers (K and V, padded slices). */
long long lmoe_sp_attn_last_gather_elements(void);

/* ---------------------------------------------------------------------------------------
 * Dense bf16 GEMM (tcgen05): C[M, N] = A[M, K] W[K, N]; A rows lda elements apart, W
 * row-major (the reference's (in x out) weight layout, model.hpp:152-160), C bf16 or fp32
 * (out_f32) with row stride ldc.  K % 64 == 0; N % 128 == 0 (bf16) / N % 64 == 0 (fp32).
 * ------------------------------------------------------------------------------------- */
size_t lmoe_gemm_workspace_size(int M);
int lmoe_gemm(const void* A, int M, int K, int lda, const void* W, int N, void* C, int ldc, int out_f32,
              void* workspace, size_t workspace_bytes, lmoe_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * One Linear-MoE block (Block, model.hpp:284-304, as model_forward / hybrid_sp_forward run
 * it, model.hpp:374-405, parallel.hpp:477-506):
 *   h = rms_norm(x, norm_mixer); x += mixer(h); h2 = rms_norm(x, norm_moe); x += MoE(h2)
 * kind 'L': LsmMixer (q, k, v, gates = h W, per-head LSM, o W_o); with world > 1 the LSM is
 * sp_lsm_masked_rank (one state all-gather).  kind 'N': AttentionMixer; with world > 1
 * sp_attention_rank (K/V all-gather, row offset from chunk_range of N_total).
 * x: fp32 residual stream [B, N_local, hidden], updated in place; aux: this block's
 * load-balance loss (device scalar).  head_dim = hidden / heads = 128.
 * num_experts == 0: the mixer layer alone, x += mixer(rms_norm(x, norm_mixer)) (the
 * "LSM-layer" unit of SURVEY 8(d); the MoE weights are not read).
 * A non-NULL nccl_comm at world 1 (a 1-rank communicator) runs the SP phase structure with
 * its all-gathers instead of the local shortcut.
 * ------------------------------------------------------------------------------------- */
typedef struct lmoe_block_desc {
    int kind;                 /* 'L' or 'N'                                            */
    int hidden, heads;
    int num_experts, top_k, ffn_dim;
    float norm_eps;           /* ModelConfig::norm_eps                                 */
    lmoe_lsm_desc lsm;        /* L blocks: the LsmSpec of every head                   */
} lmoe_block_desc;
typedef struct lmoe_block_weights {
    const float* norm_mixer;  /* [hidden] fp32                                         */
    const float* norm_moe;    /* [hidden] fp32                                         */
    const void* w_qkv;        /* bf16 [hidden, 3 hidden] = [Wq | Wk | Wv], or
                                 [hidden, 4 hidden] = [Wq | Wk | Wv | W_gate_a] for
                                 TokenVector instances (GLA / HGRN2 / RWKV6)            */
    const void* w_gate_b;     /* Mamba2: bf16 [hidden, 64], W_gate_b in columns < heads  */
    const float* a_raw;       /* Mamba2: [heads] fp32                                   */
    const void* wo;           /* bf16 [hidden, hidden]                                  */
    const void* router;       /* bf16 [hidden, E]                                       */
    const void* w_gate;       /* bf16 [E, hidden, ffn]                                  */
    const void* w_up;         /* bf16 [E, hidden, ffn]                                  */
    const void* w_down;       /* bf16 [E, ffn, hidden]                                  */
} lmoe_block_weights;
size_t lmoe_block_workspace_size(const lmoe_block_desc* desc, int B, int N_local, int N_total,
                                 int world);
int lmoe_block_fwd(const lmoe_block_desc* desc, const lmoe_block_weights* weights, int B,
                   int N_local, int N_total, float* x, float* aux, void* nccl_comm, int rank,
                   int world, void* workspace, size_t workspace_bytes, lmoe_stream_t stream);
/* One block over packed documents (model_forward, model.hpp:374-405): norms, projections and
 * the MoE over all T rows; the mixer (LSM or causal attention) per document of cu_seqlens
 * (HOST array, 0 .. T).  x: fp32 [T, hidden] residual stream, updated in place. */
size_t lmoe_block_varlen_workspace_size(const lmoe_block_desc* desc, int T, const int* cu_seqlens, int n_docs);
int lmoe_block_fwd_varlen(const lmoe_block_desc* desc, const lmoe_block_weights* weights, int T,
                          const int* cu_seqlens, int n_docs, float* x, float* aux, void* workspace,
                          size_t workspace_bytes, lmoe_stream_t stream);
/* x[t] = embedding[tokens[t]] + pos_embedding[pos0 + t % n] (model.hpp:385-386), fp32 out */
int lmoe_embed(const int* tokens, int rows, int n, int pos0, int hidden, const void* embedding,
               const void* pos_embedding, float* x, lmoe_stream_t stream);
/* out (bf16) = rms_norm(x, w, eps) (tensor.hpp:1164-1170) */
int lmoe_rmsnorm(const float* x, int rows, int hidden, const float* w, float eps, void* out,
                 lmoe_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * LSM backward: the vector-Jacobian product the reference's tape computes through
 * lsm_forward_chunked (tensor.hpp:1178-1215; ops of lsm.hpp:483-598), for every (b, h).
 * Inputs as lmoe_lsm_fwd plus dO [B,N,H,D] and the optional final-state gradient dM_final
 * [B,H,D,D] fp32 (NULL = 0).  Outputs (device, caller-owned):
 *   dq, dk, dv : [B,N,H,D] dtype
 *   db_pre     : [B,N,H] fp32 (Mamba2), da_raw : [H] fp32 (Mamba2, summed over batch)
 *   da_pre     : [B,N,H,D] dtype (TokenVector kinds)
 *   dM0        : [B,H,D,D] fp32 gradient of the initial state (may be NULL)
 * No recomputation of the forward output is needed: the passes consume q, k, v, dO only
 * (the normaliser composes two unnormalised backwards and two forwards for num / den).
 * TokenVector kinds: bf16 / head_dim 128 only.  Normalised instances: the VJP of the forward
 * with M_in = M0 and z_in = 0 (there is no z0 input; callers carrying a normaliser state in
 * must not use this entry point -- the Python mirror raises).
 * ------------------------------------------------------------------------------------- */
size_t lmoe_lsm_bwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                   lmoe_dtype dtype);
int lmoe_lsm_bwd(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                 const void* q, const void* k, const void* v, const void* a_pre,
                 const float* b_pre, const float* a_raw, const float* M0, const void* dO,
                 const float* dM_final, void* dq, void* dk, void* dv, void* da_pre,
                 float* db_pre, float* da_raw, float* dM0, void* workspace,
                 size_t workspace_bytes, lmoe_stream_t stream);

/* Packed documents (PackedBatch, model.hpp:86-121; model_forward runs the mixer per document,
 * model.hpp:374-405): q, k, v, ... are [1, T, H, D] with document i in rows
 * [cu_seqlens[i], cu_seqlens[i+1]) (HOST array, 0 .. T, strictly ascending); the state is
 * zero at every document start.  M_out: [n_docs, H, D, D] final states (may be NULL).
 * backward: da_raw sums over documents (workspace from the size query with backward = 1,
 * plus H floats when da_raw is requested). */
size_t lmoe_lsm_varlen_workspace_size(const lmoe_lsm_desc* desc, int T, const int* cu_seqlens, int n_docs,
                                      int H, int D, lmoe_dtype dtype, int backward);
int lmoe_lsm_fwd_varlen(const lmoe_lsm_desc* desc, int T, const int* cu_seqlens, int n_docs, int H, int D,
                        lmoe_dtype dtype, const void* q, const void* k, const void* v, const void* a_pre,
                        const float* b_pre, const float* a_raw, void* o, float* M_out, void* workspace,
                        size_t workspace_bytes, lmoe_stream_t stream);
int lmoe_lsm_bwd_varlen(const lmoe_lsm_desc* desc, int T, const int* cu_seqlens, int n_docs, int H, int D,
                        lmoe_dtype dtype, const void* q, const void* k, const void* v, const void* a_pre,
                        const float* b_pre, const float* a_raw, const void* dO, void* dq, void* dk, void* dv,
                        void* da_pre, float* db_pre, float* da_raw, void* workspace, size_t workspace_bytes,
                        lmoe_stream_t stream);

/* The kinds without a chunk-parallel form (DecayKind TokenOuter / FullElementwise / StateLinear
 * / Gradient: DeltaNet, GatedDeltaNet, GFW, GateLoop, TTT, Titans, RWKV7, S4, Mamba) run token
 * by token, as the reference's recurrent_step (lsm.hpp:335-441; lsm_forward_chunked evaluates
 * them sequentially inside each chunk, lsm.hpp:604-637, and parallel.hpp:309-311 gives them no
 * SP form).  One CTA per (b, h); the state lives in registers.  Gate and static inputs follow
 * LsmGates (lsm.hpp:206-247) and LsmSpec (lsm.hpp:134-177); NULL where a kind does not use them. */
typedef struct lmoe_lsm_recurrent_inputs {
    const void* a_vec;          /* RWKV7 / Mamba: a_pre [B, N, H, D] in dtype              */
    const float* a_scal;        /* DeltaNet / GatedDeltaNet / Titans: a_pre [B, N, H] fp32 */
    const float* b_pre;         /* DeltaNet / GatedDeltaNet / TTT / Titans / RWKV7 [B,N,H] */
    const void* alpha_pre;      /* GFW / GateLoop: [B, N, H, D] in dtype                   */
    const void* beta_pre;       /* GFW / GateLoop: [B, N, H, D] in dtype                   */
    const float* s4_delta_raw;  /* S4: [H, D]                                              */
    const float* s4_b;          /* S4: [H, D]                                              */
    const float* s4_A_raw;      /* S4: [H, D, D]                                           */
    const float* mamba_A_raw;   /* Mamba: [H, D, D]                                        */
} lmoe_lsm_recurrent_inputs;
/* workspace: >= 64 bytes of device memory (the device error flag; no allocation inside). */
int lmoe_lsm_fwd_recurrent(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                           const void* q, const void* k, const void* v, const lmoe_lsm_recurrent_inputs* in,
                           const float* M0, void* o, float* M_out, void* workspace, size_t workspace_bytes,
                           lmoe_stream_t stream);

/* Backward of lmoe_lsm_fwd_recurrent: the tape VJP of recurrent_step (lsm.hpp:335-441) over
 * the sequence (tensor.hpp:1178-1215) for the same kinds, with loss gradient dO [B, N, H, D]
 * (dtype) and the optional final-state gradient dM_final [B, H, D, D] fp32.  One CTA per
 * (b, h): a forward pass saving the state every 32 tokens, then the blocks in reverse (states
 * recomputed from the checkpoint).  Outputs: dq, dk, dv [B, N, H, D] dtype, the gate /
 * static-parameter gradients of `grads` (NULL where the kind has no such input; static ones
 * summed over the batch), dM0 [B, H, D, D] fp32 (may be NULL). */
typedef struct lmoe_lsm_recurrent_grads {
    void* da_vec;            /* RWKV7 / Mamba: [B, N, H, D] dtype                        */
    float* da_scal;          /* DeltaNet / GatedDeltaNet / Titans: [B, N, H]             */
    float* db_pre;           /* DeltaNet / GatedDeltaNet / TTT / Titans / RWKV7 [B,N,H]  */
    void* dalpha_pre;        /* GFW / GateLoop: [B, N, H, D] dtype                       */
    void* dbeta_pre;         /* GFW / GateLoop: [B, N, H, D] dtype                       */
    float* ds4_delta_raw;    /* S4: [H, D]                                               */
    float* ds4_b;            /* S4: [H, D]                                               */
    float* ds4_A_raw;        /* S4: [H, D, D]                                            */
    float* dmamba_A_raw;     /* Mamba: [H, D, D]                                         */
} lmoe_lsm_recurrent_grads;
size_t lmoe_lsm_bwd_recurrent_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                             lmoe_dtype dtype);
int lmoe_lsm_bwd_recurrent(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                           const void* q, const void* k, const void* v, const lmoe_lsm_recurrent_inputs* in,
                           const float* M0, const void* dO, const float* dM_final, void* dq, void* dk,
                           void* dv, const lmoe_lsm_recurrent_grads* grads, float* dM0, void* workspace,
                           size_t workspace_bytes, lmoe_stream_t stream);

/* Forward plan of lmoe_lsm_fwd for a shape: info[0] = 1 when the single-read persistent
 * kernel runs (opt-in), 2 for the local-state forward (decaying scalar kinds, bf16 / D = 128,
 * no normaliser: output pass from zero states, segment combine, correction of each segment's
 * first chunks; no state pass), 0 for the segment-parallel state pass + combine + output
 * pass; info[1] segments per (b,h), info[2] tokens per segment, info[3] CTAs per (b,h). */
int lmoe_lsm_fwd_plan(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype, int* info);

/* Number of kernels one lmoe_lsm_fwd call launches (for launch accounting). */
int lmoe_lsm_fwd_num_launches(const lmoe_lsm_desc* desc);

/* Per-phase device time of calls made with LMOE_FLAG_TIMING since the last read (CUDA
 * events on the caller's stream).  Returns the number of calls, or -status on error. */
int lmoe_timing_read(float* ms_out, int nphase);
/* Kernels of this library enqueued since process start. */
long long lmoe_launch_count(void);
/* Developer aid: clock64 phase trace of output-pass CTA (0,0,0) when LMOE_TRACE is set. */
int lmoe_debug_trace_read(unsigned long long* out /* 64 x 16 */);

/* ---------------------------------------------------------------------------------------
 * LSM sequence parallelism.  Replaces sp_lsm_masked_rank(RankGroup&, rank, q_loc, k_loc,
 * v_loc, gates_loc, spec, layer, &final_state) (parallel.hpp:303-376): the rank's
 * contiguous slice (chunk_range, parallel.hpp:192-197) is evaluated from the zero state,
 * ONE ncclAllGather moves the all-heads payload [M | z? | log D] (B*H*(D*D [+D] + 1) fp32 per
 * rank; the reference gathers per head, parallel.hpp:447-452), the decayed exclusive
 * prefix over earlier ranks (parallel.hpp:340-361) gives the carried-in state, and the
 * output pass re-evaluates the slice with it.  nccl_comm is an ncclComm_t (required for
 * world > 1).  At world 1, NULL runs the local pass; a 1-rank communicator runs the same
 * phase structure as world > 1, the ncclAllGather included (how the GPU tests execute the
 * NCCL path on one device).  The same holds for the unmasked, backward and attention SP calls.
 * ------------------------------------------------------------------------------------- */
size_t lmoe_sp_payload_floats(const lmoe_lsm_desc* desc, int B, int H, int D);
size_t lmoe_sp_lsm_fwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D,
                                      lmoe_dtype dtype, int world);
int lmoe_sp_lsm_fwd(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D, lmoe_dtype dtype,
                    const void* q, const void* k, const void* v, const void* a_pre,
                    const float* b_pre, const float* a_raw, void* o, float* M_out, float* z_out,
                    void* nccl_comm, int rank, int world, void* workspace, size_t workspace_bytes,
                    lmoe_stream_t stream);
/* Same algorithm, `world` virtual ranks on one device over the full sequence (device copies
 * instead of the all-gather): sp_forward_masked (parallel.hpp:405-418) for testing. */
size_t lmoe_sp_lsm_fwd_loopback_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H,
                                               int D, lmoe_dtype dtype, int world);
int lmoe_sp_lsm_fwd_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                             lmoe_dtype dtype, const void* q, const void* k, const void* v,
                             const void* a_pre, const float* b_pre, const float* a_raw, void* o,
                             float* M_out, float* z_out, int world, void* workspace,
                             size_t workspace_bytes, lmoe_stream_t stream);
/* LSM sequence-parallel BACKWARD of lmoe_sp_lsm_fwd for this rank's slice (SURVEY 8(f) rank
 * 1; the reference differentiates sp_lsm_masked_rank on its tape across the rank threads).
 * Two all-gathers of B*H*(D*D + lw) fp32 per rank: the forward payload again (the rank's
 * initial state), and the reverse-time payload [X | log D] (X = the adjoint at the slice
 * start from the slice's own queries); a suffix combine over later ranks gives the adjoint
 * entering the slice end, and the local backward (lmoe_lsm_bwd with M0 and dM_final) is then
 * exact for the slice.  Outputs as lmoe_lsm_bwd for the slice; da_raw is this rank's
 * contribution (the sum over ranks is the full gradient); dM0 is meaningful on rank 0.
 * Normalised instances (o = num / den) compose two unnormalised SP forwards (num over v, den
 * over e0, whose state column 0 is z) and two unnormalised SP backwards, as lmoe_lsm_bwd does
 * locally: 4 collective rounds instead of 1. */
size_t lmoe_sp_lsm_bwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D,
                                      lmoe_dtype dtype, int world);
int lmoe_sp_lsm_bwd(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D, lmoe_dtype dtype,
                    const void* q, const void* k, const void* v, const void* a_pre, const float* b_pre,
                    const float* a_raw, const void* dO, void* dq, void* dk, void* dv, void* da_pre,
                    float* db_pre, float* da_raw, float* dM0, void* nccl_comm, int rank, int world,
                    void* workspace, size_t workspace_bytes, lmoe_stream_t stream);
/* The same with `world` virtual ranks on one device over the full sequence (B == 1). */
size_t lmoe_sp_lsm_bwd_loopback_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                               lmoe_dtype dtype, int world);
int lmoe_sp_lsm_bwd_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                             const void* q, const void* k, const void* v, const void* a_pre,
                             const float* b_pre, const float* a_raw, const void* dO, void* dq, void* dk,
                             void* dv, void* da_pre, float* db_pre, float* da_raw, float* dM0, int world,
                             void* workspace, size_t workspace_bytes, lmoe_stream_t stream);
/* Elements moved by the last SP gather (RankGroup::comm_log accounting, parallel.hpp:87-93). */
long long lmoe_sp_last_gather_elements(void);
/* NCCL bootstrap: rank 0 creates the 128-byte id, the caller distributes it. */
int lmoe_nccl_unique_id(void* id128);
int lmoe_nccl_comm_init(void** comm, int world, int rank, const void* id128);
int lmoe_nccl_comm_destroy(void* comm);

/* ---------------------------------------------------------------------------------------
 * MoE expert layer (moe.hpp).  bf16 activations / weights in the reference layouts
 * (router (hidden, E); w_gate, w_up (E, hidden, ffn); w_down (E, ffn, hidden)).
 * ------------------------------------------------------------------------------------- */
size_t lmoe_moe_workspace_size(int T, int hidden, int ffn, int E, int top_k);
/* route (moe.hpp:58-85) + load_balance_loss (moe.hpp:90-103) on fp32 logits [T, E]:
 * ids [T, k] (ascending per token, ties -> lower id), gates [T, k] renormalised over the
 * selection, probs [T, E] (nullable), counts [E], aux (nullable).  E <= 256, k <= 32. */
int lmoe_moe_route(const float* logits, int T, int E, int top_k, int* ids, float* gates,
                   float* probs, int* counts, float* aux, void* workspace, size_t workspace_bytes,
                   lmoe_stream_t stream);
/* MoeLayer::forward (moe.hpp:133-149): router GEMM, route, stable dispatch (tokens ascending
 * per expert, moe.hpp:137-139), grouped SwiGLU experts (moe.hpp:45-47), combine in ascending
 * expert order, aux loss.  hidden % 256 == 0, ffn % 128 == 0.  logits/ids/gates outputs are
 * optional copies of the routing. */
int lmoe_moe_forward(int T, int hidden, int ffn, int E, int top_k, const void* x,
                     const void* w_router, const void* w_gate, const void* w_up,
                     const void* w_down, void* y, int y_f32, float* aux, float* logits_out,
                     int* ids_out, float* gates_out, void* workspace, size_t workspace_bytes,
                     lmoe_stream_t stream);
/* Dispatch of the last forward using `workspace`: slot positions [T,k], the token of each
 * permuted row [T*k], expert offsets [E+1] (device buffers, nullable). */
int lmoe_moe_dispatch_read(int T, int hidden, int ffn, int E, int top_k, const void* workspace,
                           int* slot_pos, int* perm_token, int* offsets, lmoe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LMOE_CUDA_H */
