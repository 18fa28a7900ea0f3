/*
 * lmoe_oracle.h -- CPU restatement of the Linear-MoE reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_2503_05447_b200/csrc.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it.  The product library never links it.
 *
 * Every routine is a plain-C, float64 restatement of a reference function in
 * /root/reference/proj/include/lmoe (cited per function).  Parity of this
 * restatement with the reference itself is pinned by tests/golden/*.npz, which
 * tests/golden/make_golden.py generates by compiling the reference headers
 * unmodified (oracle/ref_driver.cpp, recipe oracle/Makefile).
 *
 * Layouts: row-major, one (b,h) head slice at a time: q,k,v are (n x d);
 * state M is (d_k x d_v); z is (d_k).
 */
#ifndef LMOE_ORACLE_H
#define LMOE_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Same numbering as lmoe::LsmInstance (lsm.hpp:30-48). */
enum {
    LMO_BLA = 0, LMO_LIGHTNING = 1, LMO_RETNET = 2, LMO_GLA = 3, LMO_DELTANET = 4,
    LMO_GATED_DELTANET = 5, LMO_REBASED = 6, LMO_GFW = 7, LMO_GATELOOP = 8, LMO_TTT = 9,
    LMO_TITANS = 10, LMO_S4 = 11, LMO_MAMBA = 12, LMO_MAMBA2 = 13, LMO_HGRN2 = 14,
    LMO_RWKV6 = 15, LMO_RWKV7 = 16
};
/* lmoe::FeatureMap (lsm.hpp:50) */
enum { LMO_FM_IDENTITY = 0, LMO_FM_ELU1 = 1, LMO_FM_SQUARED = 2 };
/* lmoe::DecayKind (lsm.hpp:53-62), only the separable ones are restated */
enum { LMO_DK_NONE = 0, LMO_DK_CONST = 1, LMO_DK_TOKEN_SCALAR = 2, LMO_DK_TOKEN_VECTOR = 3,
       LMO_DK_OTHER = 4 };

typedef struct {
    int instance;       /* LMO_* */
    int feature_map;    /* LMO_FM_* */
    int use_normalizer; /* 0/1 */
    double scalar_decay;/* Lightning/RetNet a */
    double mamba2_a_raw;/* Mamba2 static param (one per head) */
} lmo_spec;

int lmo_decay_kind(int instance);
/* LsmSpec::make defaults (lsm.hpp:146-165) for feature map / normaliser / scalar decay. */
void lmo_spec_default(lmo_spec* s, int instance);
/* LsmSpec::validate (lsm.hpp:188-204); returns 0 or -1 with message in err. */
int lmo_spec_validate(const lmo_spec* s, int d_k, int d_v, char* err, int errlen);

/*
 * lsm_forward_chunked (lsm.hpp:668-708) for the separable decay kinds, with
 * chunk_forward_separable (lsm.hpp:554-598), effective_keys (:483-501) and
 * decay_vector_rows (:504-518).  a_pre is (n x d_k) for TokenVector kinds,
 * b_pre is (n) for Mamba2; NULL otherwise.  M0/z0 may be NULL (zero state;
 * the reference always starts fresh -- a non-NULL initial state is the SP
 * carried-in state of parallel.hpp:366-373).  M_out/z_out may be NULL.
 * Returns 0, or -1 with the reference's error text in err.
 */
int lmo_lsm_chunked(const lmo_spec* s, int n, int d_k, int d_v, int chunk,
                    const double* q, const double* k, const double* v,
                    const double* a_pre, const double* b_pre,
                    const double* M0, const double* z0,
                    double* o, double* M_out, double* z_out, char* err, int errlen);

/* lsm_forward_sequential / recurrent_step (lsm.hpp:335-441, 643-662), same args. */
int lmo_lsm_sequential(const lmo_spec* s, int n, int d_k, int d_v,
                       const double* q, const double* k, const double* v,
                       const double* a_pre, const double* b_pre,
                       const double* M0, const double* z0,
                       double* o, double* M_out, double* z_out, char* err, int errlen);

/* recurrent_step (lsm.hpp:335-441) token by token for DeltaNet, GatedDeltaNet, GFW, GateLoop,
 * TTT, Titans, RWKV7, S4, Mamba (no chunk-parallel form).  Gate / static-parameter layouts as
 * LsmGates (lsm.hpp:206-247) and LsmSpec (lsm.hpp:134-177); NULL where unused. */
int lmo_lsm_recurrent(const lmo_spec* s, int n, int d_k, int d_v, const double* q, const double* k,
                      const double* v, const double* a_pre, const double* b_pre, const double* alpha_pre,
                      const double* beta_pre, const double* s4_delta_raw, const double* s4_b,
                      const double* s4_A_raw, const double* mamba_A_raw, const double* M0, double* o,
                      double* M_out, char* err, int errlen);

/*
 * Reverse-mode gradient of L = sum(o .* dO) through the token recurrence
 * (the quantity the reference tape computes via backward(), tensor.hpp:1178,
 * for lsm_forward_* which are mathematically equal).  Outputs dq, dk, dv
 * (n x d), da_pre (n x d_k, TokenVector), db_pre (n, Mamba2), da_raw (scalar,
 * Mamba2), dM0 (d_k x d_v).  Normaliser not supported (returns -1).
 */
int lmo_lsm_backward(const lmo_spec* s, int n, int d_k, int d_v,
                     const double* q, const double* k, const double* v,
                     const double* a_pre, const double* b_pre, const double* M0,
                     const double* dO,
                     double* dq, double* dk, double* dv, double* da_pre, double* db_pre,
                     double* da_raw, double* dM0, const double* dM_final /* NULL = 0 */,
                     char* err, int errlen);

/*
 * route (moe.hpp:58-85): ids (t x top_k, ascending per token), gates and probs
 * dense (t x e).  Returns -1 on bad top_k ("route: bad top_k").
 */
int lmo_route(const double* logits, int t, int e, int top_k, int* ids, double* gates,
              double* probs, char* err, int errlen);
/* load_balance_loss (moe.hpp:90-103) */
double lmo_load_balance_loss(const int* ids, const double* probs, int t, int e, int top_k);
/*
 * MoeLayer::forward (moe.hpp:133-149) with Expert::forward (moe.hpp:45-47).
 * x (t x hidden), router (hidden x e), w_gate/w_up [e][hidden x ffn],
 * w_down [e][ffn x hidden] (reference row-major layouts, experts stacked).
 * Writes y (t x hidden), *aux, and optionally logits (t x e).
 */
int lmo_moe_forward(const double* x, int t, int hidden, int ffn, int e, int top_k,
                    const double* router, const double* w_gate, const double* w_up,
                    const double* w_down, double* y, double* aux, double* logits_out,
                    char* err, int errlen);

/* chunk_range (parallel.hpp:192-197) */
void lmo_chunk_range(int n, int t, int rank, int* r0, int* r1);

/*
 * sp_forward_masked (parallel.hpp:405-418) with sp_lsm_masked_rank
 * (:303-376): each rank slice evaluated as one chunk from zero, one gather of
 * [M | z? | D?], decay-weighted exclusive prefix, re-evaluation.  When
 * rank_chunk > 0 the per-rank evaluation is chunked with that chunk size
 * instead (mathematically identical; needed for long slices where the
 * single-chunk K/p form overflows).
 */
int lmo_sp_forward_masked(const lmo_spec* s, int n, int d_k, int d_v, int world,
                          int rank_chunk,
                          const double* q, const double* k, const double* v,
                          const double* a_pre, const double* b_pre, double* o,
                          char* err, int errlen);

/*
 * sp_forward_nomask (parallel.hpp:391-403) with sp_lsm_nomask_rank (:282-297): every
 * rank's local phi(K)^T V is gathered and summed; O = phi(Q) . sum.  Returns -1 with the
 * reference's texts for decayed instances or the normaliser.
 */
int lmo_sp_forward_nomask(const lmo_spec* s, int n, int d_k, int d_v, int world,
                          const double* q, const double* k, const double* v, double* o,
                          char* err, int errlen);

/*
 * The per-rank pieces of the same algorithm, so a multi-process harness
 * (tests/test_sp_gloo.py) can run the exchange itself:
 *  payload  = [M | z? | D?] of the local slice from zero (d_k x pw, pw =
 *             d_v + use_normalizer + (decay kind != None)), row-major.
 *  combine  = exclusive decayed prefix over gathered payloads[0..rank-1].
 */
int lmo_sp_payload_width(const lmo_spec* s, int d_v);
int lmo_sp_local_payload(const lmo_spec* s, int n_loc, int d_k, int d_v, int chunk,
                         const double* q, const double* k, const double* v,
                         const double* a_pre, const double* b_pre, double* payload,
                         char* err, int errlen);
void lmo_sp_combine(const lmo_spec* s, int d_k, int d_v, int rank, const double* gathered,
                    double* M_in, double* z_in);

/* softmax_attention_parallel (attention.hpp:18-38), causal with row_offset. */
void lmo_attention(const double* q, const double* k, const double* v, int nq, int nk, int d,
                   int dv, int causal, int row_offset, double* o);

#ifdef __cplusplus
}
#endif
#endif
