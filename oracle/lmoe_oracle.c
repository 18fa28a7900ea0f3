/*
 * lmoe_oracle.c -- float64 CPU restatement of the Linear-MoE reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lmoe_oracle.h).  Parity with the reference is
 * pinned by tests/golden (generated from the unmodified reference headers).
 * Each function cites the reference file:line it restates; paths are relative
 * to /root/reference/proj/include/lmoe.
 */
#include "lmoe_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static void set_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) {
        strncpy(err, msg, (size_t)errlen - 1);
        err[errlen - 1] = 0;
    }
}

static const char* kNames[] = {"bla",    "lightning", "retnet", "gla",   "deltanet",
                               "gated_deltanet", "rebased", "gfw", "gateloop", "ttt",
                               "titans", "s4",        "mamba",  "mamba2", "hgrn2",
                               "rwkv6",  "rwkv7"};

/* tensor.hpp:423-429 */
static double sigm(double x) { return x >= 0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x)); }
/* tensor.hpp:446-453 */
static double softplus(double x) { return x > 30 ? x : log1p(exp(x)); }
/* tensor.hpp:455-460 (elu+1), :462 (square) */
static double fmap(int fm, double x) {
    if (fm == LMO_FM_ELU1) return x > 0 ? x + 1.0 : exp(x);
    if (fm == LMO_FM_SQUARED) return x * x;
    return x;
}
static double fmap_grad(int fm, double x) {
    if (fm == LMO_FM_ELU1) return x > 0 ? 1.0 : exp(x);
    if (fm == LMO_FM_SQUARED) return 2.0 * x;
    return 1.0;
}

/* lsm.hpp:64-85 */
int lmo_decay_kind(int inst) {
    switch (inst) {
        case LMO_BLA: case LMO_REBASED: return LMO_DK_NONE;
        case LMO_LIGHTNING: case LMO_RETNET: return LMO_DK_CONST;
        case LMO_MAMBA2: return LMO_DK_TOKEN_SCALAR;
        case LMO_GLA: case LMO_HGRN2: case LMO_RWKV6: return LMO_DK_TOKEN_VECTOR;
        default: return LMO_DK_OTHER;
    }
}

/* LsmSpec::make (lsm.hpp:146-165) */
void lmo_spec_default(lmo_spec* s, int inst) {
    s->instance = inst;
    s->feature_map = LMO_FM_IDENTITY;
    s->use_normalizer = 0;
    s->scalar_decay = 1.0;
    s->mamba2_a_raw = 0.0;
    if (inst == LMO_BLA) { s->feature_map = LMO_FM_ELU1; s->use_normalizer = 1; }
    if (inst == LMO_REBASED) { s->feature_map = LMO_FM_SQUARED; s->use_normalizer = 1; }
    if (inst == LMO_LIGHTNING) s->scalar_decay = 0.95;
    if (inst == LMO_RETNET) s->scalar_decay = 1.0 - 1.0 / 32.0;
}

/* LsmSpec::validate (lsm.hpp:188-204) */
int lmo_spec_validate(const lmo_spec* s, int d_k, int d_v, char* err, int errlen) {
    if (d_k <= 0 || d_v <= 0) { set_err(err, errlen, "LsmSpec: nonpositive head dims"); return -1; }
    if (s->use_normalizer) {
        int dk = lmo_decay_kind(s->instance);
        if (dk == LMO_DK_OTHER || s->instance == LMO_HGRN2 || s->instance == LMO_MAMBA2) {
            char buf[128];
            snprintf(buf, sizeof buf, "LsmSpec: normalizer unsupported for instance %s",
                     kNames[s->instance]);
            set_err(err, errlen, buf);
            return -1;
        }
    }
    return 0;
}

/* Per-token decay value for dim i (decay_vector_rows, lsm.hpp:504-518). */
static double decay_at(const lmo_spec* s, int d_k, const double* a_pre, const double* b_pre,
                       int t, int i) {
    switch (lmo_decay_kind(s->instance)) {
        case LMO_DK_NONE: return 1.0;
        case LMO_DK_CONST: return s->scalar_decay;
        case LMO_DK_TOKEN_SCALAR:
            return exp(-(softplus(b_pre[t]) * softplus(s->mamba2_a_raw)));
        case LMO_DK_TOKEN_VECTOR: return sigm(a_pre[(size_t)t * d_k + i]);
    }
    return 1.0;
}

/* effective_keys (lsm.hpp:483-501) */
static double keff_at(const lmo_spec* s, int d_k, const double* k, const double* a_pre,
                      const double* b_pre, int t, int i) {
    if (s->instance == LMO_HGRN2) return 1.0 - sigm(a_pre[(size_t)t * d_k + i]);
    double pk = fmap(s->feature_map, k[(size_t)t * d_k + i]);
    if (s->instance == LMO_MAMBA2) return pk * softplus(b_pre[t]);
    return pk;
}

static int check_state(const lmo_spec* s, const double* M, size_t cnt, char* err, int errlen) {
    for (size_t i = 0; i < cnt; ++i)
        if (!isfinite(M[i])) {
            char buf[128];
            snprintf(buf, sizeof buf, "non-finite memory state in instance %s",
                     kNames[s->instance]);
            set_err(err, errlen, buf);
            return -1;
        }
    return 0;
}

/*
 * chunk_forward_separable (lsm.hpp:554-598) on rows [r0, r1) with in-state
 * (M, z) updated in place.  Uses the reference's own K/p closed form.
 */
static int chunk_separable(const lmo_spec* s, int d_k, int d_v, int r0, int r1,
                           const double* q, const double* k, const double* v,
                           const double* a_pre, const double* b_pre, double* M, double* z,
                           double* o, char* err, int errlen) {
    const int c = r1 - r0;
    double* p = (double*)malloc(sizeof(double) * c * d_k);
    double* qt = (double*)malloc(sizeof(double) * c * d_k);
    double* kt = (double*)malloc(sizeof(double) * c * d_k);
    double* sc = (double*)malloc(sizeof(double) * c * c);
    int rc = 0;
    /* cumulative decay p (lsm.hpp:558-565), inclusive of own token */
    for (int i = 0; i < d_k; ++i) {
        double cur = 1.0;
        for (int t = 0; t < c; ++t) {
            double a = decay_at(s, d_k, a_pre, b_pre, r0 + t, i);
            cur = (t == 0) ? a : cur * a;
            p[t * d_k + i] = cur;
        }
    }
    for (int t = 0; t < c; ++t)
        for (int i = 0; i < d_k; ++i) {
            double pq = fmap(s->feature_map, q[(size_t)(r0 + t) * d_k + i]);
            double ke = keff_at(s, d_k, k, a_pre, b_pre, r0 + t, i);
            qt[t * d_k + i] = pq * p[t * d_k + i];  /* q_t = phiQ . p   (:575) */
            kt[t * d_k + i] = ke / p[t * d_k + i];  /* k_t = keff / p   (:576) */
            if (!isfinite(kt[t * d_k + i])) {
                set_err(err, errlen, "non-finite output in div");
                rc = -1;
                goto done;
            }
        }
    /* scores = (q_t k_t^T) . causal mask (inclusive)  (:578) */
    for (int i = 0; i < c; ++i)
        for (int j = 0; j < c; ++j) {
            double acc = 0.0;
            if (j <= i)
                for (int e = 0; e < d_k; ++e) acc += qt[i * d_k + e] * kt[j * d_k + e];
            sc[i * c + j] = acc;
        }
    /* o = scores v + q_t M_in  (:579) */
    for (int i = 0; i < c; ++i)
        for (int jv = 0; jv < d_v; ++jv) {
            double a1 = 0.0, a2 = 0.0;
            for (int j = 0; j <= i; ++j) a1 += sc[i * c + j] * v[(size_t)(r0 + j) * d_v + jv];
            for (int e = 0; e < d_k; ++e) a2 += qt[i * d_k + e] * M[e * d_v + jv];
            o[(size_t)(r0 + i) * d_v + jv] = a1 + a2;
        }
    if (s->use_normalizer) {
        /* denom = rowsum(scores) + q_t z_in; |denom| < 1e-12 -> error (:584-592) */
        for (int i = 0; i < c; ++i) {
            double den = 0.0, qz = 0.0;
            for (int j = 0; j < c; ++j) den += sc[i * c + j];
            for (int e = 0; e < d_k; ++e) qz += qt[i * d_k + e] * z[e];
            den += qz;
            if (fabs(den) < 1e-12) {
                char buf[128];
                snprintf(buf, sizeof buf, "degenerate normalizer in instance %s",
                         kNames[s->instance]);
                set_err(err, errlen, buf);
                rc = -1;
                goto done;
            }
            for (int jv = 0; jv < d_v; ++jv) o[(size_t)(r0 + i) * d_v + jv] *= 1.0 / den;
        }
    }
    /* M_out = diag(p_C) M_in + (k_t . p_C)^T V ;  z_out = z . p_C + colsum(k2) (:581-594) */
    {
        const double* pl = p + (size_t)(c - 1) * d_k;
        for (int e = 0; e < d_k; ++e) {
            for (int jv = 0; jv < d_v; ++jv) {
                double acc = 0.0;
                for (int t = 0; t < c; ++t)
                    acc += (kt[t * d_k + e] * pl[e]) * v[(size_t)(r0 + t) * d_v + jv];
                M[e * d_v + jv] = M[e * d_v + jv] * pl[e] + acc;
            }
            if (s->use_normalizer) {
                double cs = 0.0;
                for (int t = 0; t < c; ++t) cs += kt[t * d_k + e] * pl[e];
                z[e] = z[e] * pl[e] + cs;
            }
        }
    }
    rc = check_state(s, M, (size_t)d_k * d_v, err, errlen);
done:
    free(p); free(qt); free(kt); free(sc);
    return rc;
}

static int check_separable(const lmo_spec* s, char* err, int errlen) {
    if (lmo_decay_kind(s->instance) == LMO_DK_OTHER) {
        set_err(err, errlen, "oracle: only separable decay kinds are restated");
        return -1;
    }
    return 0;
}

/* lsm_forward_chunked (lsm.hpp:668-708) */
int lmo_lsm_chunked(const lmo_spec* s, int n, int d_k, int d_v, int chunk, const double* q,
                    const double* k, const double* v, const double* a_pre,
                    const double* b_pre, const double* M0, const double* z0, double* o,
                    double* M_out, double* z_out, char* err, int errlen) {
    if (lmo_spec_validate(s, d_k, d_v, err, errlen)) return -1;
    if (chunk < 1) { set_err(err, errlen, "lsm_forward_chunked: chunk_size must be >= 1"); return -1; }
    if (check_separable(s, err, errlen)) return -1;
    double* M = (double*)calloc((size_t)d_k * d_v, sizeof(double));
    double* z = (double*)calloc((size_t)d_k, sizeof(double));
    if (M0) memcpy(M, M0, sizeof(double) * d_k * d_v);
    if (z0) memcpy(z, z0, sizeof(double) * d_k);
    int rc = 0;
    for (int c0 = 0; c0 < n && rc == 0; c0 += chunk) {
        int c1 = c0 + chunk < n ? c0 + chunk : n;
        rc = chunk_separable(s, d_k, d_v, c0, c1, q, k, v, a_pre, b_pre, M, z, o, err, errlen);
    }
    if (rc == 0) {
        if (M_out) memcpy(M_out, M, sizeof(double) * d_k * d_v);
        if (z_out) memcpy(z_out, z, sizeof(double) * d_k);
    }
    free(M); free(z);
    return rc;
}

/* recurrent_step (lsm.hpp:335-441) folded by lsm_forward_sequential (:643-662) */
int lmo_lsm_sequential(const lmo_spec* s, int n, int d_k, int d_v, const double* q,
                       const double* k, const double* v, const double* a_pre,
                       const double* b_pre, const double* M0, const double* z0, double* o,
                       double* M_out, double* z_out, char* err, int errlen) {
    if (lmo_spec_validate(s, d_k, d_v, err, errlen)) return -1;
    if (check_separable(s, err, errlen)) return -1;
    double* M = (double*)calloc((size_t)d_k * d_v, sizeof(double));
    double* z = (double*)calloc((size_t)d_k, sizeof(double));
    double* pq = (double*)malloc(sizeof(double) * d_k);
    if (M0) memcpy(M, M0, sizeof(double) * d_k * d_v);
    if (z0) memcpy(z, z0, sizeof(double) * d_k);
    int rc = 0;
    for (int t = 0; t < n && rc == 0; ++t) {
        for (int i = 0; i < d_k; ++i) {
            double a = decay_at(s, d_k, a_pre, b_pre, t, i);
            double ke = keff_at(s, d_k, k, a_pre, b_pre, t, i);
            for (int j = 0; j < d_v; ++j)
                M[i * d_v + j] = a * M[i * d_v + j] + ke * v[(size_t)t * d_v + j];
            if (s->use_normalizer) z[i] = z[i] * a + fmap(s->feature_map, k[(size_t)t * d_k + i]);
            pq[i] = fmap(s->feature_map, q[(size_t)t * d_k + i]);
        }
        rc = check_state(s, M, (size_t)d_k * d_v, err, errlen);
        if (rc) break;
        double den = 1.0;
        if (s->use_normalizer) {
            den = 0.0;
            for (int i = 0; i < d_k; ++i) den += pq[i] * z[i];
            if (fabs(den) < 1e-12) {
                char buf[128];
                snprintf(buf, sizeof buf, "degenerate normalizer in instance %s",
                         kNames[s->instance]);
                set_err(err, errlen, buf);
                rc = -1;
                break;
            }
        }
        for (int j = 0; j < d_v; ++j) {
            double acc = 0.0;
            for (int i = 0; i < d_k; ++i) acc += pq[i] * M[i * d_v + j];
            o[(size_t)t * d_v + j] = s->use_normalizer ? acc / den : acc;
        }
    }
    if (rc == 0) {
        if (M_out) memcpy(M_out, M, sizeof(double) * d_k * d_v);
        if (z_out) memcpy(z_out, z, sizeof(double) * d_k);
    }
    free(M); free(z); free(pq);
    return rc;
}

/*
 * Adjoint of the token recurrence M_s = diag(a_s) M_{s-1} + keff_s v_s^T,
 * o_s = phi(q_s)^T M_s (recurrent_step, lsm.hpp:335-441), chained through the
 * feature map, effective key and decay parameterisations.  The reference gets
 * the same numbers from its tape (tensor.hpp:1178-1215); tests/golden pins them.
 */
int lmo_lsm_backward(const lmo_spec* s, int n, int d_k, int d_v, const double* q,
                     const double* k, const double* v, const double* a_pre,
                     const double* b_pre, const double* M0, const double* dO, double* dq,
                     double* dk, double* dv, double* da_pre, double* db_pre, double* da_raw,
                     double* dM0, const double* dM_final, char* err, int errlen) {
    if (lmo_spec_validate(s, d_k, d_v, err, errlen)) return -1;
    if (check_separable(s, err, errlen)) return -1;
    /* The normaliser state z_s = Theta_s z_{s-1} + keff_s (lsm.hpp:335-441) is carried as one
     * extra value column of M whose value is 1: o = num / den with num = phi(q) M[:, :d_v],
     * den = phi(q) M[:, d_v]; its upstream gradient is [dO / den | -(dO . num) / den^2]. */
    const int nz = s->use_normalizer ? 1 : 0;
    const int dva = d_v + nz;
    const size_t dd = (size_t)d_k * dva;
    double* Ms = (double*)malloc(sizeof(double) * dd * (size_t)(n + 1)); /* M_{-1..n-1} */
    double* dM = (double*)calloc(dd, sizeof(double));
    double* dOa = (double*)malloc(sizeof(double) * dva);
    /* loss gradient w.r.t. the returned final state (lsm_forward_chunked's final_state) */
    if (dM_final)
        for (int i = 0; i < d_k; ++i)
            for (int j = 0; j < d_v; ++j) dM[i * dva + j] = dM_final[(size_t)i * d_v + j];
    memset(Ms, 0, sizeof(double) * dd);
    if (M0)
        for (int i = 0; i < d_k; ++i)
            for (int j = 0; j < d_v; ++j) Ms[i * dva + j] = M0[(size_t)i * d_v + j];
#define VA(t, j) ((j) < d_v ? v[(size_t)(t) * d_v + (j)] : 1.0)
    for (int t = 0; t < n; ++t)
        for (int i = 0; i < d_k; ++i) {
            double a = decay_at(s, d_k, a_pre, b_pre, t, i);
            double ke = keff_at(s, d_k, k, a_pre, b_pre, t, i);
            for (int j = 0; j < dva; ++j)
                Ms[(t + 1) * dd + i * dva + j] = a * Ms[t * dd + i * dva + j] + ke * VA(t, j);
        }
    const int dkind = lmo_decay_kind(s->instance);
    if (da_pre && dkind == LMO_DK_TOKEN_VECTOR) memset(da_pre, 0, sizeof(double) * n * d_k);
    if (db_pre && s->instance == LMO_MAMBA2) memset(db_pre, 0, sizeof(double) * n);
    double draw = 0.0;
    for (int t = n - 1; t >= 0; --t) {
        const double* Mt = Ms + (size_t)(t + 1) * dd;
        const double* Mp = Ms + (size_t)t * dd;
        for (int j = 0; j < d_v; ++j) dOa[j] = dO[(size_t)t * d_v + j];
        if (nz) {
            double den = 0.0, dn = 0.0;
            for (int i = 0; i < d_k; ++i) den += fmap(s->feature_map, q[(size_t)t * d_k + i]) * Mt[i * dva + d_v];
            if (fabs(den) < 1e-12) {
                set_err(err, errlen, "degenerate normalizer");
                free(Ms); free(dM); free(dOa);
                return -1;
            }
            for (int j = 0; j < d_v; ++j) {
                double num = 0.0;
                for (int i = 0; i < d_k; ++i) num += fmap(s->feature_map, q[(size_t)t * d_k + i]) * Mt[i * dva + j];
                dn += dOa[j] * num;
                dOa[j] /= den;
            }
            dOa[d_v] = -dn / (den * den);
        }
        /* dM_t += phi(q_t) (x) dO_t ; dphi(q_t) = M_t dO_t */
        for (int i = 0; i < d_k; ++i) {
            double pqi = fmap(s->feature_map, q[(size_t)t * d_k + i]);
            double dpq = 0.0;
            for (int j = 0; j < dva; ++j) {
                dM[i * dva + j] += pqi * dOa[j];
                dpq += Mt[i * dva + j] * dOa[j];
            }
            dq[(size_t)t * d_k + i] = dpq * fmap_grad(s->feature_map, q[(size_t)t * d_k + i]);
        }
        for (int j = 0; j < d_v; ++j) dv[(size_t)t * d_v + j] = 0.0;
        double da_sum = 0.0;
        const double spb = (s->instance == LMO_MAMBA2) ? softplus(b_pre[t]) : 0.0;
        const double sb = (s->instance == LMO_MAMBA2) ? sigm(b_pre[t]) : 0.0;
        for (int i = 0; i < d_k; ++i) {
            double a = decay_at(s, d_k, a_pre, b_pre, t, i);
            double ke = keff_at(s, d_k, k, a_pre, b_pre, t, i);
            double dke = 0.0, da = 0.0;
            for (int j = 0; j < dva; ++j) {
                double g = dM[i * dva + j];
                dke += g * VA(t, j);
                if (j < d_v) dv[(size_t)t * d_v + j] += g * ke;
                da += g * Mp[i * dva + j];
                dM[i * dva + j] = a * g; /* propagate to M_{t-1} */
            }
            const double kraw = k[(size_t)t * d_k + i];
            /* effective key chain (lsm.hpp:483-501) */
            if (s->instance == LMO_HGRN2) {
                double sa = sigm(a_pre[(size_t)t * d_k + i]);
                dk[(size_t)t * d_k + i] = 0.0;
                da_pre[(size_t)t * d_k + i] += -dke * sa * (1.0 - sa);
            } else if (s->instance == LMO_MAMBA2) {
                dk[(size_t)t * d_k + i] = dke * spb * fmap_grad(s->feature_map, kraw);
                db_pre[t] += dke * fmap(s->feature_map, kraw) * sb;
            } else {
                dk[(size_t)t * d_k + i] = dke * fmap_grad(s->feature_map, kraw);
            }
            /* decay chain (lsm.hpp:504-518) */
            if (dkind == LMO_DK_TOKEN_VECTOR) {
                da_pre[(size_t)t * d_k + i] += da * a * (1.0 - a);
            } else if (dkind == LMO_DK_TOKEN_SCALAR) {
                da_sum += da;
            }
        }
        if (dkind == LMO_DK_TOKEN_SCALAR) {
            double a = decay_at(s, d_k, a_pre, b_pre, t, 0);
            double spa = softplus(s->mamba2_a_raw);
            db_pre[t] += da_sum * a * (-spa) * sb;
            draw += da_sum * a * (-spb) * sigm(s->mamba2_a_raw);
        }
    }
#undef VA
    if (da_raw) *da_raw = draw;
    if (dM0)
        for (int i = 0; i < d_k; ++i)
            for (int j = 0; j < d_v; ++j) dM0[(size_t)i * d_v + j] = dM[i * dva + j];
    free(Ms); free(dM); free(dOa);
    return 0;
}

/*
 * recurrent_step (lsm.hpp:335-441) for the kinds without a chunk-parallel form: DeltaNet,
 * GatedDeltaNet (StateLinear), GFW / GateLoop (TokenOuter), TTT / Titans / RWKV7 (Gradient,
 * kern::ttt_loss_grad lsm.hpp:328-330), S4 / Mamba (FullElementwise).  Gate layouts
 * (LsmGates, lsm.hpp:206-247): a_pre (n, d_k) for RWKV7 / Mamba, (n) for DeltaNet /
 * GatedDeltaNet / Titans; b_pre (n); alpha_pre (n, d_k); beta_pre (n, d_v).  Static params
 * (LsmSpec::make lsm.hpp:166-177): s4_delta_raw (d_k), s4_b (d_k), s4_A_raw / mamba_A_raw
 * (d_k, d_v).  No normaliser for these kinds (LsmSpec::validate).  o: (n, d_v).
 */
int lmo_lsm_recurrent(const lmo_spec* s, int n, int d_k, int d_v, const double* q, const double* k,
                      const double* v, const double* a_pre, const double* b_pre, const double* alpha_pre,
                      const double* beta_pre, const double* s4_delta_raw, const double* s4_b,
                      const double* s4_A_raw, const double* mamba_A_raw, const double* M0, double* o,
                      double* M_out, char* err, int errlen) {
    if (lmo_spec_validate(s, d_k, d_v, err, errlen)) return -1;
    const int inst = s->instance;
    if (!(inst == LMO_DELTANET || inst == LMO_GATED_DELTANET || inst == LMO_GFW || inst == LMO_GATELOOP ||
          inst == LMO_TTT || inst == LMO_TITANS || inst == LMO_RWKV7 || inst == LMO_S4 || inst == LMO_MAMBA)) {
        set_err(err, errlen, "lmo_lsm_recurrent: separable kind (use lmo_lsm_sequential)");
        return -1;
    }
    const size_t dd = (size_t)d_k * d_v;
    double* M = (double*)malloc(sizeof(double) * dd);
    double* P = (double*)malloc(sizeof(double) * dd);
    double* kk = (double*)malloc(sizeof(double) * d_k);
    double* c = (double*)malloc(sizeof(double) * d_v);
    if (M0) memcpy(M, M0, sizeof(double) * dd); else memset(M, 0, sizeof(double) * dd);
    int rc = 0;
    for (int t = 0; t < n && rc == 0; ++t) {
        const double* qt = q + (size_t)t * d_k;
        const double* kt = k + (size_t)t * d_k;
        const double* vt = v + (size_t)t * d_v;
        for (int i = 0; i < d_k; ++i) kk[i] = fmap(s->feature_map, kt[i]);
        if (inst == LMO_DELTANET || inst == LMO_GATED_DELTANET) {
            double nrm = 0.0; /* l2_normalize_rows (tensor.hpp:810-825), eps 1e-12 */
            for (int i = 0; i < d_k; ++i) nrm += kk[i] * kk[i];
            nrm = sqrt(nrm + 1e-12);
            for (int i = 0; i < d_k; ++i) kk[i] /= nrm;
        }
        /* c = k^ M (vecmat) for the projection / test-time-gradient kinds */
        for (int j = 0; j < d_v; ++j) {
            double acc = 0.0;
            for (int i = 0; i < d_k; ++i) acc += kk[i] * M[(size_t)i * d_v + j];
            c[j] = acc;
        }
        for (int i = 0; i < d_k; ++i)
            for (int j = 0; j < d_v; ++j) {
                const size_t e = (size_t)i * d_v + j;
                double m = M[e];
                switch (inst) {
                    case LMO_DELTANET: {
                        const double a = sigm(a_pre[t]), b = sigm(b_pre[t]);
                        m = m - a * kk[i] * c[j] + b * kk[i] * vt[j];
                        break;
                    }
                    case LMO_GATED_DELTANET: {
                        const double a = sigm(a_pre[t]), b = sigm(b_pre[t]);
                        m = a * (m - kk[i] * c[j]) + b * kk[i] * vt[j];
                        break;
                    }
                    case LMO_GFW:
                    case LMO_GATELOOP:
                        m = sigm(alpha_pre[(size_t)t * d_k + i]) * sigm(beta_pre[(size_t)t * d_v + j]) * m +
                            kk[i] * vt[j];
                        break;
                    case LMO_TTT:
                        m = m - sigm(b_pre[t]) * kk[i] * (c[j] - vt[j]);
                        break;
                    case LMO_TITANS:
                        m = sigm(a_pre[t]) * m - sigm(b_pre[t]) * kk[i] * (c[j] - vt[j]);
                        break;
                    case LMO_RWKV7:
                        m = sigm(a_pre[(size_t)t * d_k + i]) * m - sigm(b_pre[t]) * kk[i] * (c[j] - vt[j]);
                        break;
                    case LMO_S4: {
                        const double dl = softplus(s4_delta_raw[i]);
                        m = exp(-softplus(s4_A_raw[e]) * dl) * m + dl * s4_b[i] * vt[j];
                        break;
                    }
                    case LMO_MAMBA: {
                        const double dl = softplus(a_pre[(size_t)t * d_k + i]);
                        m = exp(-softplus(mamba_A_raw[e]) * dl) * m + dl * kk[i] * vt[j];
                        break;
                    }
                }
                P[e] = m;
            }
        memcpy(M, P, sizeof(double) * dd);
        rc = check_state(s, M, dd, err, errlen);
        for (int j = 0; j < d_v && rc == 0; ++j) {
            double acc = 0.0;
            for (int i = 0; i < d_k; ++i) acc += fmap(s->feature_map, qt[i]) * M[(size_t)i * d_v + j];
            o[(size_t)t * d_v + j] = acc;
        }
    }
    if (rc == 0 && M_out) memcpy(M_out, M, sizeof(double) * dd);
    free(M); free(P); free(kk); free(c);
    return rc;
}

/* route (moe.hpp:58-85) with softmax_rows (tensor.hpp:767-789) */
int lmo_route(const double* logits, int t, int e, int top_k, int* ids, double* gates,
              double* probs, char* err, int errlen) {
    if (top_k < 1 || top_k > e) { set_err(err, errlen, "route: bad top_k"); return -1; }
    int* order = (int*)malloc(sizeof(int) * e);
    char* sel = (char*)malloc((size_t)e);
    for (int r = 0; r < t; ++r) {
        const double* l = logits + (size_t)r * e;
        /* stable descending sort, ties -> lower id (insertion sort is stable) */
        for (int i = 0; i < e; ++i) order[i] = i;
        for (int i = 1; i < e; ++i) {
            int x = order[i], j = i - 1;
            while (j >= 0 && (l[order[j]] < l[x] || (l[order[j]] == l[x] && order[j] > x))) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = x;
        }
        memset(sel, 0, (size_t)e);
        for (int i = 0; i < top_k; ++i) sel[order[i]] = 1;
        int w = 0;
        for (int i = 0; i < e; ++i) if (sel[i]) ids[(size_t)r * top_k + w++] = i; /* ascending */
        /* masked softmax over the selection */
        double mx = -INFINITY;
        for (int i = 0; i < e; ++i) if (sel[i] && l[i] > mx) mx = l[i];
        double zs = 0.0;
        for (int i = 0; i < e; ++i) {
            double g = sel[i] ? exp(l[i] - mx) : 0.0;
            gates[(size_t)r * e + i] = g;
            zs += g;
        }
        for (int i = 0; i < e; ++i) gates[(size_t)r * e + i] /= zs;
        if (probs) {
            double m2 = -INFINITY, z2 = 0.0;
            for (int i = 0; i < e; ++i) if (l[i] > m2) m2 = l[i];
            for (int i = 0; i < e; ++i) { probs[(size_t)r * e + i] = exp(l[i] - m2); z2 += probs[(size_t)r * e + i]; }
            for (int i = 0; i < e; ++i) probs[(size_t)r * e + i] /= z2;
        }
    }
    free(order); free(sel);
    return 0;
}

/* load_balance_loss (moe.hpp:90-103) */
double lmo_load_balance_loss(const int* ids, const double* probs, int t, int e, int top_k) {
    double* frac = (double*)calloc((size_t)e, sizeof(double));
    for (size_t i = 0; i < (size_t)t * top_k; ++i) frac[ids[i]] += 1.0;
    const double slots = (double)t * top_k;
    double acc = 0.0;
    for (int j = 0; j < e; ++j) {
        double pm = 0.0;
        for (int r = 0; r < t; ++r) pm += probs[(size_t)r * e + j];
        acc += (frac[j] / slots) * (pm * (1.0 / t));
    }
    free(frac);
    return acc * (double)e;
}

static double silu(double x) { return x * sigm(x); }

/* MoeLayer::forward (moe.hpp:133-149), Expert::forward (:45-47) */
int lmo_moe_forward(const double* x, int t, int hidden, int ffn, int e, int top_k,
                    const double* router, const double* w_gate, const double* w_up,
                    const double* w_down, double* y, double* aux, double* logits_out,
                    char* err, int errlen) {
    if (e < 1 || top_k < 1 || top_k > e) { set_err(err, errlen, "MoeConfig: need 1 <= top_k <= num_experts"); return -1; }
    double* logits = (double*)malloc(sizeof(double) * t * e);
    for (int r = 0; r < t; ++r)
        for (int j = 0; j < e; ++j) {
            double acc = 0.0;
            for (int h = 0; h < hidden; ++h) acc += x[(size_t)r * hidden + h] * router[(size_t)h * e + j];
            logits[(size_t)r * e + j] = acc;
        }
    if (logits_out) memcpy(logits_out, logits, sizeof(double) * t * e);
    int* ids = (int*)malloc(sizeof(int) * t * top_k);
    double* gates = (double*)malloc(sizeof(double) * t * e);
    double* probs = (double*)malloc(sizeof(double) * t * e);
    if (lmo_route(logits, t, e, top_k, ids, gates, probs, err, errlen)) {
        free(logits); free(ids); free(gates); free(probs);
        return -1;
    }
    memset(y, 0, sizeof(double) * t * hidden);
    double* hbuf = (double*)malloc(sizeof(double) * ffn);
    double* obuf = (double*)malloc(sizeof(double) * hidden);
    for (int ex = 0; ex < e; ++ex) {
        const double* wg = w_gate + (size_t)ex * hidden * ffn;
        const double* wu = w_up + (size_t)ex * hidden * ffn;
        const double* wd = w_down + (size_t)ex * ffn * hidden;
        for (int r = 0; r < t; ++r) { /* tokens_of[ex] in ascending token order */
            int hit = 0;
            for (int s = 0; s < top_k; ++s) if (ids[(size_t)r * top_k + s] == ex) hit = 1;
            if (!hit) continue;
            const double* xr = x + (size_t)r * hidden;
            for (int f = 0; f < ffn; ++f) {
                double g = 0.0, u = 0.0;
                for (int h = 0; h < hidden; ++h) {
                    g += xr[h] * wg[(size_t)h * ffn + f];
                    u += xr[h] * wu[(size_t)h * ffn + f];
                }
                hbuf[f] = silu(g) * u;
            }
            for (int h = 0; h < hidden; ++h) {
                double acc = 0.0;
                for (int f = 0; f < ffn; ++f) acc += hbuf[f] * wd[(size_t)f * hidden + h];
                obuf[h] = acc;
            }
            const double ge = gates[(size_t)r * e + ex];
            for (int h = 0; h < hidden; ++h) y[(size_t)r * hidden + h] += obuf[h] * ge;
        }
    }
    *aux = lmo_load_balance_loss(ids, probs, t, e, top_k);
    free(hbuf); free(obuf); free(logits); free(ids); free(gates); free(probs);
    return 0;
}

/* chunk_range (parallel.hpp:192-197) */
void lmo_chunk_range(int n, int t, int rank, int* r0, int* r1) {
    int base = n / t, rem = n % t;
    *r0 = rank * base + (rank < rem ? rank : rem);
    *r1 = *r0 + base + (rank < rem ? 1 : 0);
}

int lmo_sp_payload_width(const lmo_spec* s, int d_v) {
    return d_v + (s->use_normalizer ? 1 : 0) + (lmo_decay_kind(s->instance) != LMO_DK_NONE ? 1 : 0);
}

/* local_chunk + payload build (parallel.hpp:249-275, 315-327) */
int lmo_sp_local_payload(const lmo_spec* s, int n_loc, int d_k, int d_v, int chunk,
                         const double* q, const double* k, const double* v,
                         const double* a_pre, const double* b_pre, double* payload,
                         char* err, int errlen) {
    const int pw = lmo_sp_payload_width(s, d_v);
    double* o = (double*)malloc(sizeof(double) * n_loc * d_v);
    double* M = (double*)malloc(sizeof(double) * d_k * d_v);
    double* z = (double*)malloc(sizeof(double) * d_k);
    int rc = lmo_lsm_chunked(s, n_loc, d_k, d_v, chunk > 0 ? chunk : n_loc, q, k, v, a_pre,
                             b_pre, NULL, NULL, o, M, z, err, errlen);
    if (rc == 0) {
        for (int i = 0; i < d_k; ++i) {
            int col = d_v;
            for (int j = 0; j < d_v; ++j) payload[i * pw + j] = M[i * d_v + j];
            if (s->use_normalizer) payload[i * pw + col++] = z[i];
            if (lmo_decay_kind(s->instance) != LMO_DK_NONE) {
                double d = 1.0;  /* total decay: product of the slice's decay rows (:270-271) */
                for (int t = 0; t < n_loc; ++t) d *= decay_at(s, d_k, a_pre, b_pre, t, i);
                payload[i * pw + col] = d;
            }
        }
    }
    free(o); free(M); free(z);
    return rc;
}

/* decayed exclusive prefix (parallel.hpp:340-361) */
void lmo_sp_combine(const lmo_spec* s, int d_k, int d_v, int rank, const double* gathered,
                    double* M_in, double* z_in) {
    const int pw = lmo_sp_payload_width(s, d_v);
    const int decayed = lmo_decay_kind(s->instance) != LMO_DK_NONE;
    double* factor = (double*)malloc(sizeof(double) * d_k);
    for (int i = 0; i < d_k; ++i) factor[i] = 1.0;
    memset(M_in, 0, sizeof(double) * d_k * d_v);
    if (z_in) memset(z_in, 0, sizeof(double) * d_k);
    for (int r = rank - 1; r >= 0; --r) {
        const double* p = gathered + (size_t)r * d_k * pw;
        for (int i = 0; i < d_k; ++i) {
            int col = d_v;
            for (int j = 0; j < d_v; ++j) M_in[i * d_v + j] += p[i * pw + j] * factor[i];
            if (s->use_normalizer) { if (z_in) z_in[i] += factor[i] * p[i * pw + col]; ++col; }
            if (decayed) factor[i] *= p[i * pw + col];
        }
    }
    free(factor);
}

/* sp_forward_nomask (parallel.hpp:391-403) / sp_lsm_nomask_rank (:282-297) */
int lmo_sp_forward_nomask(const lmo_spec* s, int n, int d_k, int d_v, int world,
                          const double* q, const double* k, const double* v, double* o,
                          char* err, int errlen) {
    if (lmo_spec_validate(s, d_k, d_v, err, errlen)) return -1;
    if (lmo_decay_kind(s->instance) != LMO_DK_NONE) {
        set_err(err, errlen, "sp_forward_nomask: requires an undecayed instance");
        return -1;
    }
    if (s->use_normalizer) { set_err(err, errlen, "sp_forward_nomask: normalizer unsupported"); return -1; }
    if (world < 1 || n < world) { set_err(err, errlen, "chunk_range: need at least one row per rank"); return -1; }
    const size_t dd = (size_t)d_k * d_v;
    double* Mg = (double*)calloc(dd, sizeof(double));
    double* Ml = (double*)malloc(sizeof(double) * dd);
    /* per rank: m_local = phi(K_r)^T V_r, then m_global = all[0] + all[1] + ... (rank order) */
    for (int r = 0; r < world; ++r) {
        int r0, r1;
        lmo_chunk_range(n, world, r, &r0, &r1);
        memset(Ml, 0, sizeof(double) * dd);
        for (int t = r0; t < r1; ++t)
            for (int i = 0; i < d_k; ++i) {
                const double pk = fmap(s->feature_map, k[(size_t)t * d_k + i]);
                for (int j = 0; j < d_v; ++j) Ml[i * d_v + j] += pk * v[(size_t)t * d_v + j];
            }
        for (size_t e = 0; e < dd; ++e) Mg[e] += Ml[e];
    }
    for (int t = 0; t < n; ++t)
        for (int j = 0; j < d_v; ++j) {
            double acc = 0.0;
            for (int i = 0; i < d_k; ++i) acc += fmap(s->feature_map, q[(size_t)t * d_k + i]) * Mg[i * d_v + j];
            o[(size_t)t * d_v + j] = acc;
        }
    free(Mg); free(Ml);
    return 0;
}

/* sp_forward_masked (parallel.hpp:405-418) / sp_lsm_masked_rank (:303-376) */
int lmo_sp_forward_masked(const lmo_spec* s, int n, int d_k, int d_v, int world,
                          int rank_chunk, const double* q, const double* k, const double* v,
                          const double* a_pre, const double* b_pre, double* o, char* err,
                          int errlen) {
    if (lmo_spec_validate(s, d_k, d_v, err, errlen)) return -1;
    if (check_separable(s, err, errlen)) return -1;
    if (n < world) { set_err(err, errlen, "chunk_range: need at least one row per rank"); return -1; }
    const int pw = lmo_sp_payload_width(s, d_v);
    double* gathered = (double*)malloc(sizeof(double) * world * d_k * pw);
    int rc = 0;
    for (int r = 0; r < world && rc == 0; ++r) {
        int r0, r1;
        lmo_chunk_range(n, world, r, &r0, &r1);
        rc = lmo_sp_local_payload(s, r1 - r0, d_k, d_v, rank_chunk,
                                  q + (size_t)r0 * d_k, k + (size_t)r0 * d_k, v + (size_t)r0 * d_v,
                                  a_pre ? a_pre + (size_t)r0 * d_k : NULL, b_pre ? b_pre + r0 : NULL,
                                  gathered + (size_t)r * d_k * pw, err, errlen);
    }
    double* M_in = (double*)malloc(sizeof(double) * d_k * d_v);
    double* z_in = (double*)malloc(sizeof(double) * d_k);
    for (int r = 0; r < world && rc == 0; ++r) {
        int r0, r1;
        lmo_chunk_range(n, world, r, &r0, &r1);
        lmo_sp_combine(s, d_k, d_v, r, gathered, M_in, z_in);
        int len = r1 - r0;
        rc = lmo_lsm_chunked(s, len, d_k, d_v, rank_chunk > 0 ? rank_chunk : len,
                             q + (size_t)r0 * d_k, k + (size_t)r0 * d_k, v + (size_t)r0 * d_v,
                             a_pre ? a_pre + (size_t)r0 * d_k : NULL, b_pre ? b_pre + r0 : NULL,
                             M_in, s->use_normalizer ? z_in : NULL, o + (size_t)r0 * d_v, NULL,
                             NULL, err, errlen);
    }
    free(gathered); free(M_in); free(z_in);
    return rc;
}

/* softmax_attention_parallel (attention.hpp:18-38) */
void lmo_attention(const double* q, const double* k, const double* v, int nq, int nk, int d,
                   int dv, int causal, int row_offset, double* o) {
    double* sc = (double*)malloc(sizeof(double) * nk);
    const double inv = 1.0 / sqrt((double)d);
    for (int i = 0; i < nq; ++i) {
        double mx = -INFINITY;
        for (int j = 0; j < nk; ++j) {
            double acc = 0.0;
            for (int e = 0; e < d; ++e) acc += q[(size_t)i * d + e] * k[(size_t)j * d + e];
            sc[j] = acc * inv;
            int keep = !causal || j <= i + row_offset;
            if (keep && sc[j] > mx) mx = sc[j];
        }
        double zs = 0.0;
        for (int j = 0; j < nk; ++j) {
            int keep = !causal || j <= i + row_offset;
            sc[j] = keep ? exp(sc[j] - mx) : 0.0;
            zs += sc[j];
        }
        for (int c = 0; c < dv; ++c) {
            double acc = 0.0;
            for (int j = 0; j < nk; ++j) acc += (sc[j] / zs) * v[(size_t)j * dv + c];
            o[(size_t)i * dv + c] = acc;
        }
    }
    free(sc);
}
