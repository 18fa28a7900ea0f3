"""Pins the C restatement (oracle/) to the reference's own outputs.

tests/golden/*.npz come from the unmodified reference headers
(tests/golden/make_golden.py); the oracle must reproduce them to f64 rounding.
Also restates the reference KATs (test_lsm.cpp, test_moe.cpp, test_parallel.cpp).
"""
import numpy as np
import pytest

import oracle
from conftest import golden_cases, load_golden


def _gates(d, p):
    return d.get(p + "/a_pre"), d.get(p + "/b_pre")


def test_lsm_small_chunked_and_sequential_match_reference():
    d = load_golden("lsm_small")
    cases = golden_cases({k: None for k in d if "/o_" in k or "/q" in k})
    n_checked = 0
    for p in sorted({k.split("/")[0] for k in d}):
        spec = oracle.spec_from_golden(d, p)
        q, k, v = d[p + "/q"], d[p + "/k"], d[p + "/v"]
        a, b = _gates(d, p)
        o, M, z = oracle.lsm_sequential(spec, q, k, v, a, b)
        assert np.abs(o - d[p + "/o_seq"]).max() < 1e-12, p
        assert np.abs(M - d[p + "/M_seq"]).max() < 1e-12, p
        n = q.shape[0]
        for c in (1, 3, 8, n):
            o, M, z = oracle.lsm_chunked(spec, q, k, v, a, b, chunk=c)
            assert np.abs(o - d[p + "/o_c%d" % c]).max() < 1e-12, (p, c)
            assert np.abs(M - d[p + "/M_c%d" % c]).max() < 1e-12, (p, c)
            if spec["use_normalizer"]:
                assert np.abs(z - d[p + "/z_c%d" % c]).max() < 1e-12, (p, c)
            n_checked += 1
    assert n_checked >= 90
    assert cases


def test_lsm_device_sizes_match_reference():
    d = load_golden("lsm_dev")
    for p in sorted({k.split("/")[0] for k in d}):
        spec = oracle.spec_from_golden(d, p)
        chunk = int(d[p + "/chunk"][0])
        a, b = _gates(d, p)
        o, M, z = oracle.lsm_chunked(spec, d[p + "/q"], d[p + "/k"], d[p + "/v"], a, b,
                                     chunk=chunk)
        # golden outputs are stored as float32
        scale = np.abs(d[p + "/o"]).max()
        assert np.abs(o - d[p + "/o"]).max() / scale < 1e-6, p
        assert np.abs(M - d[p + "/M"]).max() / np.abs(d[p + "/M"]).max() < 1e-6, p


def test_lsm_backward_matches_reference_tape():
    d = load_golden("lsm_grad")
    for p in sorted({k.split("/")[0] for k in d}):
        spec = oracle.spec_from_golden(d, p)
        a, b = _gates(d, p)
        g = oracle.lsm_backward(spec, d[p + "/q"], d[p + "/k"], d[p + "/v"], d[p + "/dO"], a, b)
        for name in ("dq", "dk", "dv"):
            assert np.abs(g[name] - d[p + "/" + name]).max() < 1e-10, (p, name)
        if p + "/da_pre" in d:
            assert np.abs(g["da_pre"] - d[p + "/da_pre"]).max() < 1e-10, p
        if p + "/db_pre" in d:
            assert np.abs(g["db_pre"] - d[p + "/db_pre"]).max() < 1e-10, p
        if p + "/da_raw" in d:
            assert abs(g["da_raw"] - d[p + "/da_raw"][0]) < 1e-10, p


def test_route_matches_reference_bit_exact_ids():
    d = load_golden("route")
    for p in sorted({k.split("/")[0] for k in d}):
        k = int(d[p + "/top_k"][0])
        ids, gates, probs = oracle.route(d[p + "/logits"], k)
        assert np.array_equal(ids, d[p + "/ids"].astype(np.int32)), p
        assert np.abs(gates - d[p + "/gates"]).max() < 1e-15, p
        assert np.abs(probs - d[p + "/probs"]).max() < 1e-15, p
        aux = oracle.load_balance_loss(ids, probs)
        assert abs(aux - d[p + "/aux"][0]) < 1e-13, p


def test_moe_forward_matches_reference():
    d = load_golden("moe")
    for p in sorted({k.split("/")[0] for k in d}):
        k = int(d[p + "/top_k"][0])
        y, aux, _ = oracle.moe_forward(d[p + "/x"], d[p + "/router"], d[p + "/w_gate"],
                                       d[p + "/w_up"], d[p + "/w_down"], k)
        assert np.abs(y - d[p + "/y"]).max() < 1e-13, p
        assert abs(aux - d[p + "/aux"][0]) < 1e-13, p


def test_sp_masked_matches_reference_all_world_sizes():
    d = load_golden("sp")
    for p in sorted({k.split("/")[0] for k in d}):
        spec = oracle.spec_from_golden(d, p)
        a, b = _gates(d, p)
        for t in (1, 2, 4, 8):
            o = oracle.sp_forward_masked(spec, d[p + "/q"], d[p + "/k"], d[p + "/v"], t, a, b)
            assert np.abs(o - d[p + "/o_t%d" % t]).max() < 1e-12, (p, t)
            assert np.abs(o - d[p + "/o_seq"]).max() < 1e-10, (p, t)
            # one gather of T * d_k * payload_width elements (test_parallel.cpp:124-148)
            pw = oracle.sp_payload_width(spec, d[p + "/v"].shape[1])
            assert d[p + "/comm_elems_t%d" % t][0] == t * d[p + "/q"].shape[1] * pw


def test_attention_row_offset_matches_reference():
    d = load_golden("attn")
    o = oracle.attention(d["q"], d["k"], d["v"], True, 0)
    assert np.abs(o - d["o_full"]).max() < 1e-14
    o2 = oracle.attention(d["q"][16:24], d["k"], d["v"], True, 16)
    assert np.abs(o2 - d["o_off"]).max() < 1e-14
    # KV all-gather SP == full attention; 2 gathers of N*d (test_parallel.cpp:195-210)
    for t in (2, 4):
        assert np.abs(d["o_sp_t%d" % t] - d["o_full"]).max() < 1e-12
        assert d["comm_elems_t%d" % t][0] == 2 * d["k"].size


# ---- reference KATs restated (test_lsm.cpp / test_moe.cpp / test_parallel.cpp) ----

def test_kat_bla_two_tokens():
    """test_lsm.cpp:18-29: o = [4, -12]."""
    spec = {"instance": 0, "feature_map": 0, "use_normalizer": 0}
    q = np.array([[2.0], [3.0]])
    k = np.array([[0.5], [-1.0]])
    v = np.array([[4.0], [6.0]])
    o, _, _ = oracle.lsm_sequential(spec, q, k, v)
    assert np.allclose(o[:, 0], [4.0, -12.0], rtol=1e-14)
    o, _, _ = oracle.lsm_chunked(spec, q, k, v, chunk=2)
    assert np.allclose(o[:, 0], [4.0, -12.0], rtol=1e-14)


def test_kat_retnet_geometric_sum():
    """test_lsm.cpp:48-66."""
    rng = np.random.default_rng(4)
    q, k, v = (rng.normal(0, 0.7, (7, 3)) for _ in range(3))
    spec = oracle.spec_default("retnet")
    o, _, _ = oracle.lsm_chunked(spec, q, k, v, chunk=3)
    a = spec["scalar_decay"]
    want = np.zeros_like(o)
    for s in range(7):
        for j in range(s + 1):
            want[s] += a ** (s - j) * (q[s] @ k[j]) * v[j]
    assert np.abs(o - want).max() < 1e-12


def test_kat_normalizer_ratio():
    """test_lsm.cpp:68-91."""
    rng = np.random.default_rng(5)
    q, k, v = (rng.normal(0, 0.5, (6, 3)) for _ in range(3))
    spec = oracle.spec_default("bla")
    o, _, _ = oracle.lsm_chunked(spec, q, k, v, chunk=4)
    phi = lambda x: np.where(x > 0, x + 1, np.exp(x))
    pq, pk = phi(q), phi(k)
    for s in range(6):
        w = np.array([pq[s] @ pk[j] for j in range(s + 1)])
        assert np.allclose(o[s], (w[:, None] * v[:s + 1]).sum(0) / w.sum(), rtol=1e-10)


def test_normalizer_restrictions_and_errors():
    """lsm.hpp:188-204 and :672 error texts (test_lsm.cpp:237-259)."""
    q = np.ones((4, 2))
    with pytest.raises(oracle.OracleError, match="normalizer unsupported for instance mamba2"):
        oracle.lsm_chunked({"instance": 13, "use_normalizer": 1}, q, q, q, b_pre=np.zeros(4))
    with pytest.raises(oracle.OracleError, match="chunk_size must be >= 1"):
        oracle.lsm_chunked({"instance": 0}, q, q, q, chunk=0)
    # rowsum(q.k) == 0 -> degenerate
    qq = np.array([[1.0, -1.0]] * 4)
    kk = np.array([[1.0, 1.0]] * 4)
    with pytest.raises(oracle.OracleError, match="degenerate normalizer in instance bla"):
        oracle.lsm_chunked({"instance": 0, "use_normalizer": 1}, qq, kk, q, chunk=2)


def test_kat_routing_ties_and_gates():
    """test_moe.cpp:9-47."""
    logits = np.array([[0.1, 0.9, 0.9, 0.2], [-1.0] * 4])
    ids, gates, _ = oracle.route(logits, 2)
    assert ids.tolist() == [[1, 2], [0, 1]]
    assert gates[0, 0] == 0.0 and abs(gates[0, 1] - 0.5) < 1e-12 and abs(gates[1, 0] - 0.5) < 1e-12
    with pytest.raises(oracle.OracleError, match="route: bad top_k"):
        oracle.route(logits, 5)
    ids, gates, _ = oracle.route(np.array([[1.0, 3.0, 2.0]]), 2)
    z = np.exp(3.0) + np.exp(2.0)
    assert abs(gates[0, 1] - np.exp(3.0) / z) < 1e-12


def test_kat_aux_loss():
    """test_moe.cpp:49-62: 1.0 under uniformity, ~2.0 under collapse."""
    t, e = 8, 4
    _, _, probs = oracle.route(np.zeros((t, e)), 1)
    ids = np.array([[i % e] for i in range(t)], dtype=np.int32)
    assert abs(oracle.load_balance_loss(ids, probs) - 1.0) < 1e-12
    ids, _, probs = oracle.route(np.array([[50.0, 0.0], [50.0, 0.0]]), 1)
    assert abs(oracle.load_balance_loss(ids, probs) - 2.0) < 1e-6


def test_kat_chunk_range_balanced():
    """parallel.hpp:192-197."""
    for n, t in ((10, 3), (32, 8), (7, 7), (100, 6)):
        sizes = [oracle.chunk_range(n, t, r) for r in range(t)]
        assert sizes[0][0] == 0 and sizes[-1][1] == n
        lens = [b - a for a, b in sizes]
        assert max(lens) - min(lens) <= 1
        assert all(sizes[i][1] == sizes[i + 1][0] for i in range(t - 1))


def test_kat_prefix_sums():
    """test_parallel.cpp:72-85 via the SP combine: 0, A, A+B with unit decay."""
    spec = {"instance": 0, "use_normalizer": 0}  # undecayed: payload is M only
    states = np.stack([np.full((2, 2), 1.0), np.full((2, 2), 2.0), np.full((2, 2), 3.0)])
    for r, want in ((0, 0.0), (1, 1.0), (2, 3.0)):
        M, _ = oracle.sp_combine(spec, states, r, 2)
        assert np.all(M == want)


def test_sp_nomask_matches_reference():
    """sp_forward_nomask (parallel.hpp:391-403) outputs and comm volume vs the reference."""
    d = load_golden("spn")
    for p in sorted({k.split("/")[0] for k in d}):
        spec = oracle.spec_from_golden(d, p)
        q, k, v = d[p + "/q"], d[p + "/k"], d[p + "/v"]
        for t in (1, 2, 4, 8):
            o = oracle.sp_forward_nomask(spec, q, k, v, t)
            assert np.abs(o - d[p + "/o_t%d" % t]).max() < 1e-12, (p, t)
            # one all-gather of T * d_k * d_v elements (parallel.hpp:279-281)
            assert int(d[p + "/comm_elems_t%d" % t][0]) == t * q.shape[1] * v.shape[1]
    with pytest.raises(oracle.OracleError, match="requires an undecayed instance"):
        oracle.sp_forward_nomask(oracle.spec_default("retnet"), q, k, v, 2)


def test_backward_final_state_gradient_matches_finite_differences():
    """dM_final seeding of the oracle backward (the gradient the reference tape sends back
    through lsm_forward_chunked's final_state, lsm.hpp:668-708) for a TokenVector kind."""
    rng = np.random.default_rng(11)
    n, d = 37, 5
    sp = oracle.spec_default("gla")
    q, k, v, a = (rng.normal(0, 0.5, (n, d)) for _ in range(4))
    M0 = rng.normal(0, 0.3, (d, d))
    dO = rng.normal(0, 1, (n, d))
    dMf = rng.normal(0, 1, (d, d))
    g = oracle.lsm_backward(sp, q, k, v, dO, a_pre=a, M0=M0, dM_final=dMf)

    def loss(q_, k_, v_, a_, M0_):
        o, M, _ = oracle.lsm_chunked(sp, q_, k_, v_, a_pre=a_, chunk=8, M0=M0_)
        return float((o * dO).sum() + (M * dMf).sum())

    args = [q, k, v, a, M0]
    for i, name in enumerate(["dq", "dk", "dv", "da_pre", "dM0"]):
        u = rng.normal(0, 1, args[i].shape)
        plus = list(args); plus[i] = args[i] + 1e-6 * u
        minus = list(args); minus[i] = args[i] - 1e-6 * u
        fd = (loss(*plus) - loss(*minus)) / 2e-6
        an = float((g[name] * u).sum())
        assert abs(an - fd) < 1e-6 * max(1.0, abs(fd)), (name, an, fd)



def test_recurrent_kinds_match_reference():
    """lmo_lsm_recurrent against the reference's recurrent_step / lsm_forward_chunked for the
    nine kinds without a chunk-parallel form (tests/golden/lsm_seq.npz, d = 8)."""
    d = load_golden("lsm_seq")
    ran = 0
    for p in sorted({k.split("/")[0] for k in d}):
        spec = oracle.spec_from_golden(d, p)
        g = lambda n: d.get(p + "/" + n)
        o, M = oracle.lsm_recurrent(spec, g("q"), g("k"), g("v"), g("a_pre"), g("b_pre"), g("alpha_pre"),
                                    g("beta_pre"), g("s4_delta_raw"), g("s4_b"), g("s4_A_raw"), g("mamba_A_raw"))
        assert np.abs(o - g("o_seq")).max() < 1e-10, p
        assert np.abs(M - g("M_seq")).max() < 1e-10, p
        assert np.abs(g("o_c8") - g("o_seq")).max() < 1e-10, p  # chunked == sequential (reference)
        ran += 1
    assert ran == 18


REC_INPUTS = ("a_pre", "b_pre", "alpha_pre", "beta_pre", "s4_delta_raw", "s4_b", "s4_A_raw", "mamba_A_raw")


def rec_loss(d, p, x, w, Mw=None):
    """sum(o * w) [+ sum(M_N * Mw)] of the f64 oracle recurrence (lmo_lsm_recurrent) at inputs x."""
    sd = oracle.spec_from_golden(d, p)
    o, M = oracle.lsm_recurrent(sd, x["q"], x["k"], x["v"], *(x.get(n) for n in REC_INPUTS), M0=x.get("M0"))
    return float((o * w).sum() + (0.0 if Mw is None else (M * Mw).sum()))


def test_recurrent_kinds_tape_gradients_pin_the_oracle():
    """The reference tape's gradients of the nine recurrent kinds (tests/golden/lsm_rec_grad.npz,
    tensor.hpp:1178 over recurrent_step lsm.hpp:335-441) equal central differences of the f64
    oracle recurrence along random directions -- the check the GPU backward tests then use at
    sizes the tape cannot reach (tensor.hpp:1222-1240 is the reference's own FD oracle)."""
    d = load_golden("lsm_rec_grad")
    rng = np.random.default_rng(5)
    for p in golden_cases(d):
        x = {n: d[p + "/" + n] for n in ("q", "k", "v") + REC_INPUTS if p + "/" + n in d}
        w = d[p + "/dO"]
        for name in x:
            g = d[p + "/d" + name]
            for _ in range(2):
                u = rng.normal(0, 1, x[name].shape)
                eps = 1e-5
                xp, xm = dict(x), dict(x)
                xp[name] = x[name] + eps * u
                xm[name] = x[name] - eps * u
                fd = (rec_loss(d, p, xp, w) - rec_loss(d, p, xm, w)) / (2 * eps)
                an = float((g * u).sum())
                assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (p, name, fd, an)
