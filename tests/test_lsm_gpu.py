"""GPU parity of the sm_100a LSM forward (liblmoe_cuda.so via the C-ABI) against the
float64 oracle (oracle/, pinned to the reference by tests/golden) and against the
reference's own golden vectors.

Tolerances (north star): norm-relative max|got-want|/max|want| per (b,h)
  fp32 inputs (tf32 tensor cores, fp32 accumulate): 1e-3
  bf16 inputs (bf16 operands, fp32 accumulate):     2e-2
"""
import zlib

import numpy as np
import pytest

import oracle
from conftest import load_golden, norm_rel_err

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-3, "bf16": 2e-2}
DEVICE_INSTANCES = {0, 1, 2, 3, 6, 13, 14, 15}  # every separable kind (DecayKind None/Const/Token*)


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _run(spec_d, q, k, v, b_pre=None, dtype="bf16", chunk=64, final=False, a_pre=None):
    """q,k,v numpy [B,N,H,D]; returns numpy o (f64) [+ final state]."""
    torch = _torch()
    import paper_2503_05447_b200 as pk
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dev = torch.device("cuda:0")
    Q, K, V = (torch.tensor(np.ascontiguousarray(x), dtype=torch.float32, device=dev).to(tdt)
               for x in (q, k, v))
    spec = pk.LsmSpec(instance=spec_d["instance"], feature_map=spec_d.get("feature_map", 0),
                      use_normalizer=bool(spec_d.get("use_normalizer", 0)),
                      scalar_decay=spec_d.get("scalar_decay", 1.0),
                      mamba2_a_raw=spec_d.get("mamba2_a_raw_h"))
    gates = None
    if b_pre is not None:
        gates = pk.LsmGates(b_pre=torch.tensor(np.ascontiguousarray(b_pre), dtype=torch.float32, device=dev))
    if a_pre is not None:
        gates = pk.LsmGates(a_pre=torch.tensor(np.ascontiguousarray(a_pre), dtype=torch.float32, device=dev).to(tdt))
    fs = pk.MemoryState() if final else None
    o = pk.lsm_forward_batched(Q, K, V, gates, spec, chunk, final_state=fs)
    torch.cuda.synchronize()
    out = o.float().cpu().numpy().astype(np.float64)
    if final:
        return out, fs.M.cpu().numpy().astype(np.float64), (None if fs.z is None else fs.z.cpu().numpy())
    return out


def _bf16_round(x):
    torch = _torch()
    return torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).float().numpy().astype(np.float64)


def test_golden_device_cases():
    """Reference outputs (tests/golden/lsm_dev.npz, bf16-exact inputs) on the device path."""
    d = load_golden("lsm_dev")
    cases = sorted({k.split("/")[0] for k in d})
    ran = 0
    for p in cases:
        spec = oracle.spec_from_golden(d, p)
        if spec["instance"] not in DEVICE_INSTANCES:
            continue
        q, k, v = (d[p + "/" + n].astype(np.float64) for n in "qkv")
        n, dd = q.shape
        dtype = "f32" if dd == 64 else "bf16"
        spec["mamba2_a_raw_h"] = [spec["mamba2_a_raw"]]
        b_pre = d.get(p + "/b_pre")
        a_pre = d.get(p + "/a_pre")
        o, M, z = _run(spec, q[None, :, None], k[None, :, None], v[None, :, None],
                       None if b_pre is None else b_pre[None, :, None].astype(np.float64),
                       dtype=dtype, chunk=int(d[p + "/chunk"][0]), final=True,
                       a_pre=None if a_pre is None else a_pre[None, :, None].astype(np.float64))
        err = norm_rel_err(o[0, :, 0], d[p + "/o"])
        assert err < TOL[dtype], (p, err)
        errM = norm_rel_err(M[0, 0], d[p + "/M"])
        assert errM < TOL[dtype], (p, "M", errM)
        ran += 1
    assert ran >= 12


@pytest.mark.parametrize("inst,fm,norm,dtype,N,H", [
    ("bla", 0, 0, "f32", 2048, 8),        # config 1, plain (test_lsm.cpp:35 / verify.hpp:77)
    ("bla", 1, 1, "f32", 2048, 8),        # config 1, reference default elu+1 + normaliser
    ("bla", 0, 0, "bf16", 1000, 2),
    ("rebased", 2, 1, "bf16", 700, 2),
    ("lightning", 0, 0, "bf16", 1500, 3),
    ("retnet", 0, 0, "bf16", 1029, 2),
    ("retnet", 0, 0, "f32", 515, 2),
    ("mamba2", 0, 0, "bf16", 1300, 2),
    ("mamba2", 0, 0, "f32", 640, 2),
    ("gla", 0, 0, "bf16", 1000, 2),
    ("gla", 0, 0, "f32", 600, 2),
    ("gla", 1, 1, "bf16", 700, 2),
    ("hgrn2", 0, 0, "bf16", 900, 2),
    ("rwkv6", 0, 0, "f32", 515, 2),
])
def test_random_vs_oracle(inst, fm, norm, dtype, N, H):
    rng = np.random.default_rng(zlib.crc32(repr((inst, fm, norm, dtype, N)).encode()))
    D = 64 if dtype == "f32" else 128
    B = 1
    q, k, v = (rng.normal(0, 0.5, (B, N, H, D)) for _ in range(3))
    if dtype == "bf16":
        q, k, v = _bf16_round(q), _bf16_round(k), _bf16_round(v)
    spec = oracle.spec_default(inst)
    spec["feature_map"], spec["use_normalizer"] = fm, norm
    a_raw = rng.normal(0, 0.5, H)
    b_pre = None
    if inst == "mamba2":
        b_pre = rng.normal(-1.0, 1.0, (B, N, H)).astype(np.float32).astype(np.float64)
        a_raw = a_raw.astype(np.float32).astype(np.float64)
    spec["mamba2_a_raw_h"] = a_raw
    a_pre = None
    if inst in ("gla", "hgrn2", "rwkv6"):  # reference default gates N(0,1) (lsm.hpp:222-253)
        a_pre = rng.normal(0, 1, (B, N, H, D))
        a_pre = _bf16_round(a_pre) if dtype == "bf16" else a_pre.astype(np.float32).astype(np.float64)
    o, M, z = _run(spec, q, k, v, b_pre, dtype=dtype, final=True, a_pre=a_pre)
    for h in range(H):
        sh = dict(spec, mamba2_a_raw=float(a_raw[h]))
        want, Mw, zw = oracle.lsm_chunked(sh, q[0, :, h], k[0, :, h], v[0, :, h],
                                          a_pre=None if a_pre is None else a_pre[0, :, h],
                                          b_pre=None if b_pre is None else b_pre[0, :, h], chunk=64)
        err = norm_rel_err(o[0, :, h], want)
        assert err < TOL[dtype], (inst, h, err)
        assert norm_rel_err(M[0, h], Mw) < TOL[dtype], (inst, h, "M")
        if norm:
            assert norm_rel_err(z[0, h], zw) < TOL[dtype], (inst, h, "z")


def test_chunk_size_invariance_and_initial_state():
    """Chunked == sequential for any chunk size (lsm.hpp:641-642); an initial state equals
    running the prefix first (the SP carried-in state, parallel.hpp:366-373)."""
    torch = _torch()
    import paper_2503_05447_b200 as pk
    rng = np.random.default_rng(7)
    N, H, D = 900, 2, 128
    q, k, v = (torch.tensor(rng.normal(0, 0.5, (1, N, H, D)), dtype=torch.bfloat16, device="cuda")
               for _ in range(3))
    spec = pk.LsmSpec.make("retnet", D)
    o1 = pk.lsm_forward_batched(q, k, v, None, spec, 1)
    o2 = pk.lsm_forward_batched(q, k, v, None, spec, 77)
    assert torch.equal(o1, o2)
    cut = 384
    fs = pk.MemoryState()
    oa = pk.lsm_forward_batched(q[:, :cut], k[:, :cut], v[:, :cut], None, spec, 64, final_state=fs)
    ob = pk.lsm_forward_batched(q[:, cut:], k[:, cut:], v[:, cut:], None, spec, 64, initial_state=fs)
    full = o1.float()
    err = (torch.cat([oa, ob], 1).float() - full).abs().max() / full.abs().max()
    assert err.item() < 2e-2


def test_errors_mirror_reference_text():
    torch = _torch()
    import paper_2503_05447_b200 as pk
    q = torch.zeros(1, 8, 1, 128, dtype=torch.bfloat16, device="cuda")
    spec = pk.LsmSpec.make("mamba2", 128)
    spec.mamba2_a_raw = 0.5
    spec.use_normalizer = True
    with pytest.raises(pk.LmoeError, match="LsmSpec: normalizer unsupported for instance mamba2"):
        pk.lsm_forward_batched(q, q, q, None, spec, 64)
    with pytest.raises(pk.LmoeError, match="chunk_size must be >= 1"):
        pk.lsm_forward_batched(q, q, q, None, pk.LsmSpec.make("bla", 128), 0)
    # degenerate normaliser: phi(q).phi(k) sums to 0 with the squared map only if all zero
    spec = pk.LsmSpec.make("rebased", 128)
    with pytest.raises(pk.LmoeError, match="degenerate normalizer in instance rebased"):
        pk.lsm_forward_batched(q, q, q, None, spec, 64)


def test_large_config2_heads_subset():
    """Config 2 shape (Lightning/RetNet, H=16, d=128, N=32K, bf16); two heads vs the oracle."""
    torch = _torch()
    import paper_2503_05447_b200 as pk
    N, H, D = 32768, 16, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16)
               for _ in range(3))
    for inst in ("lightning", "retnet"):
        spec = pk.LsmSpec.make(inst, D)
        o = pk.lsm_forward_batched(q, k, v, None, spec, 64)
        torch.cuda.synchronize()
        assert torch.isfinite(o.float()).all()
        for h in (0, 11):
            qq, kk, vv = (t[0, :, h].float().cpu().numpy().astype(np.float64) for t in (q, k, v))
            want, _, _ = oracle.lsm_chunked(oracle.spec_default(inst), qq, kk, vv, chunk=128)
            err = norm_rel_err(o[0, :, h].float().cpu().numpy(), want)
            assert err < 2e-2, (inst, h, err)



@pytest.mark.parametrize("inst", ["retnet", "mamba2", "gla"])
def test_varlen_matches_per_document_calls(inst):
    """Packed documents (lmoe_lsm_fwd_varlen / _bwd_varlen) equal independent per-document calls
    (the state is zero at every boundary), forward and backward; one document vs the oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200.lsm import lsm_backward_varlen, lsm_forward_varlen
    bounds = [0, 300, 337, 1000, 1129]
    T, H, D = bounds[-1], 2, 128
    g = torch.Generator(device="cuda").manual_seed(4)
    q, k, v, dO = (torch.randn(1, T, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(4))
    spec = pk.LsmSpec.make(inst, D)
    gates = None
    if inst == "mamba2":
        spec.mamba2_a_raw = torch.tensor([0.3, -0.2], device="cuda")
        gates = pk.LsmGates(b_pre=torch.randn(1, T, H, device="cuda", generator=g))
    elif inst == "gla":
        gates = pk.LsmGates(a_pre=torch.randn(1, T, H, D, device="cuda", generator=g).add_(2.0).bfloat16())
    o, M = lsm_forward_varlen(q, k, v, gates, spec, bounds, final_states=True)
    gv = lsm_backward_varlen(q, k, v, gates, spec, dO, bounds)
    dar = torch.zeros(H, device="cuda")
    for i in range(len(bounds) - 1):
        r0, r1 = bounds[i], bounds[i + 1]
        sl = lambda t: None if t is None else t[:, r0:r1].contiguous()
        gd = None if gates is None else pk.LsmGates(a_pre=sl(gates.a_pre), b_pre=sl(gates.b_pre))
        fs = pk.MemoryState()
        od = pk.lsm_forward_batched(sl(q), sl(k), sl(v), gd, spec, 64, final_state=fs)
        assert torch.equal(o[:, r0:r1], od), i
        assert torch.equal(M[i], fs.M[0]), i
        gr = pk.lsm_backward_batched(sl(q), sl(k), sl(v), gd, spec, sl(dO))
        for n in ("dq", "dk", "dv", "da_pre", "db_pre"):
            a, b = getattr(gv, n), getattr(gr, n)
            if b is not None:
                assert torch.equal(a[:, r0:r1], b), (i, n)
        if gr.da_raw is not None:
            dar += gr.da_raw
    if gv.da_raw is not None:
        assert torch.allclose(gv.da_raw, dar, rtol=1e-5, atol=1e-6)
    # document 1 (37 tokens) against the oracle from the zero state
    r0, r1 = bounds[1], bounds[2]
    for h in range(H):
        sd = oracle.spec_default(inst)
        b = a = None
        if inst == "mamba2":
            sd["mamba2_a_raw"] = float(spec.mamba2_a_raw[h])
            b = gates.b_pre[0, r0:r1, h].cpu().numpy()
        if inst == "gla":
            a = gates.a_pre[0, r0:r1, h].float().cpu().numpy()
        want, _, _ = oracle.lsm_chunked(sd, *(t[0, r0:r1, h].float().cpu().numpy() for t in (q, k, v)), a_pre=a,
                                        b_pre=b)
        assert norm_rel_err(o[0, r0:r1, h].float().cpu().numpy(), want) < 2e-2
