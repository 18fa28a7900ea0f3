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


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("a_raw_h,b_mean", [(0.0, -3.0), (1.5, 0.0), (3.0, 1.5)])
def test_mamba2_decay_regimes(dtype, a_raw_h, b_mean):
    """Mamba2 across decay regimes against the sequential oracle (lsm.hpp:643-662): long
    memory; default-like; strong decays whose 32-token quarters exceed the factorisation bound
    on some chunks, so the exact per-element path runs next to the factored one in one launch.
    Short and ragged lengths (1, 63, 129) exercise single-chunk CTAs and partial chunks."""
    rng = np.random.default_rng(zlib.crc32(repr((dtype, a_raw_h, b_mean)).encode()))
    D = 64 if dtype == "f32" else 128
    H = 3
    for N in (1, 63, 129, 777):
        q, k, v = (rng.normal(0, 0.5, (1, N, H, D)) for _ in range(3))
        if dtype == "bf16":
            q, k, v = _bf16_round(q), _bf16_round(k), _bf16_round(v)
        spec = oracle.spec_default("mamba2")
        a_raw = (a_raw_h + rng.normal(0, 0.3, H)).astype(np.float32).astype(np.float64)
        spec["mamba2_a_raw_h"] = a_raw
        b_pre = rng.normal(b_mean, 1.5, (1, N, H)).astype(np.float32).astype(np.float64)
        o, M, _ = _run(spec, q, k, v, b_pre, dtype=dtype, final=True)
        for h in range(H):
            sh = dict(spec, mamba2_a_raw=float(a_raw[h]))
            want, Mw, _ = oracle.lsm_sequential(sh, q[0, :, h], k[0, :, h], v[0, :, h], b_pre=b_pre[0, :, h])
            # fp32 inputs run the chunk GEMMs in tf32 (round-to-nearest, fp32 accumulation): a
            # single-token output is one tf32 dot product and can carry ~5e-3 under cancellation
            tol = 1e-2 if (dtype == "f32" and N == 1) else TOL[dtype]
            assert norm_rel_err(o[0, :, h], want) < tol, (N, h, a_raw_h, norm_rel_err(o[0, :, h], want))
            assert norm_rel_err(M[0, h], Mw) < tol, (N, h, "M")


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


# ------------------------------------------------ kinds without a chunk-parallel form (8(f) rank 4)
REC_KINDS = ["deltanet", "gated_deltanet", "gfw", "gateloop", "ttt", "titans", "rwkv7", "s4", "mamba"]


def _rec_inputs(d, p, D, B=1, H=1, dtype="bf16"):
    """Golden lsm_seq record -> padded device inputs (zero q / k / v columns keep the first d x d
    block of the problem: padded keys add nothing, padded rows of M are never read by q)."""
    import torch
    import paper_2503_05447_b200 as pk
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dd = d[p + "/q"].shape[1]
    padc = lambda x: np.pad(x, ((0, 0), (0, D - x.shape[1])))
    dev = lambda x, dt=tdt: torch.tensor(x, dtype=torch.float32, device="cuda").to(dt)
    q, k, v = (dev(padc(d[p + "/" + n]))[None, :, None] for n in ("q", "k", "v"))
    g = pk.LsmGates()
    a = d.get(p + "/a_pre")
    if a is not None:
        g.a_pre = dev(padc(a))[None, :, None] if a.ndim == 2 else dev(a, torch.float32)[None, :, None]
    if p + "/b_pre" in d:
        g.b_pre = dev(d[p + "/b_pre"], torch.float32)[None, :, None]
    for n in ("alpha_pre", "beta_pre"):
        if p + "/" + n in d:
            setattr(g, n, dev(padc(d[p + "/" + n]))[None, :, None])
    spec = pk.LsmSpec(instance=int(d[p + "/instance"][0]), feature_map=int(d[p + "/feature_map"][0]))
    if p + "/s4_delta_raw" in d:
        spec.s4_delta_raw = dev(np.pad(d[p + "/s4_delta_raw"], (0, D - dd)), torch.float32)[None]
        spec.s4_b = dev(np.pad(d[p + "/s4_b"], (0, D - dd)), torch.float32)[None]
        spec.s4_A_raw = dev(np.pad(d[p + "/s4_A_raw"], ((0, D - dd), (0, D - dd))), torch.float32)[None]
    if p + "/mamba_A_raw" in d:
        spec.mamba_A_raw = dev(np.pad(d[p + "/mamba_A_raw"], ((0, D - dd), (0, D - dd))), torch.float32)[None]
    return q, k, v, g, spec


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_recurrent_kinds_match_reference(dtype):
    """lmoe_lsm_fwd_recurrent for the nine kinds against the f64 oracle (pinned to the
    reference's recurrent_step, tests/golden/lsm_seq.npz) on the same rounded inputs."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_05447_b200.lsm import lsm_forward_recurrent
    import paper_2503_05447_b200 as pk
    d = load_golden("lsm_seq")
    D = 64 if dtype == "f32" else 128
    tol = 1e-3 if dtype == "f32" else 2e-2
    ran = 0
    for p in sorted({k.split("/")[0] for k in d}):
        q, k, v, g, spec = _rec_inputs(d, p, D, dtype=dtype)
        fs = pk.MemoryState()
        o = lsm_forward_recurrent(q, k, v, g, spec, final_state=fs)
        torch.cuda.synchronize()
        dd = d[p + "/q"].shape[1]
        cut = lambda t: None if t is None else t.float().cpu().numpy()
        sdict = oracle.spec_from_golden(d, p)
        args = [cut(q[0, :, 0, :dd]), cut(k[0, :, 0, :dd]), cut(v[0, :, 0, :dd])]
        a = g.a_pre
        args.append(None if a is None else (cut(a[0, :, 0, :dd]) if a.dim() == 4 else cut(a[0, :, 0])))
        args.append(None if g.b_pre is None else cut(g.b_pre[0, :, 0]))
        args.append(None if g.alpha_pre is None else cut(g.alpha_pre[0, :, 0, :dd]))
        args.append(None if g.beta_pre is None else cut(g.beta_pre[0, :, 0, :dd]))
        args.append(None if spec.s4_delta_raw is None else cut(spec.s4_delta_raw[0, :dd]))
        args.append(None if spec.s4_b is None else cut(spec.s4_b[0, :dd]))
        args.append(None if spec.s4_A_raw is None else cut(spec.s4_A_raw[0, :dd, :dd]))
        args.append(None if spec.mamba_A_raw is None else cut(spec.mamba_A_raw[0, :dd, :dd]))
        want_o, want_M = oracle.lsm_recurrent(sdict, *args)
        assert norm_rel_err(o[0, :, 0, :dd].float().cpu().numpy(), want_o) < tol, (p, dtype)
        assert norm_rel_err(fs.M[0, 0, :dd, :dd].cpu().numpy(), want_M) < tol, (p, dtype)
        assert np.abs(o[0, :, 0, dd:].float().cpu().numpy()).max() == 0.0  # padded value columns
        ran += 1
    assert ran == 18


def test_recurrent_kinds_random_heads_and_errors():
    """Full head dim, several heads / batch rows, an initial state; error texts."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200.lsm import lsm_forward_recurrent
    B, N, H, D = 2, 150, 2, 128
    rng = np.random.default_rng(9)
    T = lambda x, dt=torch.bfloat16: torch.tensor(x, dtype=torch.float32, device="cuda").to(dt)
    q, k, v = (T(rng.normal(0, 0.5, (B, N, H, D))) for _ in range(3))
    M0 = rng.normal(0, 0.1, (B, H, D, D))
    for inst in ("gated_deltanet", "rwkv7"):
        spec = pk.LsmSpec.make(inst, D)
        if inst == "gated_deltanet":
            g = pk.LsmGates(a_pre=T(rng.normal(2, 1, (B, N, H)), torch.float32),
                            b_pre=T(rng.normal(0, 1, (B, N, H)), torch.float32))
        else:
            g = pk.LsmGates(a_pre=T(rng.normal(2, 1, (B, N, H, D))), b_pre=T(rng.normal(0, 1, (B, N, H)), torch.float32))
        o = lsm_forward_recurrent(q, k, v, g, spec, initial_state=pk.MemoryState(M=T(M0, torch.float32)))
        torch.cuda.synchronize()
        for b in range(B):
            for h in range(H):
                sd = oracle.spec_default(inst)
                a = g.a_pre[b, :, h].float().cpu().numpy()
                want, _ = oracle.lsm_recurrent(sd, *(t[b, :, h].float().cpu().numpy() for t in (q, k, v)), a,
                                               g.b_pre[b, :, h].cpu().numpy(), M0=M0[b, h])
                assert norm_rel_err(o[b, :, h].float().cpu().numpy(), want) < 2e-2, (inst, b, h)
    with pytest.raises(pk.LmoeError, match="needs a_pre"):
        lsm_forward_recurrent(q, k, v, pk.LsmGates(), pk.LsmSpec.make("deltanet", D))
    with pytest.raises(pk.LmoeError, match="chunk-parallel form"):
        lsm_forward_recurrent(q, k, v, None, pk.LsmSpec.make("retnet", D))


@pytest.mark.parametrize("N", [2305, 2433])
def test_decay_free_bf16_long_segments(N):
    """A decay-free bf16 state pass with identity map and no normaliser has no per-token
    transform; its decay warp must not wait for ring-slot releases nobody makes.  At H = 16
    these lengths plan 3-chunk segments (the deadlock hit every segment of >= 3 chunks)."""
    import torch
    import paper_2503_05447_b200 as pk
    H = 16
    g = torch.Generator(device="cuda").manual_seed(N)
    q, k, v = (torch.randn(1, N, H, 128, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16) for _ in range(3))
    plain = pk.LsmSpec(instance=pk.LsmInstance.BLA, feature_map=0, use_normalizer=False)
    o = pk.lsm_forward_batched(q, k, v, None, plain, 64)
    torch.cuda.synchronize()
    sd = dict(oracle.spec_default(0), feature_map=0, use_normalizer=0)
    for h in (0, H - 1):
        want, _, _ = oracle.lsm_chunked(sd, *(t[0, :, h].float().cpu().numpy() for t in (q, k, v)), chunk=64)
        assert norm_rel_err(o[0, :, h].float().cpu().numpy(), want) < 2e-2
