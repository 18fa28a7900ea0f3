"""The single-read persistent LSM forward (csrc/lsm_fused.cuh): bf16 / d = 128 scalar-decay
kinds without normaliser run as ONE launch in which P CTAs per head hand the inclusive prefix
state from segment to segment.  Checked against the float64 oracle (lsm_forward_chunked,
lsm.hpp:668-708) over ragged lengths, batch > 1, a carried-in initial state and the final
state, and against the segment-parallel three-pass path (LMOE_FUSED=0) on the same inputs."""
import os

import numpy as np
import pytest

import oracle
from conftest import norm_rel_err, record_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fused_on(monkeypatch):
    """The single-read kernel is opt-in (LMOE_FUSED=1); these tests switch it on."""
    monkeypatch.setenv("LMOE_FUSED", "1")
TOL = 2e-2
D = 128


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _spec(pk, inst):
    if inst == "bla_plain":
        return pk.LsmSpec(instance=pk.LsmInstance.BLA, feature_map=0, use_normalizer=False), {"instance": 0}
    if inst == "bla_elu":
        return pk.LsmSpec(instance=pk.LsmInstance.BLA, feature_map=1, use_normalizer=False), {"instance": 0, "feature_map": 1}
    if inst == "rebased_plain":
        return (pk.LsmSpec(instance=pk.LsmInstance.REBASED, feature_map=2, use_normalizer=False),
                {"instance": 6, "feature_map": 2})
    s = pk.LsmSpec.make(inst, D)
    sd = oracle.spec_default(inst)
    return s, sd


def _inputs(torch, B, N, H, seed, scale=0.5, long_memory=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(B, N, H, D, device="cuda", generator=g).mul_(scale).bfloat16() for _ in range(3))
    b = torch.randn(B, N, H, device="cuda", generator=g)
    if long_memory:
        b = b.mul_(0.5).sub_(3.0)
    return q, k, v, b


def _oracle_all(sd, q, k, v, b, a_raw, mamba, M0=None, heads=None):
    B, N, H, _ = q.shape
    outs, states = np.zeros((B, N, H, D)), np.zeros((B, H, D, D))
    for bi in range(B):
        for h in (range(H) if heads is None else heads):
            s = dict(sd)
            if mamba:
                s["mamba2_a_raw"] = float(a_raw[h])
            o, M, _ = oracle.lsm_chunked(s, q[bi, :, h].float().cpu().numpy(), k[bi, :, h].float().cpu().numpy(),
                                         v[bi, :, h].float().cpu().numpy(),
                                         b_pre=b[bi, :, h].cpu().numpy() if mamba else None, chunk=64,
                                         M0=None if M0 is None else M0[bi, h].cpu().numpy())
            outs[bi, :, h], states[bi, h] = o, M
    return outs, states


@pytest.mark.parametrize("inst", ["bla_plain", "bla_elu", "rebased_plain", "lightning", "retnet", "mamba2"])
@pytest.mark.parametrize("N", [1, 129, 1000, 5000])
def test_fused_vs_oracle(inst, N):
    torch = _torch()
    import paper_2503_05447_b200 as pk
    spec, sd = _spec(pk, inst)
    B, H = 2, 2
    plan = pk.lsm.forward_plan(spec, B, N, H, D)
    assert plan["fused"], plan
    mamba = inst == "mamba2"
    q, k, v, b = _inputs(torch, B, N, H, seed=N, scale=0.3 if inst == "rebased_plain" else 0.5, long_memory=mamba)
    a_raw = np.array([0.3, -0.4])
    if mamba:
        spec.mamba2_a_raw = torch.tensor(a_raw, device="cuda", dtype=torch.float32)
    gates = pk.LsmGates(b_pre=b) if mamba else None
    fs = pk.MemoryState()
    o = pk.lsm_forward_batched(q, k, v, gates, spec, 64, final_state=fs)
    torch.cuda.synchronize()
    want, Mw = _oracle_all(sd, q, k, v, b, a_raw, mamba)
    got = o.float().cpu().numpy()
    for bi in range(B):
        for h in range(H):
            err = norm_rel_err(got[bi, :, h], want[bi, :, h])
            record_parity("fused_%s_N%d_b%d_h%d" % (inst, N, bi, h), err, TOL)
            assert err < TOL, (inst, N, bi, h, err)
            errM = norm_rel_err(fs.M[bi, h].cpu().numpy(), Mw[bi, h])
            assert errM < TOL, ("final state", inst, N, bi, h, errM)


@pytest.mark.parametrize("inst", ["retnet", "mamba2"])
def test_fused_initial_state_and_segments(inst):
    """A carried-in M0 and a sequence long enough for several segments per CTA (N = 40000,
    H = 16: 9 CTAs per head) against the oracle from the same M0 (heads 0, 1 and 15)."""
    torch = _torch()
    import paper_2503_05447_b200 as pk
    spec, sd = _spec(pk, inst)
    B, N, H = 1, 40000, 16
    plan = pk.lsm.forward_plan(spec, B, N, H, D)
    assert plan["fused"] and plan["ctas_per_head"] >= 2 and plan["segments"] > plan["ctas_per_head"], plan
    mamba = inst == "mamba2"
    q, k, v, b = _inputs(torch, B, N, H, seed=3, long_memory=True)
    a_raw = np.linspace(-0.6, 0.4, H)
    if mamba:
        spec.mamba2_a_raw = torch.tensor(a_raw, device="cuda", dtype=torch.float32)
    gates = pk.LsmGates(b_pre=b) if mamba else None
    M0 = torch.randn(B, H, D, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(8))
    heads = (0, 1, H - 1)
    fs = pk.MemoryState()
    o = pk.lsm_forward_batched(q, k, v, gates, spec, 64, initial_state=pk.MemoryState(M=M0), final_state=fs)
    torch.cuda.synchronize()
    want, Mw = _oracle_all(sd, q, k, v, b, a_raw, mamba, M0=M0, heads=heads)
    for h in heads:
        err = norm_rel_err(o[0, :, h].float().cpu().numpy(), want[0, :, h])
        record_parity("fused_%s_N40000_M0_h%d" % (inst, h), err, TOL)
        assert err < TOL, (h, err)
        assert norm_rel_err(fs.M[0, h].cpu().numpy(), Mw[0, h]) < TOL


@pytest.mark.parametrize("N,H", [(262144, 16), (32768, 16), (65536, 8), (3000, 64)])
def test_fused_equals_three_pass(N, H):
    """The single-read kernel and the three-pass path (LMOE_FUSED=0) agree on the same inputs
    (different segmentations: agreement to bf16 rounding of the state operand)."""
    torch = _torch()
    import paper_2503_05447_b200 as pk
    spec = pk.LsmSpec.make("mamba2", D)
    spec.mamba2_a_raw = torch.linspace(-1, 1, H, device="cuda")
    q, k, v, b = _inputs(torch, 1, N, H, seed=N + H)
    gates = pk.LsmGates(b_pre=b)
    fs1, fs3 = pk.MemoryState(), pk.MemoryState()
    o1 = pk.lsm_forward_batched(q, k, v, gates, spec, 64, final_state=fs1)
    os.environ["LMOE_FUSED"] = "0"
    try:
        assert not pk.lsm.forward_plan(spec, 1, N, H, D)["fused"]
        o3 = pk.lsm_forward_batched(q, k, v, gates, spec, 64, final_state=fs3)
    finally:
        os.environ["LMOE_FUSED"] = "1"
    torch.cuda.synchronize()
    scale = o3.float().abs().amax(dim=(1, 3))
    err = ((o1.float() - o3.float()).abs().amax(dim=(1, 3)) / scale).max().item()
    record_parity("fused_vs_three_pass_N%d_H%d" % (N, H), err, 1e-2)
    assert err < 1e-2
    errM = ((fs1.M - fs3.M).abs().amax(dim=(2, 3)) / fs3.M.abs().amax(dim=(2, 3))).max().item()
    assert errM < 1e-2


def test_fused_is_deterministic_and_graph_capturable():
    torch = _torch()
    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200 import sp
    N, H = 70000, 16
    spec = pk.LsmSpec.make("mamba2", D)
    spec.mamba2_a_raw = torch.linspace(-1, 1, H, device="cuda")
    q, k, v, b = _inputs(torch, 1, N, H, seed=5)
    gates = pk.LsmGates(b_pre=b)
    comm = sp.NcclComm(0, 1)
    out = torch.empty_like(q)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, stream=st.cuda_stream)
        ref = out.clone()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
        out.zero_()
        for _ in range(3):
            gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
