"""Local-state forward (lsm_host.cu LsmCall::local_pass, lsm_kernels.cuh lsm_local_fix): for the
decaying scalar kinds the output pass runs every segment from a zero state, the segment combine
produces the entering states, and the first chunks of each segment get (q e^{Gseg}) M_in added
until the decay from the segment start leaves the fp32 range -- no state pass.  It must equal
the segment-parallel three-pass path (LMOE_LOCAL=0) and the float64 oracle (lsm_forward_chunked,
lsm.hpp:668-708), final state and carried-in initial state included, for strong, default and
long-memory decays (the last makes the correction span whole segments).  The TokenVector kinds
(GLA, HGRN2, RWKV6) take the same structure with per-column decay (lsm_local_fix_vec,
lsm_vec_kernels.cuh), checked the same way with gates from strong to slow decay."""
import numpy as np
import pytest

import oracle
from conftest import norm_rel_err, record_parity

pytestmark = pytest.mark.gpu
D = 128


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _case(torch, inst, N, H, gate_mean, a_raw, seed):
    import paper_2503_05447_b200 as pk
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16) for _ in range(3))
    spec = pk.LsmSpec.make(inst, D)
    gates = None
    if inst == "mamba2":
        spec.mamba2_a_raw = torch.full((H,), float(a_raw), device="cuda")
        gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g).mul_(0.5).add_(gate_mean))
    elif inst in ("gla", "hgrn2", "rwkv6"):
        a = torch.randn(1, N, H, D, device="cuda", generator=g).mul_(a_raw).add_(gate_mean)
        gates = pk.LsmGates(a_pre=a.to(torch.bfloat16))
    M0 = torch.randn(1, H, D, D, device="cuda", generator=g).mul_(0.05)
    return pk, q, k, v, spec, gates, M0


@pytest.mark.parametrize("inst,N,H,gate_mean,a_raw", [
    ("mamba2", 20000, 2, 0.0, 0.3),      # default-like decay, 74 short segments
    ("mamba2", 9000, 2, -3.0, -1.0),     # long memory: corrections span whole segments
    ("mamba2", 5000, 2, 2.0, 2.0),       # strong decay
    ("mamba2", 60000, 16, 0.0, 0.3),     # 9 long segments per head (the cfg3 layout)
    ("lightning", 120000, 16, 0.0, 0.0),  # constant decay, segments longer than the corrected span
    # TokenVector: (gate mean, gate std) -- a ~ N(0, 1) as the bench, slow columns, long memory
    ("gla", 60000, 16, 0.0, 1.0),
    ("gla", 20000, 2, 2.0, 0.5),          # sigma ~ 0.88: ~6 corrected chunks
    ("gla", 9000, 2, 5.0, 0.3),           # sigma ~ 0.993: corrections span whole segments
    ("hgrn2", 20000, 2, 1.0, 1.0),
    ("rwkv6", 20000, 2, 0.0, 1.0),
])
def test_local_equals_three_pass_and_oracle(monkeypatch, inst, N, H, gate_mean, a_raw):
    torch = _torch()
    pk, q, k, v, spec, gates, M0 = _case(torch, inst, N, H, gate_mean, a_raw, seed=N)
    plan = pk.lsm.forward_plan(spec, 1, N, H, D)
    assert plan["local"] and plan["segments"] > 1, plan
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("LMOE_LOCAL", mode)
        fs = pk.MemoryState()
        o = pk.lsm_forward_batched(q, k, v, gates, spec, 64, initial_state=pk.MemoryState(M=M0), final_state=fs)
        torch.cuda.synchronize()
        outs[mode] = (o.float(), fs.M.clone())
    (o1, m1), (o0, m0) = outs["1"], outs["0"]
    e = ((o1 - o0).abs().max() / o0.abs().max()).item()
    em = ((m1 - m0).abs().max() / m0.abs().max()).item()
    record_parity("local_vs_3pass/%s/%d" % (inst, N), e, 1e-2)
    assert e < 1e-2 and em < 1e-2, (e, em)
    for h in sorted({0, H - 1}):
        sd = oracle.spec_default(inst)
        b = a = None
        if inst == "mamba2":
            sd["mamba2_a_raw"] = float(a_raw)
            b = gates.b_pre[0, :, h].cpu().numpy()
        if gates is not None and gates.a_pre is not None:
            a = gates.a_pre[0, :, h].float().cpu().numpy()
        want, wM, _ = oracle.lsm_chunked(sd, *(t[0, :, h].float().cpu().numpy() for t in (q, k, v)), a_pre=a,
                                         b_pre=b, M0=M0[0, h].double().cpu().numpy())
        err = norm_rel_err(o1[0, :, h].cpu().numpy(), want)
        errM = norm_rel_err(m1[0, h].cpu().numpy(), wM)
        record_parity("local_vs_oracle/%s/%d/h%d" % (inst, N, h), err, 2e-2)
        assert err < 2e-2 and errM < 2e-2, (inst, h, err, errM)


def test_local_plan_selection():
    """Decaying scalar and vector kinds take the local path; undecayed, normalised and short
    constant-decay shapes (where the corrected span would cost more than the state pass) do not."""
    _torch()
    import paper_2503_05447_b200 as pk
    mk = pk.LsmSpec.make
    assert pk.lsm.forward_plan(mk("mamba2", D), 1, 262144, 16, D)["local"]
    assert pk.lsm.forward_plan(mk("retnet", D), 1, 262144, 16, D)["local"]
    assert not pk.lsm.forward_plan(mk("retnet", D), 1, 32768, 16, D)["local"]
    assert not pk.lsm.forward_plan(pk.LsmSpec(instance=0, feature_map=0), 1, 262144, 16, D)["local"]
    assert pk.lsm.forward_plan(mk("gla", D), 1, 262144, 16, D)["local"]
    assert pk.lsm.forward_plan(mk("hgrn2", D), 1, 262144, 16, D)["local"]
    assert not pk.lsm.forward_plan(mk("bla", D), 1, 262144, 16, D)["local"]
