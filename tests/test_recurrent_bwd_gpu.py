"""Backward of the recurrent kinds on the device (lmoe_lsm_bwd_recurrent): DeltaNet,
GatedDeltaNet, GFW, GateLoop, TTT, Titans, RWKV7, S4, Mamba -- the reference's tape over
recurrent_step (lsm.hpp:335-441, tensor.hpp:1178-1215).

  * against the reference tape's own gradients (tests/golden/lsm_rec_grad.npz, d = 4 zero-padded
    to the kernel width: exact for every kind here), fp32 (D = 64, 1e-3) and bf16 (D = 128, 2e-2);
  * at sizes the tape cannot reach (several 32-token checkpoint blocks, batch, heads, an initial
    state and a final-state gradient) against central differences of the f64 oracle recurrence
    along random directions (the oracle is pinned to the tape the same way,
    tests/test_oracle_golden.py::test_recurrent_kinds_tape_gradients_pin_the_oracle)."""
import numpy as np
import pytest

import oracle
from conftest import load_golden, norm_rel_err, record_parity

pytestmark = pytest.mark.gpu

REC = ("a_pre", "b_pre", "alpha_pre", "beta_pre", "s4_delta_raw", "s4_b", "s4_A_raw", "mamba_A_raw")
GATES = ("a_pre", "b_pre", "alpha_pre", "beta_pre")
STATIC = ("s4_delta_raw", "s4_b", "s4_A_raw", "mamba_A_raw")


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _golden_inputs(torch, d, p, D, dt):
    """Golden case p zero-padded to D on the device ([1, n, 1, D] layouts, static [1, D(, D)])."""
    import paper_2503_05447_b200 as pk
    dd = d[p + "/q"].shape[1]
    T = lambda x, t=dt: torch.tensor(x, dtype=torch.float32, device="cuda").to(t)
    padc = lambda x: np.pad(x, ((0, 0), (0, D - x.shape[1])))
    q, k, v, dO = (T(padc(d[p + "/" + n]))[None, :, None] for n in ("q", "k", "v", "dO"))
    g = pk.LsmGates()
    for n in GATES:
        if p + "/" + n in d:
            a = d[p + "/" + n]
            setattr(g, n, T(padc(a))[None, :, None] if a.ndim == 2 else T(a, torch.float32)[None, :, None])
    spec = pk.LsmSpec(instance=int(d[p + "/instance"][0]), feature_map=int(d[p + "/feature_map"][0]))
    for n in STATIC:
        if p + "/" + n in d:
            a = d[p + "/" + n]
            a = np.pad(a, (0, D - dd)) if a.ndim == 1 else np.pad(a, ((0, D - dd), (0, D - dd)))
            setattr(spec, n, T(a, torch.float32)[None])
    return q, k, v, dO, g, spec, dd


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_recurrent_backward_matches_reference_tape(dtype):
    torch = _torch()
    from paper_2503_05447_b200.lsm import lsm_backward_recurrent
    d = load_golden("lsm_rec_grad")
    D = 64 if dtype == "f32" else 128
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    tol = 1e-3 if dtype == "f32" else 2e-2
    cases = sorted({k.split("/")[0] for k in d})
    assert len(cases) == 9
    for p in cases:
        q, k, v, dO, g, spec, dd = _golden_inputs(torch, d, p, D, dt)
        gr = lsm_backward_recurrent(q, k, v, g, spec, dO)
        torch.cuda.synchronize()
        got = {"q": gr.dq[0, :, 0, :dd], "k": gr.dk[0, :, 0, :dd], "v": gr.dv[0, :, 0, :dd]}
        for n in GATES:
            t = getattr(gr, "d" + n)
            if t is not None:
                got[n] = t[0, :, 0, :dd] if t.dim() == 4 else t[0, :, 0]
        for n in STATIC:
            t = getattr(gr, "d" + n)
            if t is not None:
                got[n] = t[0, :dd] if t.dim() == 2 else t[0, :dd, :dd]
        for n, t in got.items():
            want = d[p + "/d" + n]
            if np.abs(want).max() == 0:  # e.g. S4 ignores k: the tape's gradient is zero
                assert float(t.abs().max()) == 0.0, (p, n)
                continue
            err = norm_rel_err(t.float().cpu().numpy(), want)
            record_parity("rec_bwd_tape/%s/%s/%s" % (dtype, p, n), err, tol)
            assert err < tol, (p, n, dtype, err)


def _fd_case(torch, inst, B, N, H, D, dt, seed):
    """Random inputs for one kind at [B, N, H, D] (bf16-exact when dt is bf16) plus M0 and dM_final."""
    import paper_2503_05447_b200 as pk
    rng = np.random.default_rng(seed)
    rnd = lambda *s, m=0.0, sd=0.5: rng.normal(m, sd, s)
    R = lambda x, t=dt: torch.tensor(x, dtype=torch.float32, device="cuda").to(t)
    q, k, v, dO = R(rnd(B, N, H, D)), R(rnd(B, N, H, D)), R(rnd(B, N, H, D)), R(rnd(B, N, H, D, sd=1.0))
    spec = pk.LsmSpec.make(inst, D)
    g = pk.LsmGates()
    if inst in ("deltanet", "gated_deltanet", "titans"):
        g.a_pre = R(rnd(B, N, H, m=2.0, sd=1.0), torch.float32)
        g.b_pre = R(rnd(B, N, H, sd=1.0), torch.float32)
    if inst == "ttt":
        g.b_pre = R(rnd(B, N, H, m=-2.0, sd=1.0), torch.float32)
    if inst == "rwkv7":
        g.a_pre = R(rnd(B, N, H, D, m=2.0, sd=1.0))
        g.b_pre = R(rnd(B, N, H, m=-2.0, sd=1.0), torch.float32)
    if inst in ("gfw", "gateloop"):
        g.alpha_pre, g.beta_pre = R(rnd(B, N, H, D, m=2.0, sd=1.0)), R(rnd(B, N, H, D, m=2.0, sd=1.0))
    if inst == "s4":
        spec.s4_delta_raw = R(rnd(H, D), torch.float32)
        spec.s4_b = R(rnd(H, D), torch.float32)
        spec.s4_A_raw = R(rnd(H, D, D), torch.float32)
    if inst == "mamba":
        g.a_pre = R(rnd(B, N, H, D, m=-1.0, sd=0.5))
        spec.mamba_A_raw = R(rnd(H, D, D), torch.float32)
    M0 = R(rnd(B, H, D, D, sd=0.1), torch.float32)
    dMf = R(rnd(B, H, D, D, sd=0.1), torch.float32)
    return q, k, v, dO, g, spec, M0, dMf, rng


def _oracle_args(torch, q, k, v, g, spec, b, h):
    c = lambda t: t.float().cpu().numpy().astype(np.float64)
    x = {"q": c(q[b, :, h]), "k": c(k[b, :, h]), "v": c(v[b, :, h])}
    for n in GATES:
        t = getattr(g, n)
        if t is not None:
            x[n] = c(t[b, :, h])
    for n in STATIC:
        t = getattr(spec, n)
        if t is not None:
            x[n] = c(t[h])
    return x


@pytest.mark.parametrize("dtype,D", [("f32", 64), ("bf16", 128)])
@pytest.mark.parametrize("inst", ["deltanet", "gated_deltanet", "gfw", "ttt", "titans", "rwkv7", "s4", "mamba"])
def test_recurrent_backward_directional_fd(inst, dtype, D):
    """Multi-block sequence (N = 100: checkpoints at 0/32/64/96), B = 2, H = 2, M0 and dM_final:
    <device gradient, u> against the f64 central difference of
    L = sum(o * dO) + sum(M_N * dM_final) along random directions u of every input."""
    torch = _torch()
    from paper_2503_05447_b200.lsm import lsm_backward_recurrent
    import paper_2503_05447_b200 as pk
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    B, N, H = 2, 100, 2
    q, k, v, dO, g, spec, M0, dMf, rng = _fd_case(torch, inst, B, N, H, D, dt, seed=sum(map(ord, inst)))
    gr = lsm_backward_recurrent(q, k, v, g, spec, dO, initial_state=pk.MemoryState(M=M0), dM_final=dMf)
    torch.cuda.synchronize()
    sd = oracle.spec_default(inst)
    tol = 2e-3 if dtype == "f32" else 2e-2
    for b in range(B):
        for h in range(H):
            x = _oracle_args(torch, q, k, v, g, spec, b, h)
            x["M0"] = M0[b, h].cpu().numpy().astype(np.float64)
            w = dO[b, :, h].float().cpu().numpy().astype(np.float64)
            Mw = dMf[b, h].cpu().numpy().astype(np.float64)

            def loss(xx):
                o, M = oracle.lsm_recurrent(sd, xx["q"], xx["k"], xx["v"], *(xx.get(n) for n in REC), M0=xx["M0"])
                return float((o * w).sum() + (M * Mw).sum())
            grads = {"q": gr.dq[b, :, h], "k": gr.dk[b, :, h], "v": gr.dv[b, :, h], "M0": gr.dM0[b, h]}
            for n in GATES:
                t = getattr(gr, "d" + n)
                if t is not None:
                    grads[n] = t[b, :, h]
            for name, gt in grads.items():
                u = rng.normal(0, 1, x[name].shape)
                eps = 1e-4
                xp, xm = dict(x), dict(x)
                xp[name], xm[name] = x[name] + eps * u, x[name] - eps * u
                fd = (loss(xp) - loss(xm)) / (2 * eps)
                gn = gt.float().cpu().numpy().astype(np.float64)
                an = float((gn * u).sum())
                # relative to the typical size of <g, u>, |g| |u| / sqrt(n) (a random direction
                # cancels most of the sum; elementwise relative error e of g then shows as ~e)
                scale = max(abs(fd), np.linalg.norm(gn) * np.linalg.norm(u) / np.sqrt(u.size), 1e-9)
                err = abs(an - fd) / scale
                record_parity("rec_bwd_fd/%s/%s/%s" % (dtype, inst, name), err, tol)
                assert err < tol, (inst, dtype, b, h, name, fd, an)
    # static parameters: the batch sum of the per-(b, h) FD derivatives
    for n in STATIC:
        t = getattr(gr, "d" + n)
        if t is None:
            continue
        for h in range(H):
            u = rng.normal(0, 1, tuple(getattr(spec, n)[h].shape))
            fd = 0.0
            for b in range(B):
                x = _oracle_args(torch, q, k, v, g, spec, b, h)
                x["M0"] = M0[b, h].cpu().numpy().astype(np.float64)
                w = dO[b, :, h].float().cpu().numpy().astype(np.float64)
                Mw = dMf[b, h].cpu().numpy().astype(np.float64)

                def loss(xx):
                    o, M = oracle.lsm_recurrent(sd, xx["q"], xx["k"], xx["v"], *(xx.get(m) for m in REC), M0=xx["M0"])
                    return float((o * w).sum() + (M * Mw).sum())
                eps = 1e-4
                xp, xm = dict(x), dict(x)
                xp[n], xm[n] = x[n] + eps * u, x[n] - eps * u
                fd += (loss(xp) - loss(xm)) / (2 * eps)
            an = float((t[h].cpu().numpy().astype(np.float64) * u).sum())
            err = abs(an - fd) / max(abs(fd), 1e-6)
            record_parity("rec_bwd_fd/%s/%s/%s" % (dtype, inst, n), err, tol)
            assert err < tol, (inst, dtype, n, h, fd, an)


def test_recurrent_backward_errors():
    torch = _torch()
    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200.lsm import lsm_backward_recurrent
    q = torch.zeros(1, 8, 1, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(pk.LmoeError, match="needs a_pre"):
        lsm_backward_recurrent(q, q, q, pk.LsmGates(), pk.LsmSpec.make("deltanet", 128), q)
    with pytest.raises(pk.LmoeError, match="chunk-parallel form"):
        lsm_backward_recurrent(q, q, q, pk.LsmGates(), pk.LsmSpec.make("retnet", 128), q)
