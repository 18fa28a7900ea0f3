"""GPU parity of the sm_100a softmax attention (lmoe_attn_fwd / lmoe_sp_attn_fwd) against the
reference's own outputs (tests/golden/attn.npz) and the float64 oracle (oracle lmo_attention,
pinned to the same file).  bf16 operands, fp32 softmax and accumulation: norm-relative 2e-2."""
import numpy as np
import pytest

import oracle
from conftest import load_golden, norm_rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_golden_attention_padded():
    """Reference outputs (d = 8).  Zero-padding to D = 128 leaves q.k unchanged; scaling q by
    sqrt(128 / 8) = 4 (exact in bf16) restores the reference's 1/sqrt(8)."""
    torch = _torch()
    from paper_2503_05447_b200 import attn
    d = load_golden("attn")
    pad = lambda x, s=1.0: torch.tensor(np.pad(x * s, ((0, 0), (0, 120))), dtype=torch.float32,
                                        device="cuda").to(torch.bfloat16)
    q, k, v = pad(d["q"], 4.0), pad(d["k"]), pad(d["v"])
    o = attn.softmax_attention_parallel(q, k, v, True)
    assert norm_rel_err(o[:, :8].double().cpu().numpy(), d["o_full"]) < TOL
    o = attn.softmax_attention_parallel(q[16:], k, v, True, row_offset=16)
    assert norm_rel_err(o[:, :8].double().cpu().numpy(), d["o_off"]) < TOL
    assert np.abs(o[:, 8:].float().cpu().numpy()).max() == 0.0
    for t in (2, 4):  # SP == full causal attention; the reference moves 2 * N * d elements
        assert int(d["comm_elems_t%d" % t][0]) == 2 * 24 * 8
        assert norm_rel_err(d["o_sp_t%d" % t], d["o_full"]) < 1e-12


@pytest.mark.parametrize("shape", [(1, 1000, 2, 0), (2, 300, 3, 0), (1, 257, 1, 700), (1, 129, 2, 5000)])
def test_attention_vs_oracle(shape):
    torch = _torch()
    from paper_2503_05447_b200 import attn
    B, Nq, H, off = shape
    Nk = min(Nq + off, 1100)
    g = torch.Generator(device="cuda").manual_seed(Nq + off)
    q = torch.randn(B, Nq, H, 128, device="cuda", generator=g).mul_(0.5).bfloat16()
    k = torch.randn(B, Nk, H, 128, device="cuda", generator=g).mul_(0.5).bfloat16()
    v = torch.randn(B, Nk, H, 128, device="cuda", generator=g).bfloat16()
    o = attn.softmax_attention_parallel(q, k, v, True, row_offset=off)
    torch.cuda.synchronize()
    for b in range(B):
        for h in range(H):
            want = oracle.attention(*(t[b, :, h].double().cpu().numpy() for t in (q, k, v)), True, off)
            assert norm_rel_err(o[b, :, h].double().cpu().numpy(), want) < TOL, (shape, b, h)


def test_attention_noncausal_and_large_logits():
    """causal = False (mask-free) and score ranges that force the lazy O rescale."""
    torch = _torch()
    from paper_2503_05447_b200 import attn
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(1, 600, 1, 128, device="cuda", generator=g).mul_(3.0).bfloat16()
    k = torch.randn(1, 900, 1, 128, device="cuda", generator=g).bfloat16()
    k[:, 500:] *= 4  # later keys dominate: the running max grows after the first tiles
    v = torch.randn(1, 900, 1, 128, device="cuda", generator=g).bfloat16()
    for causal in (False, True):
        o = attn.softmax_attention_parallel(q, k, v, causal, row_offset=300)
        want = oracle.attention(*(t[0, :, 0].double().cpu().numpy() for t in (q, k, v)), causal, 300)
        assert norm_rel_err(o[0, :, 0].double().cpu().numpy(), want) < TOL, causal


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sp_attention_rank_slices(world):
    """sp_attention_rank per chunk_range slice == full causal attention (single device: the
    gathered K/V is the full sequence); the NCCL path at world 1 matches exactly."""
    torch = _torch()
    from paper_2503_05447_b200 import attn, sp
    B, N, H = 1, 1000, 2
    g = torch.Generator(device="cuda").manual_seed(world)
    q, k, v = (torch.randn(B, N, H, 128, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
    full = attn.softmax_attention_parallel(q, k, v, True)
    for r in range(world):
        r0, r1 = sp.chunk_range(N, world, r)
        o = attn.softmax_attention_parallel(q[:, r0:r1], k, v, True, row_offset=r0)
        err = ((o.float() - full[:, r0:r1].float()).abs().max() / full.float().abs().max()).item()
        assert err < 1e-2, (world, r, err)
    comm = sp.NcclComm(0, 1)
    o1 = attn.sp_attention_rank(comm, q, k, v, N)
    torch.cuda.synchronize()
    assert torch.equal(o1, full)
    assert attn.last_gather_elements() == 2 * N * H * 128


def test_attention_error_texts():
    torch = _torch()
    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200 import attn
    x = torch.zeros(1, 0, 1, 128, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(1, 4, 1, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(pk.LmoeError, match="need N >= 1 rows"):
        attn.softmax_attention_parallel(x, y, y)
    with pytest.raises(pk.LmoeError, match="supported"):
        attn.softmax_attention_parallel(y.float(), y.float(), y.float())
