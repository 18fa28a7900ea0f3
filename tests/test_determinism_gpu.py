"""Race detection by repetition: the warp-specialised kernels hand tiles between warps through
mbarriers, and a protocol error there (an arrival counted toward the wrong phase) shows up as
an occasional wrong tile, not as a crash.  Each path below runs the same inputs many times and
must give bit-identical results every time -- the state pass (the race fixed in
lsm_kernels.cuh / lsm_fused.cuh was caught this way), the output pass, the TokenVector passes,
the backward passes and the MoE layer."""
import pytest

pytestmark = pytest.mark.gpu
D = 128


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _repeat_equal(torch, fn, reps):
    first = [t.clone() for t in fn()]
    for r in range(reps - 1):
        got = fn()
        for i, (a, b) in enumerate(zip(first, got)):
            assert torch.equal(a, b), ("run %d differs from run 0 in output %d" % (r + 1, i))


@pytest.mark.parametrize("inst", ["mamba2", "retnet", "bla_elu"])
def test_forward_bitwise_repeatable(inst):
    torch = _torch()
    import paper_2503_05447_b200 as pk
    N, H = 65536, 16
    g = torch.Generator(device="cuda").manual_seed(31)
    q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
    if inst == "bla_elu":
        spec = pk.LsmSpec(instance=pk.LsmInstance.BLA, feature_map=1, use_normalizer=True)
    else:
        spec = pk.LsmSpec.make(inst, D)
    gates = None
    if inst == "mamba2":
        spec.mamba2_a_raw = torch.linspace(-1, 1, H, device="cuda")
        gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g))

    def run():
        fs = pk.MemoryState()
        o = pk.lsm_forward_batched(q, k, v, gates, spec, 64, final_state=fs, check=False)
        return [o, fs.M]
    _repeat_equal(torch, run, 12)


def test_gla_forward_backward_bitwise_repeatable():
    torch = _torch()
    import paper_2503_05447_b200 as pk
    N, H = 32768, 16
    g = torch.Generator(device="cuda").manual_seed(32)
    q, k, v, dO, a = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(5))
    spec = pk.LsmSpec.make("gla", D)
    gates = pk.LsmGates(a_pre=a)

    def run():
        o = pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)
        gr = pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
        return [o, gr.dq, gr.dk, gr.dv, gr.da_pre]
    _repeat_equal(torch, run, 6)


def test_mamba2_backward_bitwise_repeatable():
    torch = _torch()
    import paper_2503_05447_b200 as pk
    N, H = 32768, 16
    g = torch.Generator(device="cuda").manual_seed(33)
    q, k, v, dO = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(4))
    spec = pk.LsmSpec.make("mamba2", D)
    spec.mamba2_a_raw = torch.linspace(-1, 1, H, device="cuda")
    gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g))

    def run():
        gr = pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
        return [gr.dq, gr.dk, gr.dv, gr.db_pre]
    _repeat_equal(torch, run, 6)


def test_moe_forward_bitwise_repeatable():
    torch = _torch()
    from paper_2503_05447_b200 import moe
    T, hidden, ffn, E, k = 8192, 1024, 896, 64, 8
    g = torch.Generator(device="cuda").manual_seed(34)
    x = torch.randn(T, hidden, device="cuda", generator=g).bfloat16()
    layer = moe.MoeLayer.init(moe.MoeConfig(num_experts=E, top_k=k, hidden=hidden, ffn_dim=ffn), generator=g)

    def run():
        y, aux = layer.forward(x)
        return [y, aux.reshape(1)]
    _repeat_equal(torch, run, 8)
