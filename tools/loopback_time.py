"""Device time of the cfg3 Mamba2 SP forward over `world` virtual ranks on one GPU
(lmoe_sp_lsm_fwd_loopback: phase A of every rank, then phase B of every rank), for A/B of the
rank-combine path (ranks 1..world-2 take the folded path when no final state is requested)."""
import sys

import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import sp

H, D, N = 16, 128, 262144
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
spec = pk.LsmSpec.make("mamba2", D)
spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)).mul_(0.5)
gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g))
for _ in range(2):
    sp.sp_forward_masked_loopback(q, k, v, gates, spec, world, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sp.sp_forward_masked_loopback(q, k, v, gates, spec, world, check=False)
e1.record()
torch.cuda.synchronize()
print("loopback world %d: %.3f ms per call" % (world, e0.elapsed_time(e1) / 10))
