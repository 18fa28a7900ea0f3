"""One cfg3 Mamba2 SP forward step at a given slice (default 32768: the T = 8 per-rank work),
world 1, for ncu launch lists."""
import sys

import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import sp

H, D = 16, 128
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
inst = sys.argv[2] if len(sys.argv) > 2 else "mamba2"
comm = sp.NcclComm(0, 1)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, n, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
spec = pk.LsmSpec.make(inst, D)
if inst == "mamba2":
    spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=g).mul_(0.5)
    gates = pk.LsmGates(b_pre=torch.randn(1, n, H, device="cuda", generator=g))
else:
    gates = pk.LsmGates(a_pre=torch.randn(1, n, H, D, device="cuda", generator=g).bfloat16())
out = torch.empty_like(q)
for _ in range(2):
    sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False)
torch.cuda.synchronize()
