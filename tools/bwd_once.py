"""One cfg3 Mamba2 LSM backward (for ncu launch lists)."""
import torch
import paper_2503_05447_b200 as pk
N, H, D = 262144, 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, dO = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(4))
gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g))
spec = pk.LsmSpec.make("mamba2", D)
spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=g).mul_(0.5)
for _ in range(2):
    pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
torch.cuda.synchronize()
