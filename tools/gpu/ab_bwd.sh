#!/bin/bash
export PYTHONPATH=.
cat > /tmp/bwdt.py <<'PY'
import torch, paper_2503_05447_b200 as pk
N, H, D = 262144, 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, dO = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(4))
gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g))
spec = pk.LsmSpec.make("mamba2", D); spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=g).mul_(0.5)
for _ in range(2): pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5): pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
e.record(); torch.cuda.synchronize(); print("mamba2 bwd %.3f ms" % (s.elapsed_time(e) / 5))
PY
for rep in 1 2; do for v in A B; do echo "$v $(LMOE_LIB=ab/lib$v.so timeout 120 python /tmp/bwdt.py 2>&1 | tail -1)"; done; done
