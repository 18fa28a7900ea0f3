"""Times the cfg3-shaped TokenVector (GLA) LSM backward and forward on the device
(CUDA events), and optionally runs once for an ncu capture (argv[1] == "once")."""
import sys

import torch

import paper_2503_05447_b200 as pk

N = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
H, D = 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, dO = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(4))
a = torch.randn(1, N, H, D, device="cuda", generator=g).add_(3.0).bfloat16()
gates = pk.LsmGates(a_pre=a)
spec = pk.LsmSpec.make(sys.argv[3] if len(sys.argv) > 3 else "gla", D)
once = len(sys.argv) > 1 and sys.argv[1] == "once"
for _ in range(1 if once else 2):
    pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
torch.cuda.synchronize()
if not once:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, fn in (("fwd", lambda: pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)),
                     ("bwd", lambda: pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False))):
        fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(5):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        print("%s %s N=%d H=%d: %.3f ms  %.1f Mtok/s" % (spec.instance, name, N, H, ms, N / ms / 1e3))
