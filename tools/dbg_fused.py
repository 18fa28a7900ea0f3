"""Localise a fused-forward mismatch: per-chunk error of the single-read kernel and of the
three-pass path against the f64 oracle (Mamba2, long-memory gates, carried-in M0)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import oracle
import paper_2503_05447_b200 as pk

D = 128
B, N, H = 1, int(sys.argv[1]) if len(sys.argv) > 1 else 40000, int(sys.argv[2]) if len(sys.argv) > 2 else 16
use_m0 = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn(B, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
b = torch.randn(B, N, H, device="cuda", generator=g).mul_(0.5).sub_(3.0)
a_raw = np.linspace(-0.6, 0.4, H)
spec = pk.LsmSpec.make("mamba2", D)
spec.mamba2_a_raw = torch.tensor(a_raw, device="cuda", dtype=torch.float32)
gates = pk.LsmGates(b_pre=b)
M0 = torch.randn(B, H, D, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(8)) if use_m0 else None
print("plan", pk.lsm.forward_plan(spec, B, N, H, D))
outs = {}
for fused in ("1", "0"):
    os.environ["LMOE_FUSED"] = fused
    fs = pk.MemoryState() if os.environ.get("DBG_FS") else None
    outs[fused] = pk.lsm_forward_batched(q, k, v, gates, spec, 64, final_state=fs,
                                         initial_state=pk.MemoryState(M=M0) if use_m0 else None).float().cpu().numpy()
torch.cuda.synchronize()
for h in (0, 1, H - 1):
    sd = oracle.spec_default("mamba2")
    sd["mamba2_a_raw"] = float(a_raw[h])
    want, _, _ = oracle.lsm_chunked(sd, q[0, :, h].float().cpu().numpy(), k[0, :, h].float().cpu().numpy(),
                                    v[0, :, h].float().cpu().numpy(), b_pre=b[0, :, h].cpu().numpy(), chunk=64,
                                    M0=M0[0, h].cpu().numpy() if use_m0 else None)
    sc = np.abs(want).max()
    for name, o in outs.items():
        e = np.abs(o[0, :, h] - want).max(axis=1) / sc
        per = [e[i:i + 128].max() for i in range(0, N, 128)]
        bad = [i for i, x in enumerate(per) if x > 2e-2]
        print("h%d fused=%s err %.3e  bad chunks (%d): %s" % (h, name, e.max(), len(bad), bad[:20]))
