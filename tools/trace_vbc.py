"""Phase timeline (globaltimer ns) of one lsm_vec_bwd_chunk CTA (LMOE_TRACE=1)."""
import ctypes
import os
import sys

os.environ["LMOE_TRACE"] = "1"
import numpy as np
import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
H, D = 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, dO = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(4))
a = torch.randn(1, N, H, D, device="cuda", generator=g).add_(3.0).bfloat16()
spec = pk.LsmSpec.make("gla", D)
for _ in range(3):
    pk.lsm_backward_batched(q, k, v, pk.LsmGates(a_pre=a), spec, dO, check=False)
torch.cuda.synchronize()
buf = np.zeros(64 * 16 + 4 * 4096, dtype=np.uint64)
_lib.lib().lmoe_debug_trace_read(ctypes.c_void_p(buf.ctypes.data))
t = buf[:64 * 16].reshape(64, 16)[:3].astype(np.int64)
t0 = t[0, 0]
names = {0: ["start", "scan_done", "q_free"],
         1: ["full", "mx_full", "xf", "p_full", "dq_free"],
         2: ["full", "scan", "transform", "mx_full", "s_full", "E1 done", "dq/dk full", "E2 done", "dv_full",
             "E3 done", "a_full", "S done"]}
for role, nm in names.items():
    print(["TMA", "MMA", "math"][role], "  ".join("%s=%.2fus" % (n, (t[role, i] - t0) / 1e3) for i, n in enumerate(nm)))
