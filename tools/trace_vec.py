"""Per-chunk phase timeline (clock64) of CTA (0,0,0) of lsm_output_pass_vec (LMOE_TRACE=1)."""
import ctypes, os, sys
os.environ["LMOE_TRACE"] = "1"
import numpy as np, torch
import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib
N, H, D = 262144, 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16) for _ in range(3))
a = torch.randn(1, N, H, D, device="cuda", generator=g).add_(3.0).bfloat16()
spec = pk.LsmSpec.make(sys.argv[1] if len(sys.argv) > 1 else "gla", D)
for _ in range(3):
    pk.lsm_forward_batched(q, k, v, pk.LsmGates(a_pre=a), spec, 64, check=False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 16 + 4 * 4096))()
_lib.check(_lib.lib().lmoe_debug_trace_read(buf))
t = np.array(buf, dtype=np.int64)[:64 * 16].reshape(64, 16)
t0 = t[0, 10]
names = ["full", "scan", "xform", "stateop", "s_full", "P", "mo_full", "O", "end"]
print("chunk  tma " + " ".join("%7s" % n for n in names))
for c in range(0, 24):
    row = t[c]
    if row[0] == 0:
        break
    print("%5d %5d " % (c, row[10] - t0) + " ".join("%7d" % (row[i] - t0) for i in range(9)))
print("steady cycles/chunk: %.0f" % np.diff(t[4:20, 8]).mean())
