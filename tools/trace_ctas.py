"""Per-CTA start / end (globaltimer) of the scalar output pass (LMOE_TRACE=1), cfg3 Mamba2."""
import ctypes, os, sys
os.environ["LMOE_TRACE"] = "1"
import numpy as np, torch
import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib
N, H, D = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16) for _ in range(3))
spec = pk.LsmSpec.make("mamba2", D)
spec.mamba2_a_raw = torch.full((H,), 0.3, device="cuda")
gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g))
for _ in range(3):
    pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 16 + 4 * 4096))()
_lib.check(_lib.lib().lmoe_debug_trace_read(buf))
t = np.array(buf, dtype=np.int64)[64 * 16:64 * 16 + 4096].reshape(-1, 2)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
print("CTAs %d  start: min %.1f max %.1f us | end: min %.1f median %.1f max %.1f us | busy median %.1f us"
      % (len(t), s.min(), s.max(), e.min(), np.median(e), e.max(), np.median(e - s)))
