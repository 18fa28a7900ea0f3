"""Segment timeline of the single-read forward (lsm_fused_fwd) for head 0 at the cfg3 shape
(LMOE_TRACE=1): per CTA and segment unit, globaltimer (us from the first event) of
A start, look-back start, window flags observed, entering state folded, C done.  Columns:
A (state steps), wait (publish + flag poll), chain (folding the window's aggregates), C."""
import ctypes
import os
import sys

os.environ["LMOE_TRACE"] = "1"
import numpy as np
import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib

H, D = 16, 128
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, n, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
spec = pk.LsmSpec.make("mamba2", D)
spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=g).mul_(0.5)
gates = pk.LsmGates(b_pre=torch.randn(1, n, H, device="cuda", generator=g))
plan = pk.lsm.forward_plan(spec, 1, n, H, D)
print("plan", plan)
for _ in range(3):
    pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)
e1.record()
torch.cuda.synchronize()
print("call ms %.3f" % e0.elapsed_time(e1))
buf = (ctypes.c_ulonglong * (64 * 16 + 4 * 4096))()
_lib.check(_lib.lib().lmoe_debug_trace_read(buf))
t = np.array(buf, dtype=np.int64)[64 * 16:64 * 16 + 16 * 64 * 5].reshape(16, 64, 5).astype(np.float64)
P = plan["ctas_per_head"]
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)
nseg = plan["segments"]
rows = []
for seg in range(nseg):
    jj, un = seg % P, seg // P
    if un >= 64 or jj >= 16:
        continue
    a0, a1, acq, pub, c1 = t[jj, un]
    rows.append((seg, jj, un, a0, a1, acq, pub, c1))
print("seg cta unit  A0     A1    acq    pub     C1  | A_ms  wait  chain  C")
for seg, jj, un, a0, a1, acq, pub, c1 in rows[:40] + rows[-12:]:
    print("%3d %3d %3d %7.1f %7.1f %7.1f %7.1f %7.1f | %5.1f %5.1f %5.1f %5.1f" % (
        seg, jj, un, a0, a1, acq, pub, c1, a1 - a0, acq - a1, pub - acq, c1 - pub))
r = np.array([x[3:] for x in rows])
print("medians: A %.2f  wait %.2f  chain(acq->pub) %.2f  C %.2f  hop(pub_s - pub_{s-1}) %.2f us" % (
    np.nanmedian(r[:, 1] - r[:, 0]), np.nanmedian(r[:, 2] - r[:, 1]), np.nanmedian(r[:, 3] - r[:, 2]),
    np.nanmedian(r[:, 4] - r[:, 3]), np.nanmedian(np.diff(r[:, 3]))))
