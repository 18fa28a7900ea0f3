"""Per-phase clock64 timeline of one output-pass CTA (developer aid).
   LMOE_TRACE=1 [LMOE_OP_ORDER=0|1] python tools/trace_lsm.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib
N, H, D = int(os.environ.get("N", 262144)), 16, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16) for _ in range(3))
spec = pk.LsmSpec.make(os.environ.get("INST", "mamba2"), D)
# A_RAW=<float>: every head's a_raw (default 0.3); A_RAW=rand: N(0, 0.5^2) as in bench.py
ar = os.environ.get("A_RAW", "0.3")
spec.mamba2_a_raw = (torch.randn(H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)).mul_(0.5)
                     if ar == "rand" else torch.full((H,), float(ar), device="cuda"))
gates = pk.LsmGates(b_pre=torch.randn(1, N, H, device="cuda", generator=g)) if spec.instance == 13 else None
for _ in range(3):
    pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 16 + 4 * 4096))()
_lib.check(_lib.lib().lmoe_debug_trace_read(buf))
t = np.array(buf, dtype=np.int64)[:64 * 16].reshape(64, 16)
t0 = t[0, 10]
names = {10: "load", 9: "S_iss", 6: "QMDM", 7: "PV", 8: "commit", 0: "m:S", 1: "m:xf2", 2: "m:P", 3: "m:mo", 4: "m:mrd", 5: "m:O"}
order = [10, 9, 0, 1, 2, 6, 7, 8, 3, 4, 5]
print("chunk " + " ".join("%7s" % names[i] for i in order) + "   (cycles rel. to load(0))")
for c in range(0, 64):
    row = t[c]
    if row[10] == 0:
        break
    if c < 4 or c % 8 == 0:
        print("%5d " % c + " ".join("%7d" % (row[i] - t0 if row[i] else -1) for i in order))
last = max(i for i in range(64) if t[i, 10] != 0)
per = (t[last, 5] - t[4, 5]) / (last - 4)
print("steady-state cycles per chunk (m:O deltas): %.0f" % per)
tt = np.array(buf, dtype=np.int64)[64 * 16:64 * 16 + 4096].reshape(-1, 2)
ok = tt[:, 0] > 0
busy = (tt[ok, 1] - tt[ok, 0]) / 1e3
print("globaltimer: CTA 0 busy %.1f us; all CTAs busy median %.1f, max %.1f us; kernel span %.1f us (%d CTAs)"
      % (busy[0], np.median(busy), busy.max(), (tt[ok, 1].max() - tt[ok, 0].min()) / 1e3, ok.sum()))
