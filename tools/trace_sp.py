"""Kernel timeline (globaltimer, us) of one cfg3 Mamba2 SP forward step at a rank slice
(default 32768 = the T = 8 per-rank work), world 1, replayed from a CUDA graph as bench.py
does (LMOE_TRACE=1): per kernel, CTA prologue-done / after-PDL-wait / end."""
import ctypes
import os
import sys

os.environ["LMOE_TRACE"] = "1"
import numpy as np
import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib, sp

H, D = 16, 128
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
comm = sp.NcclComm(0, 1)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, n, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
spec = pk.LsmSpec.make("mamba2", D)
ga = torch.Generator(device="cuda").manual_seed(1)  # as tools/sp_scaling_probe.py
spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=ga).mul_(0.5)
gates = pk.LsmGates(b_pre=torch.randn(1, n, H, device="cuda", generator=g))
out = torch.empty_like(q)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 16 + 4 * 4096))()
_lib.check(_lib.lib().lmoe_debug_trace_read(buf))
t = np.array(buf, dtype=np.int64)[64 * 16:].reshape(4, 2048, 2)
outp, stp, waits, smid = t[0], t[1], t[2], t[3]
o_ok, s_ok = outp[:, 0] > 0, stp[:, 0] > 0
t0 = stp[s_ok, 0].min()
us = lambda x: (x - t0) / 1e3


def show(name, start, wait, end):
    print("%-12s CTAs %4d | start %7.1f..%7.1f | after wait %7.1f..%7.1f | end %7.1f / med %7.1f / %7.1f | busy med %.1f"
          % (name, len(start), us(start.min()), us(start.max()), us(wait.min()), us(wait.max()),
             us(end.min()), us(np.median(end)), us(end.max()), np.median(end - wait) / 1e3))


show("state pass", stp[s_ok, 0], waits[s_ok, 1], stp[s_ok, 1])
show("output pass", outp[o_ok, 0], waits[o_ok, 0], outp[o_ok, 1])

# output-pass busy time per CTA against its segment / head / SM
nseg = int(o_ok.sum()) // H
busy = ((outp[:, 1] - waits[:, 0]) / 1e3)[: nseg * H].reshape(H, nseg)
print("output busy by segment (mean over heads):", " ".join("%.1f" % x for x in busy.mean(0)))
print("output busy by head (mean over segments):", " ".join("%.1f" % x for x in busy.mean(1)))
sm = smid[: nseg * H, 0]
order = np.argsort(sm)
print("output busy by SM id (sorted):", " ".join("%d:%.0f" % (sm[i], busy.reshape(-1)[i]) for i in order))
