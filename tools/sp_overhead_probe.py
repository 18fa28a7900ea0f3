"""Host vs device time of one SP forward step at slice 32768 (cfg3 per-rank work at T = 8):
event-timed back-to-back calls, the sum of the library's per-phase device timings, and a
CUDA-graph replay of the same step."""
import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import _lib, sp

import sys
H, D = 16, 128
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
comm = sp.NcclComm(0, 1)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, n, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
spec = pk.LsmSpec.make("mamba2", D)
spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=g).mul_(0.5)
gates = pk.LsmGates(b_pre=torch.randn(1, n, H, device="cuda", generator=g))
out = torch.empty_like(q)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    print("back-to-back calls: %.3f ms / step" % (e0.elapsed_time(e1) / 20))
    _lib.timing_read(8)
    for _ in range(20):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, timing=True, stream=st.cuda_stream)
    torch.cuda.synchronize()
    calls, ph = _lib.timing_read(8)
    print("device phases (ms / step):", ["%.4f" % (x / calls) for x in ph[:6]], "sum %.3f" % (sum(ph[:6]) / calls))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
    graph.replay()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(20):
        graph.replay()
    e1.record(st)
    torch.cuda.synchronize()
    print("CUDA graph replay: %.3f ms / step" % (e0.elapsed_time(e1) / 20))
