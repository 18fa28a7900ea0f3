"""Per-rank step time of the cfg3 SP forward at the slice lengths of T = 1, 2, 4, 8 ranks
(one GPU), to bound strong-scaling efficiency.  The Mamba2 per-head decays are the same at
every T (the slice length would otherwise shift the random stream).  For T > 1 the step runs
through a real 1-rank NCCL communicator: the multi-rank phase structure with its
ncclAllGather (of this rank's payload only); the T = 1 baseline is the local path bench.py
times.  The projection adds the gather of the other T - 1 ranks' payloads (B*H*(D*D + 1) fp32
each) at the measured NVLink peer-copy bandwidth (770 GB/s, B200_PROFILING.md) plus a 10 us
collective latency."""
import os

import torch

import paper_2503_05447_b200 as pk
from paper_2503_05447_b200 import sp

H, D = 16, 128
comm = sp.NcclComm(0, 1, single_rank_nccl=True)
local = sp.NcclComm(0, 1)
PAYLOAD = H * (D * D + 1) * 4
for inst in ("mamba2", "gla"):
    base = None
    for T in (1, 2, 4, 8):
        n = 262144 // T
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = (torch.randn(1, n, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
        spec = pk.LsmSpec.make(inst, D)
        if inst == "mamba2":
            ga = torch.Generator(device="cuda").manual_seed(1)  # same per-head decays at every T
            spec.mamba2_a_raw = torch.randn(H, device="cuda", generator=ga).mul_(0.5)
            gates = pk.LsmGates(b_pre=torch.randn(1, n, H, device="cuda", generator=g))
        else:
            gates = pk.LsmGates(a_pre=torch.randn(1, n, H, D, device="cuda", generator=g).bfloat16())
        cm = comm if T > 1 else local
        # graph replay, as bench.py times the step
        st = torch.cuda.Stream()
        out = torch.empty_like(q)
        with torch.cuda.stream(st):
            for _ in range(3):
                sp.sp_lsm_masked_rank(cm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                sp.sp_lsm_masked_rank(cm, q, k, v, gates, spec, 64, out=out, check=False, stream=st.cuda_stream)
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(50):
                graph.replay()
            e1.record(st)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        # evented phases of the same call outside the graph (phase layout: lsm_host.cu marks)
        from paper_2503_05447_b200 import _lib
        _lib.timing_read(8)
        for _ in range(10):
            sp.sp_lsm_masked_rank(cm, q, k, v, gates, spec, 64, out=out, check=False, timing=True)
        torch.cuda.synchronize()
        calls, ph = _lib.timing_read(8)
        print("  phases (ms, evented, not graphed):", " ".join("%.4f" % (x / max(calls, 1)) for x in ph))
        base = base or ms
        gather_ms = 0.0 if T == 1 else ((T - 1) * PAYLOAD / 770e9 + 10e-6) * 1e3
        print("%s T=%d slice=%d: %.3f ms per rank step (graph, NCCL 1-rank); + modelled gather %.3f ms; "
              "ideal %.3f; efficiency bound %.1f%%, with the gather %.1f%%"
              % (inst, T, n, ms, gather_ms, base / T, 100 * base / (T * ms), 100 * base / (T * (ms + gather_ms))))
