"""Throughput of lmoe_attn_fwd at the cfg5 per-rank shapes (SP T=8 over N=131072, H=16, d=128):
rank r has 16384 queries with row_offset 16384 r against the gathered keys.  CUDA events."""
import json
import sys

import torch

from paper_2503_05447_b200 import attn

N, T, H, D = 131072, 8, 16, 128
L = N // T
ranks = [int(a) for a in sys.argv[1:]] or [0, 3, 7]
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn(1, N, H, D, device="cuda", generator=g).bfloat16()
v = torch.randn(1, N, H, D, device="cuda", generator=g).bfloat16()
q = torch.randn(1, L, H, D, device="cuda", generator=g).bfloat16()
for r in ranks:
    off = r * L
    nk = off + L
    for _ in range(2):
        attn.softmax_attention_parallel(q, k[:, :nk], v[:, :nk], True, row_offset=off)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    it = 5
    for _ in range(it):
        attn.softmax_attention_parallel(q, k[:, :nk], v[:, :nk], True, row_offset=off)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / it
    # causal-effective flops: 4 d per (query, allowed key)
    pairs = L * off + L * (L + 1) / 2
    tf = 4 * D * pairs * H / ms / 1e9
    print(json.dumps({"rank": r, "Nq": L, "Nk": nk, "ms": round(ms, 3), "tflops": round(tf, 1)}))
