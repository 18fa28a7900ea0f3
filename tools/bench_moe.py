"""MoE layer throughput at BASELINE config 4 (A0.3B-2B: hidden 1024, ffn 896, E=64, k=8,
seq 8192 x batch 8 = 65536 tokens), bf16; prints one JSON line (developer tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_05447_b200 import moe
T, H, F, E, K = 65536, 1024, 896, 64, 8
g = torch.Generator(device="cuda").manual_seed(0)
layer = moe.MoeLayer.init(moe.MoeConfig(E, K, H, F), generator=g)
x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
y = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    layer.forward(x, out=y)
torch.cuda.synchronize()
steps = int(os.environ.get("STEPS", "10"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    layer.forward(x, out=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
flops = 6.0 * T * K * H * F + 2.0 * T * H * E
print(json.dumps({"workload": "cfg4 MoE layer", "tokens": T, "ms_per_step": ms, "tokens_per_s": T / ms * 1e3,
                  "tflops": flops / ms / 1e9, "frac_of_bf16_peak": flops / ms / 1e9 / 1629.1}))
