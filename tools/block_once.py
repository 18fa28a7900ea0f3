"""One cfg4 Linear-MoE block (GLA + 64-expert top-8 MoE, 8 x 8192 tokens) for ncu launch lists."""
import torch

from paper_2503_05447_b200.lsm import LsmInstance
from paper_2503_05447_b200.model import Model, ModelConfig

cfg = ModelConfig(hidden=1024, ffn_dim=896, num_heads=8, num_experts=64, num_active=8, vocab_size=256,
                  instance=LsmInstance.GLA, pattern="L", max_seq_len=8192)
m = Model.init(cfg, seed=0, device="cuda")
B, N = 8, 8192
x = torch.randn(B * N, cfg.hidden, device="cuda")
for _ in range(2):
    m.run_block(0, x, B, N)
torch.cuda.synchronize()
