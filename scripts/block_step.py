import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2602_00777_b200.engine import HybridDecoder
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch
cfg = CONFIGS["cfg2"].with_(batch=8)
q, k, v = generate_torch(cfg, "cuda")
dec = HybridDecoder(cfg.actions, k, v, cfg.budget // 128, q_heads=cfg.q_heads, block_size=128)
for _ in range(3):
    dec.step(q, cfg.context)
torch.cuda.synchronize()
