"""Profiling driver: a few eager hybrid decode steps of a BASELINE config (for ncu).

    python scripts/prof_step.py [--config cfg2] [--batch 8] [--steps 3]

Kernels per step by --schedule: single = step_mma_kernel (every FULL item with its select
fused, then every REUSE item); fusedsel = attn_mma_kernel (FULL, selects of the layers that
feed REUSE fused) -> topk_select_kernel (other FULL layers, side stream) -> attn_mma_kernel
(REUSE gather); fused3 = FULL -> SELECT -> REUSE; sequential = LayerwiseDecoder (per layer:
FULL + its select, or REUSE); auto = HybridDecoder's choice.
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--block-size", type=int, default=1)
ap.add_argument("--schedule", default="auto",
                choices=["auto", "single", "fusedsel", "fused3", "dual", "sequential"])
a = ap.parse_args()
cfg = CONFIGS[a.config]
if a.batch:
    cfg = cfg.with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
torch.cuda.synchronize()
bs = a.block_size
if a.schedule == "sequential":
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
else:
    kw = {"auto": {}, "single": {"single_launch": True},
          "fusedsel": {"single_launch": False}, "fused3": {"fuse_select": False},
          "dual": {"fuse_select": False, "dual_stream": True}}[a.schedule]
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget // bs if bs > 1 else cfg.budget,
                        q_heads=cfg.q_heads, block_size=bs, **kw)
for _ in range(a.steps):
    dec.step(q, cfg.context)
torch.cuda.synchronize()
dec.check_flags()
print("ok", cfg.name, cfg.batch)
