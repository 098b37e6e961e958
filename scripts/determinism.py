"""Run-to-run determinism of each step schedule at a BASELINE config: the same inputs
stepped repeatedly must give bit-identical outputs and selections.
    python scripts/determinism.py [--config cfg2] [--batch 8] [--reps 6]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--norefine", action="store_true")
a = ap.parse_args()
cfg = CONFIGS[a.config].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
kinds = {"fused3": {"fuse_select": False},
         "fusedsel": {"fuse_select": True, "single_launch": False},
         "single": {"single_launch": True},
         "dual": {"dual_stream": True, "fuse_select": False}}
for name, kw in kinds.items():
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads,
                        refine=not a.norefine, **kw)
    dec.step(q, cfg.context)
    torch.cuda.synchronize()
    out0, idx0 = dec.out.clone(), dec.idx.clone()
    bad = []
    for r in range(a.reps):
        dec.step(q, cfg.context)
        torch.cuda.synchronize()
        if not torch.equal(dec.idx, idx0):
            bad.append((r, "idx"))
        diff = [l for l in range(dec.out.shape[0]) if not torch.equal(dec.out[l], out0[l])]
        if diff:
            bad.append((r, diff))
    print(name, "deterministic" if not bad else f"DIFFERS {bad}", flush=True)
