import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from oracle import hylra_oracle as orc
from paper_2602_00777_b200.engine import HybridDecoder
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch

def rel(x, r): return float(np.linalg.norm(x - r) / np.linalg.norm(r))
cfg = CONFIGS["cfg2"].with_(batch=1)
q, k, v = generate_torch(cfg, "cuda")
dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
res = dec.step(q, cfg.context)
torch.cuda.synchronize()
N = cfg.context
for l in range(cfg.layers):
    qn = q[l, 0].double().cpu().numpy(); kn = k[l, 0, 3].double().cpu().numpy(); vn = v[l, 0, 3].double().cpu().numpy()
    slot = res.slot_of_layer[l]
    sel = res.selections[slot, 0, 3].cpu().numpy()
    if cfg.actions[l] == "full":
        ref, _ = orc.full_attention(qn[13], kn, vn)
    else:
        ref = orc.subset_attention(qn[13], kn, vn, sel)
    got = res.outputs[l, 0, 13].double().cpu().numpy()
    print(l, cfg.actions[l], slot, round(rel(got, ref), 5), got[:3], ref[:3], flush=True)
