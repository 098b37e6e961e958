"""Block-mode SELECT diagnostics on real FULL-kernel scores (cfg2 by default):
    python scripts/block_diag.py [config] [batch] [block_size] [block_budget]
Prints info[2] mode counts (0 fast, 2 fast+refined, 1+16*r generic) and phase cycles,
plus eager timings of block_select with and without the float64 refinement."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_00777_b200.attention import block_select, full_attention  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
bs = int(sys.argv[3]) if len(sys.argv) > 3 else 128
bb = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.budget // bs
cfg = cfg.with_(batch=B)
q, kk, v = generate_torch(cfg, "cuda")
fl = list(cfg.full_layers)
out, sc = full_attention(q, kk, v, cfg.context, layers=fl)
for refine in (True, False):
    kw = dict(q=q, k=kk, layers=fl) if refine else {}
    res = block_select(sc, bb, bs, cfg.context, info=True, **kw)
    torch.cuda.synchronize()
    i = res[3].view(-1, 8).cpu().numpy()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        block_select(sc, bb, bs, cfg.context, **kw)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{cfg.name} B={B} bs={bs} bb={bb} refine={refine} rows={len(i)} "
          f"eager {ev[0].elapsed_time(ev[1]) / 10 * 1e3:.1f} us/call")
    print("  mode counts", dict(zip(*[x.tolist() for x in np.unique(i[:, 2], return_counts=True)])))
    print("  window min/med/max", i[:, 1].min(), np.median(i[:, 1]), i[:, 1].max())
    for j, name in zip(range(4, 8), ["A sample", "B pass", "C+D", "E window+compact"]):
        print(f"  {name}: median {np.median(i[:, j]):.0f} cycles, max {i[:, j].max()}")
