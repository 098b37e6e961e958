"""Per-phase SELECT diagnostics on a BASELINE config's real scores (FULL kernel output)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_00777_b200.attention import full_attention, topk_select  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
q, k, v = generate_torch(cfg, "cuda")
fl = list(cfg.full_layers)
out, sc = full_attention(q, k, v, cfg.context, layers=fl)
for refine in (True, False):
    idx, inf = topk_select(sc, cfg.budget, cfg.context, q=q if refine else None,
                           k=k if refine else None, layers=fl, info=True)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        topk_select(sc, cfg.budget, cfg.context, q=q if refine else None, k=k if refine else None,
                    layers=fl)
    ev[1].record()
    torch.cuda.synchronize()
    i = inf.view(-1, 8).cpu().numpy()
    print(f"refine={refine} ms/launch={ev[0].elapsed_time(ev[1]) / 10:.3f} rows={len(i)}")
    print("  mode counts", np.unique(i[:, 2], return_counts=True))
    print("  band size min/med/max", i[:, 3].min(), np.median(i[:, 3]), i[:, 3].max())
    print("  refine cands min/med/max", i[:, 1].min(), np.median(i[:, 1]), i[:, 1].max())
    for j, name in zip(range(4, 8), ["A sample", "B pass", "C+D", "E compact"]):
        print(f"  {name}: median {np.median(i[:, j]):.0f} cycles, max {i[:, j].max()}")
