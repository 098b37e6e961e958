"""Per-phase SELECT diagnostics on real FULL-kernel scores:
    python scripts/select_diag.py [config] [context] [top_k] [batch] [layers]
info[2] = mode: 0 fast, 2 fast+refined, 1+16*r generic (r: 1 bad brackets, 2 cgt>=k,
3 k beyond band, 4 candidate overflow, 5 window outside bins), 5 tie pass."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_00777_b200.attention import full_attention, topk_select  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
if len(sys.argv) > 2:
    N, k, B, L = (int(x) for x in sys.argv[2:6])
    cfg = cfg.with_(context=N, budget=k, batch=B, layers=L,
                    full_layers=tuple(f for f in cfg.full_layers if f < L))
q, kk, v = generate_torch(cfg, "cuda")
fl = list(cfg.full_layers)
out, sc = full_attention(q, kk, v, cfg.context, layers=fl)
for refine in (True, False):
    idx, inf = topk_select(sc, cfg.budget, cfg.context, q=q if refine else None,
                           k=kk if refine else None, layers=fl, info=True)
    torch.cuda.synchronize()
    i = inf.view(-1, 8).cpu().numpy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        topk_select(sc, cfg.budget, cfg.context, q=q if refine else None,
                    k=kk if refine else None, layers=fl)
    e1.record()
    torch.cuda.synchronize()
    print(f"  launch time {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
    print(f"{cfg.name} N={cfg.context} k={cfg.budget} B={cfg.batch} refine={refine} rows={len(i)}")
    print("  mode counts", dict(zip(*[x.tolist() for x in np.unique(i[:, 2], return_counts=True)])))
    print("  band size min/med/max", i[:, 3].min(), np.median(i[:, 3]), i[:, 3].max())
    print("  window min/med/max", i[:, 1].min(), np.median(i[:, 1]), i[:, 1].max())
    for j, name in zip(range(4, 8), ["A sample", "B pass", "C+D", "E window+compact"]):
        print(f"  {name}: median {np.median(i[:, j]):.0f} cycles, max {i[:, j].max()}")
