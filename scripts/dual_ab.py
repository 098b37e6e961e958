"""Graph-replayed step time of every batched schedule including "dual" (selects on a
high-priority side stream under the next streaming launch), per config / batch:
    python scripts/dual_ab.py [cfg2:1,2,4] [cfg3:1] ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

for arg in sys.argv[1:] or ["cfg2:1,2,4"]:
    name, bs = arg.split(":")
    for B in (int(x) for x in bs.split(",")):
        cfg = CONFIGS[name].with_(batch=B)
        q, k, v = generate_torch(cfg, "cuda")
        dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
        t = dec.autotune(q, cfg.context, reps=20)
        print(f"{name} B={B}: " + "  ".join(f"{n} {ms * 1e3:.1f}" for n, ms in t.items())
              + f"  -> {dec.schedule}", flush=True)
        del dec, q, k, v
        torch.cuda.empty_cache()
