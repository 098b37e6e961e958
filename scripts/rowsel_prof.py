"""Per-phase clock marks of the shared-memory-resident select (diagnostics build
-DHYLRA_ROWSEL_PROF loaded through HYLRA_LIB): load | minmax | hist | band pass | T | window |
re-score+rank | compaction cycles, for one config's FULL-layer score rows.
    HYLRA_LIB=.../libhylra_rsprof.so python scripts/rowsel_prof.py cfg2 1 [cluster]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.attention import full_attention, topk_select  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name].with_(batch=B)
q, k, v = generate_torch(cfg, "cuda")
fl = [l for l, a in enumerate(cfg.actions) if a == "full"][:1]
_, sc = full_attention(q, k, v, cfg.context, layers=fl)
for c in ([int(sys.argv[3])] if len(sys.argv) > 3 else [1, 2, 4, 8]):
    for refine in (True, False):
        kw = dict(q=q, k=k, layers=fl) if refine else dict(layers=fl)
        with _abi.tuning(rowsel=1, rowsel_cluster=c):
            for _ in range(3):
                _, inf = topk_select(sc, cfg.budget, cfg.context, info=True, **kw)
        print(f"{name} B={B} C>={c} refine={refine}:",
              inf.reshape(-1, 8)[:2].tolist(), flush=True)
