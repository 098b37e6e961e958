"""Timeline of one dual-stream step (eager) from per-layer completion events:
    python scripts/dual_timeline.py [--batch 8]
Prints when FULL(A), REUSE (last chunk), FULL(B) finished and when the step ended,
relative to an event recorded just before the step, for dual and single-stream steps."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
a = ap.parse_args()
cfg = CONFIGS["cfg2"].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
L = cfg.layers
acts = cfg.actions
for dual in (False, True, "fused"):
    dec = HybridDecoder(acts, k, v, cfg.budget, q_heads=cfg.q_heads, dual_stream=dual is True,
                        fuse_select=dual == "fused")
    feeds = [l for l in range(L) if acts[l] == "full" and l + 1 < L and acts[l + 1] == "reuse"]
    others = [l for l in range(L) if acts[l] == "full" and l not in feeds]
    last_reuse = max(l for l in range(L) if acts[l] == "reuse")
    marks = {feeds[0]: "FULL(A) done", others[0]: "FULL(B) done", last_reuse: "REUSE done"}
    for rep in range(4):
        evs = [torch.cuda.Event(enable_timing=True) if l in marks else None for l in range(L)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for e in evs:
            if e is not None:
                e.record()  # creates the event (torch does so lazily); the step re-records it
        torch.cuda.synchronize()
        e0.record()
        dec.step(q, cfg.context, layer_events=evs)
        e1.record()
        torch.cuda.synchronize()
    line = {name: round(e0.elapsed_time(evs[l]) * 1e3, 1) for l, name in marks.items()}
    line["end"] = round(e0.elapsed_time(e1) * 1e3, 1)
    print(f"B={a.batch} dual={dual}", line)
