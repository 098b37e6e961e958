"""A/B of step schedules (graph replays, CUDA events), interleaved repetitions:
    python scripts/ab_schedules.py [--batch 8] [--reps 5] [--steps 50]"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--context", type=int, default=None)
ap.add_argument("--budget", type=int, default=None)
ap.add_argument("--layers", type=int, default=None)
a = ap.parse_args()
cfg = CONFIGS[a.config].with_(batch=a.batch)
if a.context:
    cfg = cfg.with_(context=a.context)
if a.budget:
    cfg = cfg.with_(budget=a.budget)
if a.layers:
    cfg = cfg.with_(layers=a.layers, full_layers=tuple(f for f in cfg.full_layers if f < a.layers))
q, k, v = generate_torch(cfg, "cuda")
kinds = {"fused3": {"fuse_select": False},
         "fusedsel": {"fuse_select": True, "single_launch": False},
         "dual": {"dual_stream": True, "fuse_select": False},
         "single": {"single_launch": True}}
graphs = {}
for name, kw in kinds.items():
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads, **kw)
    for _ in range(3):
        dec.step(q, cfg.context)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cfg.context)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dec.step(q, cfg.context)
    graphs[name] = (g, dec)
torch.cuda.synchronize()
ref = graphs["fused3"][1]
for name, (g, dec) in graphs.items():
    # dual splits the FULL launch (other split-K partitions): same sets, outputs to rounding
    assert torch.equal(dec.idx, ref.idx), name
    if name != "dual" and not torch.equal(dec.out, ref.out):
        bad = [(l, float((dec.out[l] - ref.out[l]).abs().max()))
               for l in range(dec.out.shape[0]) if not torch.equal(dec.out[l], ref.out[l])]
        print(f"{name}: outputs differ from fused3 at layers {bad}", flush=True)
res = {n: [] for n in kinds}
for _ in range(a.reps):
    for name, (g, _) in graphs.items():
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / a.steps * 1e3)
print(f"{a.config} N={cfg.context} k={cfg.budget} L={cfg.layers} B={a.batch}", {n: (round(statistics.median(v), 1), round(min(v), 1))
                                  for n, v in res.items()})
