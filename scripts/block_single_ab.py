"""Block-mode step (cfg2, block_size 128, 16 blocks = 2048 tokens): single launch vs the
multi-launch block step, graph replays.   python scripts/block_single_ab.py [--batch 8]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
cfg = CONFIGS["cfg2"].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
res, outs = {}, {}
for single in (False, True, False, True):
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget // 128, q_heads=cfg.q_heads, block_size=128,
                        single_launch=single)
    for _ in range(3):
        dec.step(q, cfg.context)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cfg.context)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dec.step(q, cfg.context)
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    name = "single" if single else "multi"
    res.setdefault(name, []).append(round(e0.elapsed_time(e1) / a.steps * 1e3, 1))
    outs[name] = (dec.out.clone(), dec.idx.clone())
same = all(torch.equal(x, y) for x, y in zip(outs["single"], outs["multi"]))
print(f"cfg2 blocks B={a.batch} step us", res, "bit-identical", same)
