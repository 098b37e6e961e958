"""Graph variants of the e2e step, each timed by CUDA events over back-to-back replays:
which part of H2D / append / step / D2H costs what.  python scripts/e2e_parts.py [--batch 1]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
cfg = CONFIGS[a.config].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda", capacity=cfg.context)
dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
L, B, Hq, d = q.shape
Hkv = k.shape[2]
pos = cfg.context - 1
q_host = torch.zeros((L, B, Hq, d), dtype=q.dtype).pin_memory()
kv_host = torch.zeros((2, L, B, Hkv, d), dtype=q.dtype).pin_memory()
out_host = torch.zeros((L, B, Hq, d), dtype=torch.float32).pin_memory()
q_dev = q.clone()
kv_dev = torch.stack([k[:, :, :, pos], v[:, :, :, pos]]).contiguous()
# host buffers hold the real step inputs (all-zero queries would make every score tie)
q_host.copy_(q.cpu())
kv_host.copy_(kv_dev.cpu())


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def ev_time(g, n=30):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n * 1e3, 1)


k_rows = kv_host[0]
v_rows = kv_host[1]
parts = {
    "step": lambda: dec.step(q_dev, pos + 1),
    "step_out_pinned": lambda: dec.step(q_dev, pos + 1, out=out_host),
    "append_zero_copy": lambda: dec.append(k_rows, v_rows, pos),
    "step_q_out_pinned": lambda: dec.step(q_host, pos + 1, out=out_host),
    "h2d": lambda: (q_dev.copy_(q_host, non_blocking=True), kv_dev.copy_(kv_host, non_blocking=True)),
    "append": lambda: (dec.k[:, :, :, pos].copy_(kv_dev[0]), dec.v[:, :, :, pos].copy_(kv_dev[1])),
    "d2h": lambda: out_host.copy_(dec.out, non_blocking=True),
    # the new rows written by the step itself (single-launch kernel: no append launch)
    "zc_step_append": lambda: dec.step(q_host, pos + 1, out=out_host,
                                       append=(k_rows, v_rows, pos)),
}
res = {}
for name, fn in parts.items():
    res[name] = ev_time(graph_of(fn))
combos = {
    "h2d+step": ("h2d", "step"), "append+step": ("append", "step"), "step+d2h": ("step", "d2h"),
    "all": ("h2d", "append", "step", "d2h"),
    "zc_all": ("h2d", "append_zero_copy", "step_out_pinned"),
    "zc_all_q": ("append_zero_copy", "step_q_out_pinned"),
}
for name, names in combos.items():
    res[name] = ev_time(graph_of(lambda names=names: [parts[n]() for n in names]))
print(a.batch, res)
