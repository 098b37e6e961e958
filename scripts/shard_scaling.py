"""Per-GPU work of the multi-GPU partitions, measured one shard at a time on ONE B200: for
N in {1, 2, 4, 8}, the step of one shard of BASELINE config 3 (128K, global B=4, sharded by
KV head: Hkv 8/N, Hq 32/N per GPU) and config 4 (Qwen 64K, global B=16, 4 KV heads:
sharded by batch, B 16/N per GPU), autotuned and graph-replayed. No collective is timed:
the data path has none (north_star), and the all-gather of the shard outputs is reported
separately by bench.py at N>1. The efficiency column T_1 / (N T_N) is the bound the shard's
own kernels put on strong scaling. python scripts/shard_scaling.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402


def graph_ms(dec, q, n, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            dec.step(q, n)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, n)
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for name, B, mode in (("cfg3", 4, "kv"), ("cfg4", 16, "batch")):
    base = CONFIGS[name].with_(batch=B)
    t1 = None
    for N in (1, 2, 4, 8):
        if mode == "kv":
            cfg = base.with_(kv_heads=base.kv_heads // N, q_heads=base.q_heads // N)
        else:
            if B % N:
                continue
            cfg = base.with_(batch=B // N)
        q, k, v = generate_torch(cfg, "cuda")
        dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
        dec.autotune(q, cfg.context)
        t = graph_ms(dec, q, cfg.context)
        kvb = 2 * k.element_size() * k.shape[-1]  # K + V bytes per row
        L_full = sum(1 for a in cfg.actions if a == "full")
        L_reuse = len(cfg.actions) - L_full
        rows = cfg.batch * cfg.kv_heads * (L_full * cfg.context + L_reuse * cfg.budget)
        gbs = rows * kvb / (t * 1e-3) / 1e9
        t1 = t if N == 1 else t1
        eff = t1 / (N * t)
        print(f"{name} {mode}-shard N={N}: per-GPU shard B={cfg.batch} Hkv={cfg.kv_heads} "
              f"Hq={cfg.q_heads}: {t:.3f} ms ({dec.schedule}), {gbs:.0f} GB/s, "
              f"strong-scaling efficiency of the shard kernels {eff:.3f}", flush=True)
        del dec, q, k, v
        torch.cuda.empty_cache()
