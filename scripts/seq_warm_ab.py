"""Layer-sequential decode with / without the L2 warm-up of the FULL layer that follows
each REUSE run (LayerwiseDecoder l2_prefetch), graph-replayed:
    python scripts/seq_warm_ab.py [cfg2:1,8] ...
prints ms per step for each prefetch fraction and the batched step's."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder, LayerwiseDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402



def graph_ms(dec, q, n, reps=20):
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

VARIANTS = [("none", None, 0), ("1/4", (1, 4), 0), ("1/2", (1, 2), 0), ("3/4", (3, 4), 0),
            ("1/1", (1, 1), 0), ("1/2 evict_last", (1, 2), 1), ("3/4 evict_last", (3, 4), 1)]

for arg in sys.argv[1:] or ["cfg2:1,8"]:
    name, bs = arg.split(":")
    for B in (int(x) for x in bs.split(",")):
        cfg = CONFIGS[name].with_(batch=B)
        q, k, v = generate_torch(cfg, "cuda")
        n = cfg.context
        bat = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
        bat.autotune(q, n)
        t_b = graph_ms(bat, q, n)
        del bat
        ref = None
        out = []
        for label, frac, fl in VARIANTS:
            dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads,
                                   l2_prefetch=frac, l2_prefetch_flags=fl)
            t = graph_ms(dec, q, n)
            res = dec.step(q, n)
            torch.cuda.synchronize()
            o = res.outputs.clone()
            if ref is None:
                ref = o
            same = bool(torch.equal(o, ref))
            out.append(f"{label} {t * 1e3:.1f} us ({t / t_b:.2f}x{'' if same else ' DIFF'})")
            del dec
        print(f"{name} B={B}: batched {t_b * 1e3:.1f} us | " + " | ".join(out), flush=True)
        del q, k, v
        torch.cuda.empty_cache()
