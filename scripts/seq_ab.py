"""Layer-sequential decode (LayerwiseDecoder) against the batched step, graph-replayed:
    python scripts/seq_ab.py [cfg2:1,8] ...
prints ms per step for sequential with / without early loads and for the autotuned batched
step, and the ratio."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
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


for arg in sys.argv[1:] or ["cfg2:1,8"]:
    name, bs = arg.split(":")
    for B in (int(x) for x in bs.split(",")):
        cfg = CONFIGS[name].with_(batch=B)
        q, k, v = generate_torch(cfg, "cuda")
        n = cfg.context
        bat = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
        bat.autotune(q, n)
        t_b = graph_ms(bat, q, n)
        res = {}
        for label, kw, tun in (("seq", {}, {}), ("seq-noprefetch", {"prefetch": False}, {}),
                               ("seq-streamsel", {}, {"rowsel": 0})):
            with _abi.tuning(**tun) if tun else _abi.tuning():
                dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads, **kw)
                res[label] = graph_ms(dec, q, n)
            del dec
        print(f"{name} B={B}: batched({bat.schedule}) {t_b * 1e3:.1f} us | " +
              " | ".join(f"{k_} {t * 1e3:.1f} us ({t / t_b:.2f}x)" for k_, t in res.items()),
              flush=True)
        del bat, q, k, v
        torch.cuda.empty_cache()
