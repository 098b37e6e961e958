"""Where a layer-sequential REUSE layer's time goes at small batch: graph-replayed runs of
24 REUSE-layer launches (LayerwiseDecoder.layer, early loads on), over
  * the 24 distinct REUSE layers (their rows mostly come from HBM: 201 MB at cfg2 B=1), and
  * one REUSE layer 24 times (its 8.4 MB of rows stay L2-resident after the first),
plus a FULL layer and its select alone. python scripts/seq_l2_probe.py [B]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import LayerwiseDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402


def graph_us(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


import os  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402

# optional tuning knobs for the whole run: SEQ_TUNING="rowsel_cluster=4,bulk_merge=0"
_tun = dict((kv.split("=")[0], int(kv.split("=")[1]))
            for kv in os.environ.get("SEQ_TUNING", "").split(",") if kv)
if _tun:
    _abi.tuning(**_tun).__enter__()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = CONFIGS["cfg2"].with_(batch=B)
q, k, v = generate_torch(cfg, "cuda")
n = cfg.context
dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
dec.step(q, n)
torch.cuda.synchronize()
reuse = [l for l, a in enumerate(cfg.actions) if a == "reuse"]
full = [l for l, a in enumerate(cfg.actions) if a == "full"]


def run(layers):
    def f():
        dec._prev = "reuse"
        for l in layers:
            dec.layer(l, q, n)
        dec.finish()
    return f


t_step = graph_us(lambda: dec.step(q, n))
t_cold = graph_us(run(reuse))
t_warm = graph_us(run([reuse[0]] * len(reuse)))
t_full = graph_us(run([full[0]] * 4))  # FULL layer 0 does not feed: select on the side
feed = full[2]
t_feed = graph_us(run([feed] * 4))
print(f"cfg2 B={B}: step {t_step:.1f} us | 24 REUSE distinct {t_cold:.1f} us "
      f"({t_cold / 24:.2f}/layer) | 24 x one REUSE (L2-warm) {t_warm:.1f} us "
      f"({t_warm / 24:.2f}/layer) | FULL(non-feeding) {t_full / 4:.2f}/layer | "
      f"FULL+select (feeding) {t_feed / 4:.2f}/layer", flush=True)
