"""Where does the e2e step time go? Times (cfg2, B=8 by default):
  step   : graph of the bare hybrid step, back-to-back replays, CUDA events
  loop_ev: DecodeLoop graph (H2D + append + step + D2H), back-to-back replays, CUDA events
  loop_wc: DecodeLoop.run() (replay + host sync) per step, wall clock
for overlap on/off.   python scripts/e2e_diag.py [--batch 8] [--steps 50]"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import DecodeLoop, HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
cfg = CONFIGS[a.config].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda", capacity=cfg.context)
dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)


def ev_time(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    dec.step(q, cfg.context)
torch.cuda.current_stream().wait_stream(s)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    dec.step(q, cfg.context)
res = {"step": ev_time(gr.replay, a.steps)}
for ov in (False, True):
    loop = DecodeLoop(dec, cfg.context - 1, zero_copy=ov)
    pos = cfg.context - 1
    loop.q_host.copy_(q.cpu())  # real inputs: all-zero queries would make every score tie
    loop.k_host.copy_(k[:, :, :, pos].cpu())
    loop.v_host.copy_(v[:, :, :, pos].cpu())
    loop.capture()
    res[f"loop_ev_overlap{int(ov)}"] = ev_time(loop.graph.replay, a.steps)
    for _ in range(3):
        loop.run()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        loop.run()
    res[f"loop_wc_overlap{int(ov)}"] = (time.perf_counter() - t0) / a.steps * 1e3
    # the same with a spin on an event instead of the blocking stream sync
    ev = torch.cuda.Event()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        loop.graph.replay()
        ev.record()
        while not ev.query():
            pass
    res[f"loop_wc_spin_overlap{int(ov)}"] = (time.perf_counter() - t0) / a.steps * 1e3
    # host-side cost of one replay call alone
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loop.graph.replay()
    res[f"replay_call_ms_overlap{int(ov)}"] = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    del loop
print({k_: round(v_, 4) for k_, v_ in res.items()})

# raw link: pinned H2D / D2H of the step's buffer sizes, and the append copies alone
L, B, Hq, d = q.shape
Hkv = k.shape[2]
out = {}
for name, nbytes in (("q", q.numel() * 2), ("kv_rows", 2 * L * B * Hkv * d * 2),
                     ("out_f32", L * B * Hq * d * 4)):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dv = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    t_h2d = ev_time(lambda: dv.copy_(h, non_blocking=True), 20)
    t_d2h = ev_time(lambda: h.copy_(dv, non_blocking=True), 20)
    out[name] = {"bytes": nbytes, "h2d_us": round(t_h2d * 1e3, 1), "d2h_us": round(t_d2h * 1e3, 1),
                 "h2d_gbs": round(nbytes / t_h2d / 1e6, 1), "d2h_gbs": round(nbytes / t_d2h / 1e6, 1)}
kvd = torch.zeros((2, L, B, Hkv, d), dtype=k.dtype, device="cuda")
pos = cfg.context - 1


def app():
    k[:, :, :, pos].copy_(kvd[0])
    v[:, :, :, pos].copy_(kvd[1])


out["append_us"] = round(ev_time(app, 20) * 1e3, 1)
print(out)
