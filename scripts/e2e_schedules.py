"""End-to-end step (DecodeLoop: pinned host I/O, one graph launch + host sync per step) for
every schedule the decoder supports, at a config/batch: wall clock per step, interleaved.
    python scripts/e2e_schedules.py [--config cfg2] [--batch 1]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import DecodeLoop, HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
cfg = CONFIGS[a.config].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
pos = cfg.context - 1
loops = {}
for name in ("dual", "fusedsel", "fused3", "single", "singlecoop"):
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    try:
        dec.set_schedule(name)
    except Exception as e:  # noqa: BLE001
        print(name, "n/a:", e)
        continue
    loop = DecodeLoop(dec, pos)
    loop.q_host.copy_(q.cpu())
    loop.k_host.copy_(k[:, :, :, pos].cpu())
    loop.v_host.copy_(v[:, :, :, pos].cpu())
    loop.capture()
    loops[name] = loop
res = {n: [] for n in loops}
for _ in range(3):
    for n, loop in loops.items():
        for _ in range(5):
            loop.run()
        t0 = time.perf_counter()
        for _ in range(50):
            loop.run()
        res[n].append((time.perf_counter() - t0) / 50 * 1e6)
print(f"{a.config} B={a.batch} e2e us/step: " +
      " | ".join(f"{n} {min(t):.1f} (q_copy {loops[n].q_copy})" for n, t in res.items()))
