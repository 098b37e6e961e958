"""e2e (DecodeLoop, host I/O incl. index sets) vs the device-only graph-replayed step:
    python scripts/e2e_check.py [batch ...]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import DecodeLoop, HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

for B in [int(x) for x in sys.argv[1:]] or [1, 8]:
    cfg = CONFIGS["cfg2"].with_(batch=B)
    q, k, v = generate_torch(cfg, "cuda")
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    dec.autotune(q, cfg.context)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cfg.context)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        dec.step(q, cfg.context)
    for _ in range(5):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    e1.synchronize()
    dev = e0.elapsed_time(e1) / 50
    pos = cfg.context - 1
    res = {}
    for qc in (False, True):
        loop = DecodeLoop(dec, pos, q_copy=qc)
        loop.q_host.copy_(q.cpu())
        loop.capture()
        for _ in range(5):
            loop.run()
        t0 = time.perf_counter()
        for _ in range(50):
            loop.run()
        res[qc] = (time.perf_counter() - t0) / 50 * 1e3
        del loop
    print(f"B={B} schedule={dec.schedule}: device step {dev:.3f} ms; e2e q in place "
          f"{res[False]:.3f} ms, q copied {res[True]:.3f} ms", flush=True)
    del dec, q, k, v, g
    torch.cuda.empty_cache()
