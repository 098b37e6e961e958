"""Split-K sizing sweep for the FULL and REUSE launches (B200).

    python scripts/split_sweep.py            # driver: one subprocess per knob setting
    python scripts/split_sweep.py --worker   # one measurement (knobs from the environment)

Knobs (read once by libhylra.so): HYLRA_{FULL,REUSE}_WAVES, HYLRA_{FULL,REUSE}_MIN_TILES.
Worker: cfg2 shapes, B in {1, 4, 8}; REUSE over all 24 REUSE layers and over a 5-layer
chunk, FULL over the 8 FULL layers; CUDA-event mean of 20 launches each."""
import itertools
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def worker():
    import torch

    from paper_2602_00777_b200 import _abi
    from paper_2602_00777_b200.attention import geometry, scores_row_stride
    from paper_2602_00777_b200.engine import HybridDecoder
    from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch

    lib = _abi.lib()
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    N = int(os.environ.get("SWEEP_N", CONFIGS["cfg2"].context))
    K = int(os.environ.get("SWEEP_K", CONFIGS["cfg2"].budget))
    for B in [int(x) for x in os.environ.get("SWEEP_B", "1,4,8").split(",")]:
        cfg = CONFIGS["cfg2"].with_(batch=B, context=N, budget=K)
        q, k, v = generate_torch(cfg, "cuda")
        dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
        dec.step(q, cfg.context)
        torch.cuda.synchronize()
        g = geometry(q, k, v, dec.out)
        rl = [l for l in range(cfg.layers) if cfg.actions[l] == "reuse"]
        fl = [l for l in range(cfg.layers) if cfg.actions[l] == "full"]
        ke = min(cfg.budget, cfg.context)
        need = max(lib.hylra_attention_workspace_bytes(g, n, r)
                   for n, r in ((len(rl), ke), (5, ke), (len(fl), cfg.context)))
        ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
        scores = torch.empty((len(fl), B, cfg.kv_heads, scores_row_stride(cfg.context)),
                             dtype=torch.float32, device="cuda")

        def reuse(layers):
            src = [dec.slot_of_layer[l] for l in layers]
            _abi.check(lib.hylra_reuse_decode(g, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                              cfg.context, len(layers), _abi.int32_array(layers),
                                              _abi.int32_array(src), dec.idx.data_ptr(), None,
                                              dec.k_stride, ke, 1, dec.out.data_ptr(),
                                              ws.data_ptr(), ws.numel(), st))

        def full():
            _abi.check(lib.hylra_full_decode(g, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             cfg.context, len(fl), _abi.int32_array(fl),
                                             dec.out.data_ptr(), scores.data_ptr(), ws.data_ptr(),
                                             ws.numel(), st))

        def t(fn, n=20):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n * 1e3

        row = 2 * ke * cfg.head_dim * 2 * B * cfg.kv_heads  # bytes per REUSE layer
        fl_bytes = len(fl) * B * cfg.kv_heads * 2 * cfg.context * cfg.head_dim * 2
        t24 = t(lambda: reuse(rl))
        t5 = t(lambda: reuse(rl[:5]))
        tf = t(full)
        fb = fl_bytes
        res[f"B{B}"] = {"reuse24_us": round(t24, 1), "reuse24_gbs": round(24 * row / t24 / 1e3),
                        "reuse5_us": round(t5, 1), "reuse5_gbs": round(5 * row / t5 / 1e3),
                        "full_us": round(tf, 1), "full_gbs": round(fb / tf / 1e3)}
        del q, k, v, dec, ws, scores
        torch.cuda.empty_cache()
    print(json.dumps(res))


def driver():
    settings = [{}] if os.environ.get("SWEEP_DEFAULT", "1") == "1" else []
    waves = [int(x) for x in os.environ.get("SWEEP_WAVES", "1,2,3,4,8").split(",")]
    tiles = [int(x) for x in os.environ.get("SWEEP_TILES", "2,4,8,16").split(",")]
    for w, mt in itertools.product(waves, tiles):
        settings.append({"HYLRA_REUSE_WAVES": str(w), "HYLRA_REUSE_MIN_TILES": str(mt),
                         "HYLRA_FULL_WAVES": str(w), "HYLRA_FULL_MIN_TILES": str(mt)})
    for s in settings:
        env = dict(os.environ, **s)
        r = subprocess.run([sys.executable, __file__, "--worker"], env=env, capture_output=True,
                           text=True, timeout=300)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(json.dumps(s), line, flush=True)


if __name__ == "__main__":
    worker() if "--worker" in sys.argv else driver()
