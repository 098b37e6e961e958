"""A/B of the standalone selects on real score rows: the shared-memory-resident rowsel
(rowsel.cuh) against the streaming select_row (select.cuh), float64 refinement on, on an idle
GPU (CUDA-event time of one hylra_topk_select launch, mean of reps), plus the equality check.
    python scripts/select_ab.py [cfg2:1,8] [cfg3:4] ...   (rows = FULL layers x B x Hkv)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.attention import full_attention, geometry, topk_select  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / reps * 1e3


for arg in sys.argv[1:] or ["cfg2:1,8", "cfg3:4", "cfg4:16"]:
    name, bs = arg.split(":")
    for B in (int(x) for x in bs.split(",")):
        cfg = CONFIGS[name].with_(batch=B)
        q, k, v = generate_torch(cfg, "cuda")
        fl = [l for l, a in enumerate(cfg.actions) if a == "full"]
        for nl in (1, len(fl)):
            layers = fl[:nl]
            _, sc = full_attention(q, k, v, cfg.context, layers=layers)
            kw = dict(q=q, k=k, layers=layers)
            g = geometry(q, k, v)
            idx = torch.empty((nl, B, cfg.kv_heads, cfg.budget), dtype=torch.int32,
                              device="cuda")
            ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
            ids = _abi.int32_array(layers)
            st = torch.cuda.current_stream().cuda_stream

            def launch():  # the C ABI directly: no host work inside the timed region
                _abi.check(_abi.lib().hylra_topk_select(
                    g, sc.data_ptr(), nl, cfg.context, cfg.budget, 1, q.data_ptr(),
                    k.data_ptr(), ids, idx.data_ptr(), cfg.budget, None, ws.data_ptr(),
                    ws.numel(), st))
            res = {}
            for csz in (1, 2, 4, 8):
                with _abi.tuning(rowsel=1, rowsel_cluster=csz):
                    t = timed(launch)
                print(f"{name} B={B} layers={nl} rowsel cluster>={csz}: {t:.1f} us", flush=True)
            for impl, knob in (("rowsel", 1), ("stream", 0)):
                with _abi.tuning(rowsel=knob):
                    res[impl] = topk_select(sc, cfg.budget, cfg.context, **kw)
                    t = timed(launch)
                print(f"{name} B={B} layers={nl} rows={nl * B * cfg.kv_heads} {impl}: "
                      f"{t:.1f} us", flush=True)
            print(f"  equal: {torch.equal(res['rowsel'], res['stream'])}", flush=True)
            with _abi.tuning(rowsel=1):
                _, inf = topk_select(sc, cfg.budget, cfg.context, info=True, **kw)
            inf = inf.reshape(-1, 8).cpu()
            print("  rowsel info [k, nw, mode, C, cyc load, cyc minmax+hist, cyc band+T+window, "
                  "cyc compaction] first rows:", inf[:3].tolist(), flush=True)
            with _abi.tuning(rowsel=0):
                _, inf = topk_select(sc, cfg.budget, cfg.context, info=True, **kw)
            print("  stream info [k, nw, mode, cin, cyc A, B, C+D, E]:",
                  inf.reshape(-1, 8)[:3].tolist(), flush=True)
            del sc
        del q, k, v
        torch.cuda.empty_cache()
