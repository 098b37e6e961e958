"""BASELINE config 5 decode sweep: context x top-k ratio x batch on the Llama-3-8B shape,
per-kernel times and HBM roofline fractions (FULL, SELECT, REUSE) + the whole step.

    python scripts/sweep.py [--quick] > sweep.jsonl

Layer count: the full 32-layer cfg2 policy when the KV cache fits in ~150 GB, else the
longest prefix of that policy that fits (at least [FULL, REUSE]); per-kernel fractions do
not depend on the layer count, and each line records the layers used. Lines run on a
prefix also carry the 32-layer step EXTRAPOLATED by layer count (`extrapolated_32_layers`,
with the factor and the reason), never as a measured value.

Times: per-kernel = mean of back-to-back launches between two CUDA events (device time per
launch, no host gaps); step = the autotuned schedule's CUDA-graph replay time (the eager
step, with its host overhead, is `step_ms_eager`).
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.attention import geometry, scores_row_stride  # noqa: E402
from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()
                  ).get("hbm_gbs", 6650.0) if (Path(__file__).resolve().parent.parent /
                                               "MEASURED_PEAKS.json").exists() else 6650.0
BUDGET_BYTES = 150e9


def time_ms(fn, reps=20):
    """Mean device time per launch of `reps` back-to-back launches."""
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def time_eager_ms(fn, reps=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for x, y in ev:
        x.record()
        fn()
        y.record()
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ev)


def point(N, ratio, B):
    base = CONFIGS["cfg2"]
    k = max(1, int(N * ratio))
    per_layer = B * base.kv_heads * N * base.head_dim * 2 * 2
    L = base.layers
    while L > 2 and L * per_layer > BUDGET_BYTES:
        L -= 1
    full = tuple(f for f in base.full_layers if f < L) or (0,)
    if L < 2 or per_layer * L > BUDGET_BYTES:
        return {"context": N, "top_k": k, "batch": B, "skipped": "KV does not fit one GPU"}
    cfg = base.with_(layers=L, context=N, budget=k, batch=B, full_layers=full)
    q, kk, vv = generate_torch(cfg, "cuda")
    dec = HybridDecoder(cfg.actions, kk, vv, k, q_heads=cfg.q_heads)
    tuned = dec.autotune(q, N)
    dec.step(q, N)
    torch.cuda.synchronize()
    dec.check_flags()
    g = geometry(q, kk, vv, dec.out)
    fl = [l for l in range(L) if cfg.actions[l] == "full"]
    rl = [l for l in range(L) if cfg.actions[l] == "reuse"]
    lib = _abi.lib()
    st = torch.cuda.current_stream().cuda_stream
    sc = torch.empty((len(fl), B, cfg.kv_heads, scores_row_stride(N)), dtype=torch.float32,
                     device="cuda")
    wsf = torch.zeros(lib.hylra_attention_workspace_bytes(g, len(fl), N), dtype=torch.uint8,
                      device="cuda")
    wsr = torch.zeros(max(256, lib.hylra_attention_workspace_bytes(g, max(1, len(rl)), min(k, N))),
                      dtype=torch.uint8, device="cuda")
    wss = torch.zeros(256, dtype=torch.uint8, device="cuda")
    fid, rid = _abi.int32_array(fl), _abi.int32_array(rl)
    rsrc = _abi.int32_array(dec.slot_of_layer[l] for l in rl)
    t_full = time_ms(lambda: _abi.check(lib.hylra_full_decode(
        g, q.data_ptr(), kk.data_ptr(), vv.data_ptr(), N, len(fl), fid, dec.out.data_ptr(),
        sc.data_ptr(), wsf.data_ptr(), wsf.numel(), st)))
    t_sel = time_ms(lambda: _abi.check(lib.hylra_topk_select(
        g, sc.data_ptr(), len(fl), N, k, 1, q.data_ptr(), kk.data_ptr(), fid, dec.idx.data_ptr(),
        dec.k_stride, None, wss.data_ptr(), wss.numel(), st)))
    t_reuse = time_ms(lambda: _abi.check(lib.hylra_reuse_decode(
        g, q.data_ptr(), kk.data_ptr(), vv.data_ptr(), N, len(rl), rid, rsrc, dec.idx.data_ptr(), None,
        dec.k_stride, min(k, N), 1, dec.out.data_ptr(), wsr.data_ptr(), wsr.numel(), st))) \
        if rl else 0.0
    t_eager = time_eager_ms(lambda: dec.step(q, N))
    t_step = tuned[dec.schedule]  # graph replay of the autotuned schedule
    fb = len(fl) * B * cfg.kv_heads * 2 * N * cfg.head_dim * 2
    rb = len(rl) * B * cfg.kv_heads * 2 * min(k, N) * cfg.head_dim * 2
    res = {"context": N, "top_k": k, "ratio": ratio, "batch": B, "layers": L,
           "schedule": dec.schedule, "autotune_ms": tuned,
           "full_layers": len(fl), "reuse_layers": len(rl),
           "full_ms": t_full, "select_ms": t_sel, "reuse_ms": t_reuse, "step_ms": t_step,
           "step_ms_eager": t_eager,
           "full_frac": fb / (t_full * 1e-3) / 1e9 / PEAK,
           "reuse_frac": (rb / (t_reuse * 1e-3) / 1e9 / PEAK) if rl else None,
           "select_frac_of_full_plus_select": t_sel / (t_full + t_sel),
           "step_gbs": (fb + rb) / (t_step * 1e-3) / 1e9,
           "tok_per_s_for_these_layers": B / (t_step * 1e-3)}
    if L < base.layers:
        f = base.layers / L
        res["extrapolated_32_layers"] = {
            "step_ms": t_step * f, "tok_per_s": B / (t_step * f * 1e-3), "factor": f,
            "by": "layer count (step time x 32 / layers run)",
            "why": f"32 layers of KV = {per_layer * base.layers / 1e9:.0f} GB > "
                   f"{BUDGET_BYTES / 1e9:.0f} GB on one GPU"}
    del q, kk, vv, dec, sc, wsf, wsr
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    ctxs = [8192, 32768, 131072, 262144]
    ratios = [1 / 64, 1 / 32, 1 / 16]
    batches = [1, 8, 32]
    if a.quick:
        ctxs, batches = [8192, 32768], [1, 8]
    for N in ctxs:
        for r in ratios:
            for B in batches:
                print(json.dumps(point(N, r, B)), flush=True)
