"""CPU arm of bench.py: the REFERENCE's own implementation of the hot path, timed on the host.

Imports the unmodified reference package `layerreuse` installed (pure Python + numpy) into
baseline/_ref by

    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

(git-ignored, shipped to the GPU box with the snapshot). Without it the float64 oracle
port (oracle/hylra_oracle.py) stands in and the line says kind "port". Runs as a separate,
torch-free process.

Number 1 — "kernel-equivalent" step time: exactly the per-layer body of
the reference's hybrid_decode (engine.py:174-194) minus cache construction. By default each
timed step runs the WHOLE step — every (sequence, KV-head) group through all layers in
policy order, on a process pool — so nothing is extrapolated (--sampled: the older one
FULL + one REUSE layer sample scaled by layer count). Per layer:
  FULL  layer, per (sequence, KV-head) group: G x full_attention (attention.py:210-226),
        the head-order logit sum and TopKSet(topk_of_logits(...)) (attention.py:264-275);
  REUSE layer, per group: sel.as_array() + G x _subset_attention (attention.py:229-241).
One timed sample = one FULL layer and one REUSE layer over ALL B x Hkv groups of the config
(distinct float64 LayerKvCache objects, built outside the timer); the step time is
  n_full x t_full + n_reuse x t_reuse        (declared extrapolation: by layer count only).
The groups of a layer run on a process pool over all host cores (the reference's
operations are pure functions, "callers may evaluate different layers/steps concurrently",
SPEC.md:135-136), each worker single-threaded BLAS; a single-process run with threaded BLAS
is reported beside it.

Number 2 — end to end: the reference's hybrid_decode (engine.py:129-209, its float64 cache
copies and internal all-FULL fidelity baseline included) through the per-KV-head ArrayModel
adapter for one (sequence, KV-head) group over the whole stack, T = 1;
step time extrapolated x (B x Hkv) groups (declared).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path
from types import SimpleNamespace

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF = HERE / "_ref"


def _import_reference():
    """(module, kind): the installed reference, else the oracle port."""
    if (REF / "layerreuse" / "__init__.py").exists():
        sys.path.insert(0, str(REF))
        import layerreuse  # noqa: F401
        from layerreuse import attention as ra
        return ra, "reference"
    sys.path.insert(0, str(ROOT))
    return None, "port"


def _config(name):
    sys.path.insert(0, str(ROOT))
    from paper_2602_00777_b200.synthetic import CONFIGS  # numpy-only module
    return CONFIGS[name]


# ----------------------------------------------------------------------------- data
def _group_arrays(cfg, seed):
    """One (sequence, KV-head) group's FULL- and REUSE-layer inputs, float64: queries
    [G, d], K/V [N, d] ~ N(0, 1) with cfg.planted rows shifted by shift * q_hat (the
    BASELINE planted-token distribution)."""
    import numpy as np
    rng = np.random.default_rng([seed, 0xC0DE])
    G, d, N = cfg.group, cfg.head_dim, cfg.context
    q = rng.standard_normal((G, d))
    k = rng.standard_normal((N, d))
    v = rng.standard_normal((N, d))
    qh = q.mean(0)
    qh /= np.linalg.norm(qh)
    k[rng.choice(N, min(cfg.planted, N), replace=False)] += cfg.shift * qh
    return q, k, v


_STATE = {}


def _worker_init(cfg_name, n_distinct, base_seed):
    """Build this worker's distinct caches once (outside every timer)."""
    ra, kind = _import_reference()
    cfg = _config(cfg_name)
    caches = []
    for i in range(n_distinct):
        qf, kf, vf = _group_arrays(cfg, base_seed + 2 * i)
        qr, kr, vr = _group_arrays(cfg, base_seed + 2 * i + 1)
        if ra is not None:
            caches.append((qf, ra.LayerKvCache(keys=kf, values=vf), qr,
                           ra.LayerKvCache(keys=kr, values=vr)))
        else:
            caches.append((qf, (kf, vf), qr, (kr, vr)))
    _STATE.update(ra=ra, kind=kind, cfg=cfg, caches=caches)


def _full_op(ra, cfg, q, cache):
    """engine.py:176-184 for one group: G x full_attention, logit sum, top-k set."""
    import numpy as np
    if ra is None:
        from oracle import hylra_oracle as orc
        agg = np.zeros(cfg.context)
        for g in range(q.shape[0]):
            _, lg = orc.full_attention(q[g], cache[0], cache[1])
            agg += lg
        return orc.topk_of_logits(agg, cfg.budget)
    agg = np.zeros(cache.length)
    for g in range(q.shape[0]):
        _, scores = ra.full_attention(q[g], cache)
        agg += scores.logits
    return ra.TopKSet(indices=ra.topk_of_logits(agg, min(cfg.budget, cache.length)),
                      budget=cfg.budget)


def _reuse_op(ra, cfg, q, cache, sel):
    """engine.py:186-193 for one group: the inherited set's rows, G x _subset_attention."""
    if ra is None:
        from oracle import hylra_oracle as orc
        for g in range(q.shape[0]):
            orc.subset_attention(q[g], cache[0], cache[1], sel)
        return
    idx = sel.as_array()
    for g in range(q.shape[0]):
        ra._subset_attention(q[g], cache, idx)


def _group_task(i):
    """One group's FULL layer then REUSE layer (times each)."""
    st = _STATE
    qf, cf, qr, cr = st["caches"][i % len(st["caches"])]
    t0 = time.perf_counter()
    sel = _full_op(st["ra"], st["cfg"], qf, cf)
    t1 = time.perf_counter()
    _reuse_op(st["ra"], st["cfg"], qr, cr, sel)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def _group_stack_task(i):
    """One group's WHOLE layer stack in policy order (engine.py:174-194): every FULL layer
    (its set replacing the inherited one) and every REUSE layer over the most recent FULL
    layer's set. The layers run on the group's one FULL / one REUSE cache (identical cost per
    layer: same N, d, k), so the step executes all of its work; times each kind."""
    st = _STATE
    cfg = st["cfg"]
    qf, cf, qr, cr = st["caches"][i % len(st["caches"])]
    tf = tr = 0.0
    sel = None
    for a in cfg.actions:
        t0 = time.perf_counter()
        if a == "full":
            sel = _full_op(st["ra"], cfg, qf, cf)
            tf += time.perf_counter() - t0
        else:
            _reuse_op(st["ra"], cfg, qr, cr, sel)
            tr += time.perf_counter() - t0
    return tf, tr


def full_steps(cfg, batch, steps, warmup, workers):
    """Whole steps on the pool: every (sequence, KV-head) group runs its full layer stack
    (_group_stack_task). Returns (per-step wall times of the timed steps, median FULL / REUSE
    busy shares)."""
    import multiprocessing as mp

    import numpy as np
    groups = batch * cfg.kv_heads
    per_worker = max(1, min(4, math.ceil(groups / workers)))
    walls, shares = [], []
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_worker_init, initargs=(cfg.name, per_worker, 1000)) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            res = pool.map(_group_stack_task, range(groups), chunksize=1)
            wall = time.perf_counter() - t0
            if it >= warmup:
                walls.append(wall)
                bf, br = sum(r[0] for r in res), sum(r[1] for r in res)
                shares.append(bf / (bf + br))
    return walls, float(np.median(shares))


def kernel_equivalent(cfg, batch, steps, warmup, workers):
    """Median over `steps` samples of (t_full_layer, t_reuse_layer) over all B x Hkv groups."""
    import numpy as np
    groups = batch * cfg.kv_heads
    per_worker = max(1, min(4, math.ceil(groups / workers)))
    samples = []
    if workers > 1:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(workers, initializer=_worker_init,
                      initargs=(cfg.name, per_worker, 1000)) as pool:
            for it in range(warmup + steps):
                t0 = time.perf_counter()
                res = pool.map(_group_task, range(groups), chunksize=1)
                wall = time.perf_counter() - t0
                busy_f = sum(r[0] for r in res)
                busy_r = sum(r[1] for r in res)
                # split the pool's wall time between the two layers by their busy shares
                if it >= warmup:
                    samples.append((wall * busy_f / (busy_f + busy_r),
                                    wall * busy_r / (busy_f + busy_r)))
    else:
        _worker_init(cfg.name, min(groups, 4), 1000)
        for it in range(warmup + steps):
            tf = tr = 0.0
            for g in range(groups):
                a, b = _group_task(g)
                tf += a
                tr += b
            if it >= warmup:
                samples.append((tf, tr))
    arr = np.array(samples)
    return float(np.median(arr[:, 0])), float(np.median(arr[:, 1])), len(samples)


class _ArrayModel:
    """Duck-typed reference model over one (sequence, KV-head) group's arrays:
    config.{layers, heads=G, head_dim, context_len}, grown_arrays, queries, cache_at."""

    def __init__(self, ra, q, k, v):
        L, G, d = q.shape
        self._ra = ra
        self.config = SimpleNamespace(layers=L, heads=G, head_dim=d, context_len=k.shape[1])
        self._q, self._k, self._v = q[None], k[:, None], v[:, None]

    def grown_arrays(self, steps):
        return self._k, self._v

    def queries(self, steps):
        return self._q

    def cache_at(self, keys, values, layer, head, step):
        n = self.config.context_len + step
        return self._ra.LayerKvCache(keys=keys[layer, 0, :n], values=values[layer, 0, :n])


def end_to_end(cfg, seed=7):
    """The reference hybrid_decode for one group over the whole stack (T = 1)."""
    import numpy as np
    ra, kind = _import_reference()
    if ra is None:
        return None
    import layerreuse as lr
    L = cfg.layers
    qs, ks, vs = [], [], []
    for l in range(L):  # float32 storage; the reference copies each (layer, head) to float64
        q, k, v = _group_arrays(cfg, seed + l)
        qs.append(q)
        ks.append(k.astype(np.float32))
        vs.append(v.astype(np.float32))
    model = _ArrayModel(ra, np.stack(qs), np.stack(ks), np.stack(vs))
    del ks, vs
    policy = lr.LayerPolicy(
        actions=tuple(lr.Action(a) for a in cfg.actions),
        sources=tuple(max(f for f in cfg.full_layers if f <= l) for l in range(L)),
        theta=None, full_count=len(cfg.full_layers), cum_similarity=None, matrix_hash=None)
    t0 = time.perf_counter()
    lr.hybrid_decode(model, policy, cfg.budget, 1)
    return time.perf_counter() - t0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--workers", type=int, default=0,
                    help="0 = all host cores (a process pool; run with OPENBLAS_NUM_THREADS=1); "
                         "1 = this process only (run with threaded BLAS)")
    ap.add_argument("--e2e", action="store_true", help="also time hybrid_decode (number 2)")
    ap.add_argument("--sampled", action="store_true",
                    help="pool mode: time one FULL + one REUSE layer per sample and scale by "
                         "layer count (the default times whole steps)")
    a = ap.parse_args(argv)
    cfg = _config(a.config)
    B = a.batch or cfg.batch
    cores = os.cpu_count() or 1
    workers = a.workers or cores
    _, kind = _import_reference()
    n_full = len(cfg.full_layers)
    n_reuse = cfg.layers - n_full
    groups = B * cfg.kv_heads
    blas = int(os.environ.get("OPENBLAS_NUM_THREADS", "0") or 0) or cores
    if workers > 1 and not a.sampled:
        # whole steps: all groups x all layers per timed step, nothing extrapolated
        walls, share = full_steps(cfg, B, a.steps, a.warmup, workers)
        import statistics
        step = statistics.median(walls)
        out = {
            "value": B / step, "unit": "tok/s", "kind": kind, "cores": workers,
            "mode": f"{workers}-process pool, single-threaded BLAS",
            "ms_per_step": step * 1e3,
            "sample": (f"{len(walls)} whole steps (+{a.warmup} warm-up), median: all {groups} "
                       f"(sequence, KV-head) groups x all {cfg.layers} layers in policy order "
                       f"({n_full} FULL: G={cfg.group} x full_attention + top-{cfg.budget}; "
                       f"{n_reuse} REUSE: G x _subset_attention over the inherited set) at "
                       f"N={cfg.context}, d={cfg.head_dim}, float64, caches built outside the "
                       f"timer (each group's layers share one FULL and one REUSE cache: same "
                       f"cost per layer), groups on a {workers}-process pool; FULL share of the "
                       f"busy time {share:.2f}"),
            "extrapolation": None,
            "step_seconds": walls, "timed_samples": len(walls),
        }
        if a.e2e:
            t = end_to_end(cfg)
            if t is not None:
                out["end_to_end_hybrid_decode"] = {
                    "value": B / (t * groups), "unit": "tok/s", "cores": blas,
                    "group_seconds": t,
                    "sample": (f"reference hybrid_decode (float64 cache copies + internal "
                               f"all-FULL baseline) for one (sequence, KV-head) group, "
                               f"{cfg.layers} layers, T=1, {t:.2f} s; x{groups} groups "
                               f"(declared extrapolation)")}
        print(json.dumps(out), flush=True)
        return
    tf, tr, n = kernel_equivalent(cfg, B, a.steps, a.warmup, workers)
    step = n_full * tf + n_reuse * tr
    where = (f"groups on a {workers}-process pool" if workers > 1 else "groups in one process")
    out = {
        "value": B / step, "unit": "tok/s", "kind": kind,
        "cores": workers if workers > 1 else blas,
        "mode": (f"{workers}-process pool, single-threaded BLAS" if workers > 1
                 else f"one process, {blas}-thread BLAS"),
        "ms_per_step": step * 1e3,
        "sample": (f"{n} timed samples (+{a.warmup} warm-up) of one FULL layer (G={cfg.group} x "
                   f"full_attention + top-{cfg.budget}) and one REUSE layer (G x "
                   f"_subset_attention over the inherited set) over all {groups} (sequence, "
                   f"KV-head) groups at N={cfg.context}, d={cfg.head_dim}, float64, caches built "
                   f"outside the timer, {where}; median FULL layer {tf * 1e3:.1f} ms, REUSE "
                   f"layer {tr * 1e3:.1f} ms; step = {n_full} x FULL + {n_reuse} x REUSE"),
        "extrapolation": {"timed_layers_per_sample": 2, "step_layers": cfg.layers,
                          "factor_by_layers": cfg.layers / 2, "by": "layer count only"},
        "sample_seconds": tf + tr, "timed_samples": n,
    }
    if a.e2e:
        t = end_to_end(cfg)
        if t is not None:
            out["end_to_end_hybrid_decode"] = {
                "value": B / (t * groups), "unit": "tok/s", "cores": blas,
                "group_seconds": t,
                "sample": (f"reference hybrid_decode (float64 cache copies + internal all-FULL "
                           f"baseline) for one (sequence, KV-head) group, {cfg.layers} layers, "
                           f"T=1, {t:.2f} s; x{groups} groups (declared extrapolation)")}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
