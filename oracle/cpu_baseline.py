"""ORACLE-side CPU timing — test/bench infrastructure only (never the product path).

Times the reference algorithm, restated in numpy float64 (oracle/hylra_oracle.py, which
follows pkg/src/layerreuse/attention.py:185-275 and engine.py:167-197), on the host's
cores for one decode-step sample of a BASELINE config, and extrapolates to the whole
step. Run as a separate process WITHOUT torch so BLAS threading is not
disturbed:

    OPENBLAS_NUM_THREADS=<n> python -m oracle.cpu_baseline --config cfg2 --batch 8

Sample = one (sequence, KV-head) group: for each timed iteration one FULL layer (G x
full_attention + top-k of the head-summed logits) and one REUSE layer (G x
subset_attention over the inherited set); the float64 cache copies are built outside the
timer ("kernel-equivalent" time). Step time =
Hkv * B * (n_full * t_full + n_reuse * t_reuse); tok/s = B / step time.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS  # noqa: E402


def group_data(cfg, n_layers, seed=0):
    rng = np.random.default_rng(seed)
    G, d, N = cfg.group, cfg.head_dim, cfg.context
    data = []
    for _ in range(n_layers):
        q = rng.standard_normal((G, d))
        k = rng.standard_normal((N, d))
        v = rng.standard_normal((N, d))
        qh = q.mean(0)
        qh /= np.linalg.norm(qh)
        k[rng.choice(N, min(cfg.planted, N), replace=False)] += cfg.shift * qh
        data.append((q, np.ascontiguousarray(k), np.ascontiguousarray(v)))
    return data


def full_layer(q, k, v, budget):
    agg = np.zeros(k.shape[0])
    for g in range(q.shape[0]):
        _, logits = orc.full_attention(q[g], k, v)
        agg += logits
    return orc.topk_of_logits(agg, budget)


def reuse_layer(q, k, v, idx):
    for g in range(q.shape[0]):
        orc.subset_attention(q[g], k, v, idx)


def time_group(cfg, seconds: float, n_distinct: int = 2):
    data = group_data(cfg, n_distinct)
    t_full, t_reuse = [], []
    idx = full_layer(*data[0], cfg.budget)  # warm-up
    deadline = time.perf_counter() + seconds
    i = 0
    while time.perf_counter() < deadline or len(t_full) < 3:
        q, k, v = data[i % n_distinct]
        t0 = time.perf_counter()
        idx = full_layer(q, k, v, cfg.budget)
        t1 = time.perf_counter()
        q2, k2, v2 = data[(i + 1) % n_distinct]
        reuse_layer(q2, k2, v2, idx)
        t2 = time.perf_counter()
        t_full.append(t1 - t0)
        t_reuse.append(t2 - t1)
        i += 1
    return float(np.median(t_full)), float(np.median(t_reuse)), i


def baseline(cfg, batch: int, seconds: float) -> dict:
    tf, tr, iters = time_group(cfg, seconds)
    n_full = len(cfg.full_layers)
    n_reuse = cfg.layers - n_full
    step = cfg.kv_heads * batch * (n_full * tf + n_reuse * tr)
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    return {
        "value": batch / step,
        "unit": "tok/s",
        "cores": threads,
        "kind": "port",
        "sample": (f"{iters} iterations of one (sequence, KV-head) group: 1 FULL layer "
                   f"({cfg.group} x full_attention + top-{cfg.budget}) + 1 REUSE layer "
                   f"({cfg.group} x subset_attention) at N={cfg.context}, d={cfg.head_dim}; "
                   f"median t_full={tf * 1e3:.2f} ms, t_reuse={tr * 1e3:.2f} ms, extrapolated "
                   f"x{cfg.kv_heads * batch} groups x ({n_full} FULL + {n_reuse} REUSE) layers"),
        "step_seconds": step,
    }


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--seconds", type=float, default=10.0)
    a = ap.parse_args(argv)
    cfg = CONFIGS[a.config]
    print(json.dumps(baseline(cfg, a.batch or cfg.batch, a.seconds)))


if __name__ == "__main__":
    main()
