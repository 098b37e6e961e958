"""Oracle check of a whole decode step at BASELINE sizes (test helper; GPU tests only).

For every (layer, b, kv-head) pair of a step: a FULL pair's index set must equal the
float64 oracle's top-k of the head-summed logits exactly (orc.group_scores +
orc.topk_of_logits, engine.py:177-183 / attention.py:264-275), and its output for one query
head (rotating with the pair) must lie within the bf16 tolerance of orc.full_attention
(attention.py:210-226); a REUSE pair's output for one query head must lie within tolerance
of orc.subset_attention over its inherited set (attention.py:229-241). The oracle reads the
exact stored (bf16) values. Pairs are checked on a thread pool: the per-pair work is a
device-to-host copy and numpy float64 BLAS, both of which release the GIL.
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from oracle import hylra_oracle as orc


def rel(x, r):
    return float(np.linalg.norm(x - r) / np.linalg.norm(r))


def check_step(q, k, v, n_valid, actions, budget, outputs, selections, slot_of_layer,
               tol=2e-2, all_heads_pairs=4, workers=16):
    """q [L,B,Hq,d] (device), k/v [L,B,Hkv,cap,d] (device, after the step), outputs
    [L,B,Hq,d] fp32 and selections [n_full,B,Hkv,k] (device or host). Returns a summary
    dict; raises AssertionError on the first mismatch."""
    L, B, Hq, d = q.shape
    Hkv = k.shape[2]
    G = Hq // Hkv
    k_eff = min(budget, n_valid)
    sel_host = selections.cpu().numpy() if hasattr(selections, "cpu") else np.asarray(selections)
    out_host = outputs.cpu().numpy() if hasattr(outputs, "cpu") else np.asarray(outputs)
    q_host = q.double().cpu().numpy()
    full_layers = [l for l in range(L) if actions[l] == "full"]
    jobs = []
    for l in range(L):
        for b in range(B):
            for h in range(Hkv):
                jobs.append((l, b, h))

    def head_list(l, b, h, idx):
        # one query head per pair (rotating), every head for the first few pairs
        return range(G) if idx < all_heads_pairs else [(l + b + h) % G]

    def run(job_i):
        l, b, h = jobs[job_i]
        slot = slot_of_layer[l]
        qn = q_host[l, b, h * G:(h + 1) * G]
        errs = []
        if actions[l] == "full":
            kn = k[l, b, h, :n_valid].double().cpu().numpy()
            vn = v[l, b, h, :n_valid].double().cpu().numpy()
            sc = orc.group_scores(qn[None], kn[None, None], n_valid, G, 1)[0, 0]
            want = orc.topk_of_logits(sc, budget)
            got = sel_host[slot, b, h, :k_eff]
            assert np.array_equal(got, want), (
                f"FULL set mismatch at layer {l} b {b} kv head {h}: "
                f"{int(np.sum(~np.isin(got, want)))} of {k_eff} indices differ")
            for g in head_list(l, b, h, job_i):
                ref, _ = orc.full_attention(qn[g], kn, vn)
                errs.append(rel(out_host[l, b, h * G + g].astype(np.float64), ref))
        else:
            idx = torch.as_tensor(sel_host[slot, b, h, :k_eff].astype(np.int64), device=k.device)
            kn = k[l, b, h].index_select(0, idx).double().cpu().numpy()
            vn = v[l, b, h].index_select(0, idx).double().cpu().numpy()
            ar = np.arange(k_eff)
            for g in head_list(l, b, h, job_i):
                ref = orc.subset_attention(qn[g], kn, vn, ar)
                errs.append(rel(out_host[l, b, h * G + g].astype(np.float64), ref))
        worst = max(errs)
        assert worst < tol, f"output error {worst:.3e} at layer {l} b {b} kv head {h}"
        return worst

    with ThreadPoolExecutor(max_workers=workers) as ex:
        worst = list(ex.map(run, range(len(jobs))))
    n_full = sum(1 for (l, _, _) in jobs if actions[l] == "full")
    return {"pairs": len(jobs), "full_pairs_sets_exact": n_full,
            "max_rel_err": max(worst), "full_layers": full_layers,
            "tol": tol, "k_eff": k_eff, "scale": 1 / math.sqrt(d)}
