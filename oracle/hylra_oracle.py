"""ORACLE — test infrastructure only. CPU float64 restatement of the reference path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module, and only as the checker (or the timed CPU arm). The product path
(paper_2602_00777_b200) never imports it.

Restates, in numpy float64, the reference package `layerreuse` (pkg/src/layerreuse/):
  softmax            attention.py:185-194
  full_attention     attention.py:210-226  (logits = K q / sqrt(d); w = softmax; out = w V)
  subset_attention   attention.py:229-241  (gather, subset-renormalised softmax)
  topk_of_logits     attention.py:264-275  (stable argsort of -logits: ties -> lower index;
                                            result ascending)
  hybrid step        engine.py:167-197     (FULL: per-head attention + head-order logit sum
                                            + top-min(budget, n); REUSE: previous selection)
  overlap / fold     profiling.py:38-47, 126-145, 148-163
  brute-force DP     policy.py:226-270     (exhaustive search with the reference tie order)
extended to GQA the way SURVEY.md §0.2 / §8c define it: query head h reads KV head
h // G, and one selection set is made per group of `sel_group` KV heads by summing the
logits of all query heads of the group in head order (sel_group = Hkv reproduces the
reference's layer-wide set).

Pinned against the reference's own golden vectors and against outputs of the reference
itself run in the build container (tests/golden/make_golden.py, committed fixtures under
tests/golden/, checked by tests/test_oracle.py).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

__all__ = [
    "softmax", "full_attention", "subset_attention", "topk_of_logits", "group_scores",
    "hybrid_step", "hybrid_replay", "overlap_counts", "similarity_fold", "merge_fold",
    "brute_force_dp",
]


def softmax(logits):
    """attention.py:185-194."""
    x = np.asarray(logits, dtype=np.float64)
    e = np.exp(x - x.max())
    return e / e.sum()


def full_attention(q, keys, values):
    """attention.py:210-226 -> (output [d], logits [N])."""
    q = np.asarray(q, dtype=np.float64)
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    logits = keys @ q / math.sqrt(keys.shape[1])
    return softmax(logits) @ values, logits


def subset_attention(q, keys, values, idx):
    """attention.py:229-241 -> output [d] over rows idx only."""
    idx = np.asarray(idx, dtype=np.int64)
    sub_k = np.asarray(keys, dtype=np.float64)[idx]
    sub_v = np.asarray(values, dtype=np.float64)[idx]
    logits = sub_k @ np.asarray(q, dtype=np.float64) / math.sqrt(sub_k.shape[1])
    return softmax(logits) @ sub_v


def topk_of_logits(logits, budget: int) -> np.ndarray:
    """attention.py:264-275: min(budget, N) highest, ties to lower index, ascending."""
    x = np.asarray(logits, dtype=np.float64)
    take = min(int(budget), x.shape[0])
    order = np.argsort(-x, kind="stable")[:take]
    return np.sort(order)


def group_scores(q_l, k_l, n_valid: int, G: int, sel_group: int):
    """Selection scores of one layer: q_l [B, Hq, d], k_l [B, Hkv, N, d] ->
    [B, Hkv/sel_group, n_valid], agg = 0 then += logits of each query head of the group
    in head order (engine.py:177-181)."""
    B, Hq, d = q_l.shape
    Hkv = k_l.shape[1]
    groups = Hkv // sel_group
    out = np.zeros((B, groups, n_valid))
    for b in range(B):
        for grp in range(groups):
            agg = np.zeros(n_valid)
            for kh in range(grp * sel_group, (grp + 1) * sel_group):
                K = np.asarray(k_l[b, kh, :n_valid], dtype=np.float64)
                for g in range(G):
                    qv = np.asarray(q_l[b, kh * G + g], dtype=np.float64)
                    agg += K @ qv / math.sqrt(d)
            out[b, grp] = agg
    return out


def hybrid_step(q, k, v, n_valid: int, actions, budget: int, sel_group: int = 1,
                layers=None, want_scores: bool = False):
    """One decode step of Algorithm 2 over a GQA stack (engine.py:167-197).

    q [L, B, Hq, d]; k, v [L, B, Hkv, >= n_valid, d]; actions: sequence of "full"/"reuse".
    Returns (outputs [L, B, Hq, d] float64, sets {layer: int64 [B, groups, k_eff]} for every
    layer — a REUSE layer maps to its source's array object —, scores {full layer: ...}).
    `layers` restricts the computed layers (others are left NaN) for large inputs.
    """
    L, B, Hq, d = q.shape
    Hkv = k.shape[2]
    G = Hq // Hkv
    groups = Hkv // sel_group
    b_t = min(budget, n_valid)
    todo = set(range(L)) if layers is None else set(layers)
    out = np.full((L, B, Hq, d), np.nan)
    sets, scores = {}, {}
    sel = None
    for l in range(L):
        act = actions[l] if isinstance(actions[l], str) else actions[l].value
        if act == "full":
            need_sel = any(l2 in todo for l2 in range(l, L))
            if l in todo:
                for b in range(B):
                    for h in range(Hq):
                        o, _ = full_attention(q[l, b, h], k[l, b, h // G, :n_valid],
                                              v[l, b, h // G, :n_valid])
                        out[l, b, h] = o
            if need_sel:
                sc = group_scores(q[l], k[l], n_valid, G, sel_group)
                sel = np.stack([np.stack([topk_of_logits(sc[b, grp], b_t)
                                          for grp in range(groups)]) for b in range(B)])
                if want_scores:
                    scores[l] = sc
        else:
            if sel is None:
                raise ValueError("the first layer of a policy must run full attention")
            if l in todo:
                for b in range(B):
                    for h in range(Hq):
                        kh = h // G
                        out[l, b, h] = subset_attention(q[l, b, h], k[l, b, kh, :n_valid],
                                                        v[l, b, kh, :n_valid],
                                                        sel[b, kh // sel_group])
        sets[l] = sel
    return out, sets, scores


def hybrid_replay(queries, keys, values, actions, budget: int, context_len: int):
    """Reference-model replay (engine.py:129-209 without the fidelity baseline):
    queries [T, L, H, d], grown keys/values [L, H, N+T, d], MHA heads sharing one
    layer-wide selection. Returns (outputs [T, L, H, d], sets [T][L] int64 arrays)."""
    T = queries.shape[0]
    L, H = keys.shape[0], keys.shape[1]
    outs, all_sets = [], []
    for t in range(T):
        n_t = context_len + t
        q = np.asarray(queries[t])[:, None]                    # [L, 1, H, d]
        k = np.asarray(keys)[:, None]                          # [L, 1, H, N+T, d]
        v = np.asarray(values)[:, None]
        o, sets, _ = hybrid_step(q, k, v, n_t, actions, budget, sel_group=H)
        outs.append(o[:, 0])
        all_sets.append([sets[l][0, 0] for l in range(L)])
    return np.stack(outs), all_sets


def overlap_counts(sets_per_step) -> np.ndarray:
    """|S_i & S_j| for every step and layer pair (profiling.py:38-47): [T, L, L]."""
    T = len(sets_per_step)
    L = len(sets_per_step[0])
    c = np.zeros((T, L, L), dtype=np.int64)
    for t in range(T):
        ss = [set(int(x) for x in s) for s in sets_per_step[t]]
        for j in range(L):
            for i in range(L):
                c[t, j, i] = len(ss[i] & ss[j])
    return c


def similarity_fold(counts, k: int) -> np.ndarray:
    """profiling.py:139-145: per-step |S_i & S_j| / k below the diagonal, mean over steps,
    zero above the diagonal, unit diagonal."""
    counts = np.asarray(counts)
    T, L, _ = counts.shape
    per_step = np.ones((T, L, L))
    for t in range(T):
        for j in range(L):
            for i in range(j):
                per_step[t, j, i] = int(counts[t, j, i]) / k
    values = per_step.mean(axis=0)
    values[np.triu_indices(L, k=1)] = 0.0
    np.fill_diagonal(values, 1.0)
    return values


def merge_fold(values_list) -> np.ndarray:
    """profiling.py:148-163."""
    v = np.stack(values_list).mean(axis=0)
    np.fill_diagonal(v, 1.0)
    return v


def brute_force_dp(values, theta: float):
    """Exhaustive planner with the reference objective and tie order (policy.py:226-270):
    minimise FULL count, then maximise credit accumulated in ascending layer order, then
    compare sources from the last layer down preferring the smaller.
    Returns (actions tuple of "full"/"reuse", sources tuple, full_count, credit)."""
    M = np.asarray(values, dtype=np.float64)
    L = M.shape[0]
    best_key, best = None, None
    for tail in itertools.product(("full", "reuse"), repeat=L - 1):
        acts = ("full",) + tail
        src = [0] * L
        credit, fulls, ok = 1.0, 1, True
        for j in range(1, L):
            if acts[j] == "full":
                src[j] = j
                fulls += 1
                credit += 1.0
            else:
                src[j] = src[j - 1]
                m = float(M[j, src[j]])
                if m < theta:
                    ok = False
                    break
                credit += m
        if not ok:
            continue
        key = (fulls, -credit, tuple(reversed(src)))
        if best_key is None or key < best_key:
            best_key, best = key, (acts, tuple(src), fulls, credit)
    return best


# ----------------------------------------------------------------------------- blocks
def block_max_of_logits(logits, block_size: int) -> np.ndarray:
    """attention.py:287-295: max-pool into ceil(N / block_size) block scores."""
    x = np.asarray(logits, dtype=np.float64)
    return np.maximum.reduceat(x, np.arange(0, x.shape[0], block_size))


def block_coverage(blocks, block_size: int, n: int) -> np.ndarray:
    """attention.py:166-182 BlockSet.token_coverage: ascending tokens of the selected blocks,
    the final block truncated at n."""
    return np.concatenate([np.arange(b * block_size, min((b + 1) * block_size, n))
                           for b in blocks]).astype(np.int64)


def hybrid_step_blocks(q, k, v, n_valid: int, actions, block_budget: int, block_size: int,
                       sel_group: int = 1):
    """Block-mode decode step (engine.py:212-286): FULL layers keep the top
    min(block_budget, n_blocks) blocks of the max-pooled head-summed logits (ties -> lower
    block, ascending); REUSE layers attend over the inherited blocks' token coverage.
    Returns (outputs [L, B, Hq, d], blocks {layer: int64 [B, groups, bb]})."""
    L, B, Hq, d = q.shape
    Hkv = k.shape[2]
    G = Hq // Hkv
    groups = Hkv // sel_group
    nb = -(-n_valid // block_size)
    bb = min(block_budget, nb)
    out = np.zeros((L, B, Hq, d))
    blocks, sel = {}, None
    for l in range(L):
        act = actions[l] if isinstance(actions[l], str) else actions[l].value
        if act == "full":
            for b in range(B):
                for h in range(Hq):
                    out[l, b, h], _ = full_attention(q[l, b, h], k[l, b, h // G, :n_valid],
                                                     v[l, b, h // G, :n_valid])
            sc = group_scores(q[l], k[l], n_valid, G, sel_group)
            sel = np.stack([np.stack([topk_of_logits(block_max_of_logits(sc[b, g], block_size), bb)
                                      for g in range(groups)]) for b in range(B)])
        else:
            for b in range(B):
                for h in range(Hq):
                    kh = h // G
                    cov = block_coverage(sel[b, kh // sel_group], block_size, n_valid)
                    out[l, b, h] = subset_attention(q[l, b, h], k[l, b, kh, :n_valid],
                                                    v[l, b, kh, :n_valid], cov)
        blocks[l] = sel
    return out, blocks
