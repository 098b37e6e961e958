"""Generate the committed golden fixtures from the REFERENCE itself (build container only).

Run from the repo root:  python tests/golden/make_golden.py
It imports the read-only reference package from /root/reference/pkg/src (pure Python +
numpy), runs it on small seeded inputs and writes its outputs under tests/golden/. The
GPU box never runs this script (the reference tree does not exist there); tests consume
the committed .npz / .json files.

Fixtures
  fixture_engine.npz   reference tests/test_engine.py:24-32 FIXTURE (L6 d32 N96 seed21
                       rho0.85 H1, trace T=3 k=12, theta=0.6): model arrays, trace sets,
                       matrix, DP policy, hybrid outputs, fidelity aggregate (golden
                       1.1709555430500145).
  fixture_overlap.npz  tests/test_synthetic.py:15-17,121-127 (L8 d32 N256 seed11 rho0.9,
                       T=4 k=32): arrays, trace sets, matrix (adjacent golden 0.9084821...).
  mha_reference.npz    H=2 multi-head model (layer-wide selection over both heads), T=2.
  cfg1_reference.npz   BASELINE config 1 (planted generator of this repo, fp32 values):
                       the reference run once per (batch, KV head) through the duck-typed
                       ArrayModel adapter of SURVEY.md §8c: outputs, per-FULL-layer sets
                       and the summed logits.
  topk_cases.json      topk_of_logits on random, tied and saturated logit vectors.
  dp_cases.json        dp_optimize on random similarity matrices x theta grid.
  brute_force_cases.json  brute_force_policy (policy.py:226-270) on random and quantised
                       (exact-tie) matrices up to 12 layers x theta grid.
  artifacts/           versioned JSON artifacts WRITTEN BY THE REFERENCE (formats.py) for an
                       H=2 model (L6 d32 N96 seed21 rho0.85): decode-trace (+ sidecars,
                       block_size 4), similarity-matrix, layer-policy, decode-run (token and
                       block mode), cost-report, sensitivity-report.
  artifacts_reference.npz  the same model's arrays, the sensitivity probe noise, both hybrid
                       runs' outputs/selections and the reference fidelity_report values.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import layerreuse as lr  # noqa: E402
from layerreuse.attention import LayerKvCache  # noqa: E402

from paper_2602_00777_b200.synthetic import CONFIGS, generate_numpy  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sets_array(sets_2d):
    return np.array([[list(s.indices) for s in row] for row in sets_2d], dtype=np.int64)


def engine_fixture():
    cfg = lr.SynthModelConfig(layers=6, head_dim=32, context_len=96, seed=21,
                              inter_layer_correlation=0.85, heads=1)
    model = lr.generate_model(cfg)
    keys, values = model.grown_arrays(3)
    queries = model.queries(3)
    trace = lr.run_full_trace(model, 3, 12)
    matrix = lr.build_similarity_matrix(trace)
    policy = lr.dp_optimize(matrix, 0.6)
    run = lr.hybrid_decode(model, policy, 12, 3)
    np.savez_compressed(
        HERE / "fixture_engine.npz", keys=keys, values=values, queries=queries,
        trace_sets=sets_array(trace.topk), trace_outputs=trace.outputs,
        matrix=matrix.values, matrix_sha=np.array(matrix.sha256()),
        actions=np.array([a.value for a in policy.actions]),
        sources=np.array(policy.sources), full_count=policy.full_count,
        cum_similarity=policy.cum_similarity, policy_sha=np.array(policy.sha256()),
        outputs=run.outputs, run_sets=sets_array(run.selections),
        aggregate=run.fidelity.aggregate, per_step_layer=run.fidelity.per_step_layer,
        context_len=96, budget=12, theta=0.6)
    print("engine fixture: actions", [a.value for a in policy.actions], "agg",
          repr(run.fidelity.aggregate))


def overlap_fixture():
    cfg = lr.SynthModelConfig(layers=8, head_dim=32, context_len=256, seed=11,
                              inter_layer_correlation=0.9)
    model = lr.generate_model(cfg)
    keys, values = model.grown_arrays(4)
    queries = model.queries(4)
    trace = lr.run_full_trace(model, 4, 32)
    matrix = lr.build_similarity_matrix(trace)
    adjacent = float(np.mean([matrix.values[j, j - 1] for j in range(1, 8)]))
    np.savez_compressed(HERE / "fixture_overlap.npz", keys=keys, values=values,
                        queries=queries, trace_sets=sets_array(trace.topk),
                        matrix=matrix.values, matrix_sha=np.array(matrix.sha256()),
                        adjacent=adjacent, context_len=256, budget=32)
    print("overlap fixture: adjacent", repr(adjacent))


def block_fixture():
    """tests/test_engine.py:34-38,196-206 BLOCK_FIXTURE (L5 d32 N512 seed33 rho0.8 H2):
    block mode, static_jump_policy(5, 2), 2 blocks of 128, 2 steps; golden aggregate
    0.4524886792120594."""
    cfg = lr.SynthModelConfig(layers=5, head_dim=32, context_len=512, seed=33,
                              inter_layer_correlation=0.8, heads=2)
    model = lr.generate_model(cfg)
    keys, values = model.grown_arrays(2)
    queries = model.queries(2)
    policy = lr.static_jump_policy(5, 2)
    run = lr.hybrid_decode_blocks(model, policy, 2, 128, 2)
    blocks = np.array([[list(s.block_indices) for s in row] for row in run.selections])
    gathered = np.array([[-1 if g is None else g for g in row] for row in run.reuse_gathered_rows])
    np.savez_compressed(HERE / "block_reference.npz", keys=keys, values=values, queries=queries,
                        actions=np.array([a.value for a in policy.actions]),
                        outputs=run.outputs, blocks=blocks, gathered=gathered,
                        aggregate=run.fidelity.aggregate, context_len=512, block_budget=2,
                        block_size=128)
    print("block fixture: agg", repr(run.fidelity.aggregate))


def mha_fixture():
    cfg = lr.SynthModelConfig(layers=4, head_dim=32, context_len=128, seed=5,
                              inter_layer_correlation=0.7, heads=2)
    model = lr.generate_model(cfg)
    keys, values = model.grown_arrays(2)
    queries = model.queries(2)
    policy = lr.static_jump_policy(4, 2)
    run = lr.hybrid_decode(model, policy, 16, 2)
    np.savez_compressed(HERE / "mha_reference.npz", keys=keys, values=values, queries=queries,
                        actions=np.array([a.value for a in policy.actions]),
                        outputs=run.outputs, run_sets=sets_array(run.selections),
                        aggregate=run.fidelity.aggregate, context_len=128, budget=16)
    print("mha fixture: agg", repr(run.fidelity.aggregate))


class ArrayModel:
    """Duck-typed reference model over one (batch, KV head) slice of a GQA stack."""

    def __init__(self, q, k, v, b, kh, G):
        L, _, _, N, d = k.shape
        self.config = SimpleNamespace(layers=L, heads=G, head_dim=d, context_len=N)
        self._k = np.asarray(k[:, b, kh], dtype=np.float64)[:, None]   # [L, 1, N, d]
        self._v = np.asarray(v[:, b, kh], dtype=np.float64)[:, None]
        self._q = np.asarray(q[:, b, kh * G:(kh + 1) * G], dtype=np.float64)[None]  # [1, L, G, d]

    def grown_arrays(self, steps):
        assert steps == 1
        return self._k, self._v

    def queries(self, steps):
        assert steps == 1
        return self._q

    def cache_at(self, keys, values, layer, head, step):
        n = self.config.context_len + step
        return LayerKvCache(keys=keys[layer, 0, :n], values=values[layer, 0, :n])


def cfg1_fixture():
    cfg = CONFIGS["cfg1"]
    q, k, v = generate_numpy(cfg)
    L, B, Hq, d = q.shape
    Hkv, G = cfg.kv_heads, cfg.group
    policy = lr.LayerPolicy(
        actions=tuple(lr.Action(a) for a in cfg.actions),
        sources=tuple(max(f for f in cfg.full_layers if f <= l) for l in range(L)),
        theta=None, full_count=len(cfg.full_layers), cum_similarity=None, matrix_hash=None)
    outputs = np.zeros((L, B, Hq, d))
    sets = np.zeros((len(cfg.full_layers), B, Hkv, cfg.budget), dtype=np.int64)
    scores = np.zeros((len(cfg.full_layers), B, Hkv, cfg.context))
    for b in range(B):
        for kh in range(Hkv):
            m = ArrayModel(q, k, v, b, kh, G)
            run = lr.hybrid_decode(m, policy, cfg.budget, 1)
            outputs[:, b, kh * G:(kh + 1) * G] = run.outputs[0]
            for s, l in enumerate(cfg.full_layers):
                sets[s, b, kh] = run.selections[0][l].indices
                agg = np.zeros(cfg.context)
                for g in range(G):
                    _, sc = lr.full_attention(m._q[0, l, g], m.cache_at(m._k, m._v, l, g, 0))
                    agg += sc.logits
                scores[s, b, kh] = agg
    np.savez_compressed(HERE / "cfg1_reference.npz", outputs=outputs, sets=sets, scores=scores,
                        input_sha=np.array(sha(q, k, v)))
    print("cfg1 fixture: input sha", sha(q, k, v)[:16])


def topk_cases():
    rng = np.random.default_rng(7)
    cases = [([3.0, 1.0, 2.0], 2), ([5.0, 5.0, 5.0], 2), ([1.0, 2.0], 10)]
    for _ in range(150):
        n = int(rng.integers(1, 300))
        if rng.random() < 0.4:
            x = rng.integers(-3, 4, size=n).astype(float)  # heavy ties
        else:
            x = rng.standard_normal(n)
        cases.append((x.tolist(), int(rng.integers(1, n + 4))))
    out = [{"logits": x, "budget": b, "expected": list(lr.topk_of_logits(np.array(x), b))}
           for x, b in cases]
    (HERE / "topk_cases.json").write_text(json.dumps(out))
    print("topk cases:", len(out))


def dp_cases():
    rng = np.random.default_rng(20240817)
    out = []
    for _ in range(120):
        L = int(rng.integers(2, 13))
        vals = np.zeros((L, L))
        for j in range(L):
            vals[j, j] = 1.0
            for i in range(j):
                vals[j, i] = float(rng.random())
        m = lr.SimilarityMatrix(values=vals, budget=8)
        res = []
        for theta in (0.0, 0.3, 0.5, 0.7, 0.9, 1.0):
            p = lr.dp_optimize(m, theta)
            res.append({"theta": theta, "actions": [a.value for a in p.actions],
                        "sources": list(p.sources), "full_count": p.full_count,
                        "cum_similarity": p.cum_similarity, "policy_sha": p.sha256()})
        out.append({"values": vals.tolist(), "matrix_sha": m.sha256(), "results": res})
    (HERE / "dp_cases.json").write_text(json.dumps(out))
    print("dp matrices:", len(out))


def brute_force_cases():
    rng = np.random.default_rng(7031)
    out = []
    for trial in range(60):
        L = int(rng.integers(2, 13))
        vals = np.zeros((L, L))
        for j in range(L):
            vals[j, j] = 1.0
            for i in range(j):
                vals[j, i] = float(rng.random())
        if trial % 2 == 0:  # exact ties
            vals = np.round(vals * 4) / 4
            np.fill_diagonal(vals, 1.0)
            vals[np.triu_indices(L, 1)] = 0.0
        m = lr.SimilarityMatrix(values=vals, budget=8)
        res = []
        for theta in (0.0, 0.25, 0.5, 0.75, 1.0):
            p = lr.brute_force_policy(m, theta)
            res.append({"theta": theta, "actions": [a.value for a in p.actions],
                        "sources": list(p.sources), "full_count": p.full_count,
                        "cum_similarity": p.cum_similarity, "policy_sha": p.sha256()})
        out.append({"values": vals.tolist(), "matrix_sha": m.sha256(), "results": res})
    (HERE / "brute_force_cases.json").write_text(json.dumps(out))
    print("brute-force matrices:", len(out))


def artifacts_fixture():
    from layerreuse import formats as fm
    from layerreuse.synthetic import _S_PROBE, _rng

    adir = HERE / "artifacts"
    adir.mkdir(exist_ok=True)
    cfg = lr.SynthModelConfig(layers=6, head_dim=32, context_len=96, seed=21,
                              inter_layer_correlation=0.85, heads=2)
    model = lr.generate_model(cfg)
    T, k, bs = 3, 12, 4
    keys, values = model.grown_arrays(T)
    queries = model.queries(T)
    trace = lr.run_full_trace(model, T, k, block_size=bs)
    fm.write_trace(trace, str(adir / "trace.json"))
    matrix = lr.build_similarity_matrix(trace)
    fm.write_similarity_matrix(matrix, str(adir / "matrix.json"))
    policy = lr.dp_optimize(matrix, 0.6)
    fm.write_policy(policy, str(adir / "policy.json"))
    run = lr.hybrid_decode(model, policy, k, T)
    fm.write_run_result(run, str(adir / "run.json"))
    runb = lr.hybrid_decode_blocks(model, policy, 3, bs, T)
    fm.write_run_result(runb, str(adir / "run_blocks.json"))
    cost = lr.cost_model(policy, 32768, 2048, head_dim=1024, bytes_per_elem=2)
    fm.write_cost_report(cost, str(adir / "cost.json"), contextLen=32768, budget=2048)
    costb = lr.cost_model(policy, 1000, 7, block_size=128, head_dim=64)
    fm.write_cost_report(costb, str(adir / "cost_blocks.json"))
    sens_step = 1
    sens = lr.sensitivity_profile(model, sens_step, k)
    fm.write_sensitivity_report(sens, str(adir / "sensitivity.json"))
    probe = np.stack([np.stack([_rng(cfg.seed, _S_PROBE, nl, h, sens_step).standard_normal(32)
                                for h in range(2)]) for nl in range(7)])
    fid = lr.fidelity_report(trace, run)
    fidb = lr.fidelity_report(trace, runb)
    np.savez_compressed(
        HERE / "artifacts_reference.npz", keys=keys, values=values, queries=queries,
        probe=probe, sens_step=sens_step, rho=0.85, context_len=96, budget=k, block_size=bs,
        run_outputs=run.outputs, run_sets=sets_array(run.selections),
        runb_outputs=runb.outputs,
        runb_blocks=np.array([[list(s.block_indices) for s in row] for row in runb.selections]),
        fid_overlap=fid.selection_overlap, fid_per_layer=fid.per_layer_overlap,
        fid_rnmse=fid.rnmse.per_step_layer, fid_aggregate=fid.rnmse.aggregate,
        fidb_overlap=fidb.selection_overlap, fidb_rnmse=fidb.rnmse.per_step_layer,
        sens_rnmse=sens.rnmse, sens_kl=sens.kl)
    print("artifacts: policy", [a.value for a in policy.actions], "sens", sens.rnmse)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # named fixtures only, e.g. `make_golden.py brute_force_cases`
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    engine_fixture()
    overlap_fixture()
    mha_fixture()
    block_fixture()
    cfg1_fixture()
    topk_cases()
    dp_cases()
    brute_force_cases()
    artifacts_fixture()
