"""Pin the float64 oracle against the reference's own golden vectors and against outputs
of the reference itself (committed fixtures made by tests/golden/make_golden.py)."""
import hashlib
import json
import math

import numpy as np
import pytest

from oracle import hylra_oracle as orc
from refmodel import load_npz


def test_known_answers_from_reference_tests():
    # tests/test_attention.py:33-59 (single token, orthogonal query, two-token fixture)
    out, logits = orc.full_attention([0.5, 0.5], [[1.0, 2.0]], [[5.0, -3.0]])
    assert np.array_equal(out, np.array([5.0, -3.0]))
    out, logits = orc.full_attention([0.0, 1.0], [[1.0, 0.0], [2.0, 0.0], [-1.0, 0.0]],
                                     [[3.0, 0.0], [0.0, 3.0], [0.0, 0.0]])
    assert np.allclose(out, [1.0, 1.0], atol=1e-15)
    out, logits = orc.full_attention([1.0, 0.0], [[10.0, 0.0], [0.0, 0.0]], [[1.0, 0.0], [0.0, 1.0]])
    assert logits[0] == pytest.approx(10 / math.sqrt(2), rel=1e-15)
    w1 = 1.0 / (1.0 + math.exp(-10 / math.sqrt(2)))
    assert out == pytest.approx([w1, 1 - w1], rel=1e-12)
    # subset fixture tests/test_attention.py:192-200
    keys = [[10.0, 0.0], [0.0, 0.0], [1.0, 1.0], [-2.0, 0.5]]
    values = [[1.0, 0.0], [0.0, 1.0], [2.0, 2.0], [3.0, -1.0]]
    got = orc.subset_attention([1.0, 0.0], keys, values, [0, 2])
    l0, l2 = 10 / math.sqrt(2), 1 / math.sqrt(2)
    w0 = 1 / (1 + math.exp(l2 - l0))
    assert got == pytest.approx([w0 * 1 + (1 - w0) * 2, (1 - w0) * 2], rel=1e-12)
    # top-k ties and saturation tests/test_attention.py:100-105
    assert list(orc.topk_of_logits([3.0, 1.0, 2.0], 2)) == [0, 2]
    assert list(orc.topk_of_logits([5.0, 5.0, 5.0], 2)) == [0, 1]
    assert list(orc.topk_of_logits([1.0, 2.0], 10)) == [0, 1]


def test_topk_cases_match_reference(golden_dir):
    cases = json.loads((golden_dir / "topk_cases.json").read_text())
    for c in cases:
        assert list(orc.topk_of_logits(c["logits"], c["budget"])) == c["expected"]


def test_engine_fixture_golden(golden_dir):
    z = load_npz(golden_dir / "fixture_engine.npz")
    # the reference's frozen goldens (tests/test_engine.py:30-32)
    assert tuple(z["actions"]) == ("full", "reuse", "reuse", "full", "reuse", "reuse")
    assert tuple(z["sources"]) == (0, 0, 0, 3, 3, 3)
    assert float(z["aggregate"]) == pytest.approx(1.1709555430500145, rel=1e-12)
    N, k, T = int(z["context_len"]), int(z["budget"]), 3
    # all-FULL trace: sets and outputs
    full = ("full",) * 6
    outs, sets = orc.hybrid_replay(z["queries"], z["keys"], z["values"], full, k, N)
    np.testing.assert_allclose(outs, z["trace_outputs"], rtol=1e-12, atol=1e-15)
    assert np.array_equal(np.array([[list(s) for s in row] for row in sets]), z["trace_sets"])
    # similarity fold is bit-identical, DP (exhaustive) reproduces the golden policy
    values = orc.similarity_fold(orc.overlap_counts(sets), k)
    assert np.array_equal(values, z["matrix"])
    acts, srcs, fc, credit = orc.brute_force_dp(values, float(z["theta"]))
    assert acts == tuple(z["actions"]) and srcs == tuple(z["sources"])
    assert fc == int(z["full_count"]) and credit == float(z["cum_similarity"])
    # hybrid replay under the golden policy, and the fidelity aggregate
    hyb, hsets = orc.hybrid_replay(z["queries"], z["keys"], z["values"], tuple(z["actions"]), k, N)
    np.testing.assert_allclose(hyb, z["outputs"], rtol=1e-12, atol=1e-15)
    assert np.array_equal(np.array([[list(s) for s in row] for row in hsets]), z["run_sets"])
    table = np.array([[np.linalg.norm(hyb[t, l].ravel() - outs[t, l].ravel())
                       / np.linalg.norm(outs[t, l].ravel()) for l in range(6)] for t in range(T)])
    assert float(table.mean()) == pytest.approx(1.1709555430500145, rel=1e-12)


def test_overlap_fixture_golden(golden_dir):
    z = load_npz(golden_dir / "fixture_overlap.npz")
    N, k = int(z["context_len"]), int(z["budget"])
    _, sets = orc.hybrid_replay(z["queries"], z["keys"], z["values"], ("full",) * 8, k, N)
    assert np.array_equal(np.array([[list(s) for s in row] for row in sets]), z["trace_sets"])
    values = orc.similarity_fold(orc.overlap_counts(sets), k)
    assert np.array_equal(values, z["matrix"])
    adjacent = float(np.mean([values[j, j - 1] for j in range(1, 8)]))
    assert adjacent == pytest.approx(0.9084821428571429, rel=1e-12)  # tests/test_synthetic.py:127


def test_mha_fixture_layer_wide_selection(golden_dir):
    z = load_npz(golden_dir / "mha_reference.npz")
    outs, sets = orc.hybrid_replay(z["queries"], z["keys"], z["values"], tuple(z["actions"]),
                                   int(z["budget"]), int(z["context_len"]))
    np.testing.assert_allclose(outs, z["outputs"], rtol=1e-12, atol=1e-15)
    assert np.array_equal(np.array([[list(s) for s in row] for row in sets]), z["run_sets"])


def test_cfg1_gqa_adapter_golden(golden_dir):
    from paper_2602_00777_b200.synthetic import CONFIGS, generate_numpy
    cfg = CONFIGS["cfg1"]
    q, k, v = generate_numpy(cfg)
    h = hashlib.sha256()
    for a in (q, k, v):
        h.update(np.ascontiguousarray(a).tobytes())
    z = load_npz(golden_dir / "cfg1_reference.npz")
    assert h.hexdigest() == str(z["input_sha"]), "planted generator drifted"
    out, sets, scores = orc.hybrid_step(q.astype(np.float64), k.astype(np.float64),
                                        v.astype(np.float64), cfg.context, cfg.actions,
                                        cfg.budget, want_scores=True)
    np.testing.assert_allclose(out, z["outputs"], rtol=1e-12, atol=1e-14)
    for s, l in enumerate(cfg.full_layers):
        assert np.array_equal(sets[l], z["sets"][s])
        np.testing.assert_allclose(scores[l], z["scores"][s], rtol=1e-12, atol=1e-12)


def test_block_mode_golden(golden_dir):
    """Block-level selection (engine.py:212-286) vs the reference's BLOCK_FIXTURE run:
    golden aggregate 0.4524886792120594 (tests/test_engine.py:34-38,196-206)."""
    z = load_npz(golden_dir / "block_reference.npz")
    assert float(z["aggregate"]) == pytest.approx(0.4524886792120594, rel=1e-12)
    N, bb, bs = int(z["context_len"]), int(z["block_budget"]), int(z["block_size"])
    acts = tuple(z["actions"])
    for t in range(2):
        n_t = N + t
        q = np.asarray(z["queries"][t])[:, None]
        k = np.asarray(z["keys"])[:, None]
        v = np.asarray(z["values"])[:, None]
        H = k.shape[2]
        out, blocks = orc.hybrid_step_blocks(q, k, v, n_t, acts, bb, bs, sel_group=H)
        np.testing.assert_allclose(out[:, 0], z["outputs"][t], rtol=1e-12, atol=1e-14)
        for l in range(len(acts)):
            assert list(blocks[l][0, 0]) == list(z["blocks"][t][l])
            if acts[l] == "reuse":
                cov = orc.block_coverage(blocks[l][0, 0], bs, n_t)
                assert cov.shape[0] == int(z["gathered"][t][l])
    # reference known answers (tests/test_attention.py:245-270)
    assert list(orc.block_max_of_logits([1.0, 9.0, 2.0, 3.0], 2)) == [9.0, 3.0]
    assert list(orc.block_max_of_logits([1.0, 9.0, 2.0], 8)) == [9.0]
    assert list(orc.topk_of_logits(np.array([0.5, 3.0, 1.0]), 2)) == [1, 2]
    assert list(orc.block_coverage([0, 2], 4, 10)) == [0, 1, 2, 3, 8, 9]
