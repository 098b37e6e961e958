"""Host-side planning: the DP, validator, static policies and the similarity fold must be
bit-identical to the reference (policy.py, profiling.py)."""
import json

import numpy as np
import pytest

from oracle import hylra_oracle as orc
from paper_2602_00777_b200 import (Action, InvalidInputError, LayerPolicy, SimilarityMatrix,
                                   dp_optimize, merge_similarity_matrices, policy_from_actions,
                                   similarity_from_counts, static_jump_policy, validate_policy)


def random_matrix(rng, L, budget=8):
    v = np.zeros((L, L))
    for j in range(L):
        v[j, j] = 1.0
        for i in range(j):
            v[j, i] = float(rng.random())
    return SimilarityMatrix(values=v, budget=budget)


def test_dp_matches_reference_goldens(golden_dir):
    cases = json.loads((golden_dir / "dp_cases.json").read_text())
    for c in cases:
        m = SimilarityMatrix(values=np.array(c["values"]), budget=8)
        assert m.sha256() == c["matrix_sha"]
        for r in c["results"]:
            p = dp_optimize(m, r["theta"])
            assert [a.value for a in p.actions] == r["actions"]
            assert list(p.sources) == r["sources"]
            assert p.full_count == r["full_count"]
            assert p.cum_similarity == r["cum_similarity"]  # bit-identical credit
            assert p.sha256() == r["policy_sha"]


def test_dp_equals_exhaustive_search():
    # acceptance criterion 01 (tests/test_acceptance.py:34-56), against the oracle's
    # independent brute force; exact ties included via quantised matrices
    rng = np.random.default_rng(20240817)
    for trial in range(300):
        L = int(rng.integers(2, 9))
        m = random_matrix(rng, L)
        if trial % 3 == 0:
            v = np.round(m.values * 4) / 4
            np.fill_diagonal(v, 1.0)
            v[np.triu_indices(L, 1)] = 0.0
            m = SimilarityMatrix(values=v, budget=8)
        for theta in (0.0, 0.25, 0.5, 0.75, 1.0):
            fast = dp_optimize(m, theta)
            acts, srcs, fc, credit = orc.brute_force_dp(m.values, theta)
            assert tuple(a.value for a in fast.actions) == acts
            assert fast.sources == srcs
            assert fast.full_count == fc
            assert fast.cum_similarity == credit
            assert validate_policy(fast, m, theta) == []


def test_threshold_is_inclusive_and_monotone():
    for theta in (0.3, 0.5, 0.9):
        at = SimilarityMatrix(values=np.array([[1.0, 0.0], [theta, 1.0]]), budget=8)
        assert dp_optimize(at, theta).full_count == 1
        below = SimilarityMatrix(values=np.array([[1.0, 0.0], [theta - 1e-9, 1.0]]), budget=8)
        assert dp_optimize(below, theta).full_count == 2
    rng = np.random.default_rng(31)
    for _ in range(50):
        m = random_matrix(rng, 10)
        counts = [dp_optimize(m, t).full_count for t in [x / 10 for x in range(11)]]
        assert counts == sorted(counts)


def test_policy_examples():
    m = SimilarityMatrix(values=np.array([[1.0, 0, 0], [1.0, 1.0, 0], [1.0, 0.9, 1.0]]), budget=4)
    p = dp_optimize(m, 0.5)
    assert p.actions == (Action.FULL, Action.REUSE, Action.REUSE) and p.sources == (0, 0, 0)
    m = SimilarityMatrix(values=np.array([[1.0, 0, 0], [0.1, 1.0, 0], [0.1, 0.1, 1.0]]), budget=4)
    p = dp_optimize(m, 0.5)
    assert p.full_count == 3 and p.cum_similarity == 3.0
    with pytest.raises(InvalidInputError):
        dp_optimize(m, 1.5)


def test_validate_and_static_policies():
    s = static_jump_policy(7, 3)
    assert [a.value for a in s.actions] == ["full", "reuse", "reuse", "full", "reuse", "reuse",
                                            "full"]
    assert s.sources == (0, 0, 0, 3, 3, 3, 6)
    m = SimilarityMatrix(values=np.tril(np.full((3, 3), 0.5)) + np.eye(3) * 0.5, budget=4)
    bad = LayerPolicy((Action.REUSE, Action.FULL, Action.REUSE), (0, 1, 0), None, 1, None, None)
    v = validate_policy(bad, m, 0.4)
    assert (0, "first-layer-full") in v and (2, "source-not-full") in v
    chain = LayerPolicy((Action.FULL, Action.FULL, Action.REUSE), (0, 1, 0), None, 2, None, None)
    assert validate_policy(chain, m, 0.4) == [(2, "chain")]
    assert validate_policy(chain, m, 0.6) == [(2, "chain"), (2, "threshold")]
    p = policy_from_actions(["full", "reuse", "full", "reuse", "reuse"])
    assert p.sources == (0, 0, 2, 2, 2)
    with pytest.raises(InvalidInputError):
        LayerPolicy((Action.FULL,), (0,), None, 2, None, None)


def test_similarity_fold_matches_oracle_bitwise():
    rng = np.random.default_rng(4)
    for _ in range(20):
        T, L, k = int(rng.integers(1, 6)), int(rng.integers(2, 12)), int(rng.integers(1, 3000))
        c = rng.integers(0, k + 1, size=(T, L, L))
        got = similarity_from_counts(c, k).values
        want = orc.similarity_fold(c, k)
        assert np.array_equal(got, want)
    a = SimilarityMatrix(values=np.array([[1.0, 0], [0.5, 1.0]]), budget=2)
    b = SimilarityMatrix(values=np.array([[1.0, 0], [0.25, 1.0]]), budget=2)
    assert merge_similarity_matrices([a, b]).values[1, 0] == 0.375
    assert np.array_equal(merge_similarity_matrices([a, b]).values,
                          orc.merge_fold([a.values, b.values]))


def test_similarity_matrix_validation():
    with pytest.raises(InvalidInputError):
        SimilarityMatrix(values=np.array([[0.9]]), budget=1)
    with pytest.raises(InvalidInputError):
        SimilarityMatrix(values=np.array([[1.0, 0.1], [0.5, 1.0]]), budget=1)
    with pytest.raises(InvalidInputError):
        SimilarityMatrix(values=np.array([[1.0, 0.0], [1.5, 1.0]]), budget=1)
    with pytest.raises(InvalidInputError):
        similarity_from_counts(np.zeros((0, 2, 2)), 4)


def test_matrix_hash_matches_reference_fixture(golden_dir):
    from refmodel import load_npz
    z = load_npz(golden_dir / "fixture_engine.npz")
    m = SimilarityMatrix(values=z["matrix"], budget=int(z["budget"]))
    assert m.sha256() == str(z["matrix_sha"])
    p = dp_optimize(m, float(z["theta"]))
    assert p.sha256() == str(z["policy_sha"])


def test_brute_force_policy_matches_reference_goldens(golden_dir):
    """brute_force_policy (policy.py:226-270) against the reference's own exhaustive planner
    on random and exact-tie matrices (tests/golden/brute_force_cases.json), and against
    dp_optimize (acceptance criterion 01)."""
    from paper_2602_00777_b200 import brute_force_policy

    cases = json.loads((golden_dir / "brute_force_cases.json").read_text())
    assert len(cases) == 60
    for c in cases:
        m = SimilarityMatrix(values=np.array(c["values"]), budget=8)
        assert m.sha256() == c["matrix_sha"]
        for r in c["results"]:
            p = brute_force_policy(m, r["theta"])
            assert [a.value for a in p.actions] == r["actions"]
            assert list(p.sources) == r["sources"]
            assert p.full_count == r["full_count"]
            assert p.cum_similarity == r["cum_similarity"]
            assert p.sha256() == r["policy_sha"]
            assert dp_optimize(m, r["theta"]).sha256() == r["policy_sha"]


def test_brute_force_policy_refuses_large_stacks():
    from paper_2602_00777_b200 import BRUTE_FORCE_MAX_LAYERS, brute_force_policy

    L = BRUTE_FORCE_MAX_LAYERS + 1
    with pytest.raises(InvalidInputError):
        brute_force_policy(SimilarityMatrix(values=np.eye(L), budget=8), 0.5)
    with pytest.raises(InvalidInputError):
        brute_force_policy(SimilarityMatrix(values=np.eye(3), budget=8), 1.5)
