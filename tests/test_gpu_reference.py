"""GPU parity against the reference's own goldens (committed fixtures made by running the
reference) through the drop-in entry points, and at the BASELINE configs' full sizes
against the float64 oracle on sampled rows.

Tolerances: outputs 1e-3 relative L2 per (b, head) for fp32 inputs, 2e-2 for bf16 inputs
(north_star); index sets, similarity matrices and DP policies exactly equal.
"""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import dp_optimize, policy_from_actions  # noqa: E402
from paper_2602_00777_b200.engine import (HybridDecoder, build_similarity_matrix,  # noqa: E402
                                          hybrid_decode, run_full_trace)
from paper_2602_00777_b200.profiling import (merge_similarity_matrices,  # noqa: E402
                                             overlap_counts, similarity_from_counts)
from paper_2602_00777_b200.synthetic import (CONFIGS, generate_numpy,  # noqa: E402
                                             generate_torch)
from refmodel import FixtureModel, load_npz  # noqa: E402


def rel(x, r):
    return float(np.linalg.norm(x - r) / np.linalg.norm(r))


def sets_of(sel):
    return np.array([[list(s.indices) for s in row] for row in sel])


def test_engine_fixture_drop_in(golden_dir):
    """tests/test_engine.py FIXTURE: trace -> GPU overlap matrix -> DP -> hybrid decode."""
    z = load_npz(golden_dir / "fixture_engine.npz")
    model = FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]))
    trace = run_full_trace(model, 3, int(z["budget"]))
    assert np.array_equal(sets_of(trace.topk), z["trace_sets"])
    np.testing.assert_allclose(trace.outputs, z["trace_outputs"], rtol=1e-4, atol=1e-5)
    matrix = build_similarity_matrix(trace)          # OVERLAP kernel + reference fold
    assert np.array_equal(matrix.values, z["matrix"])  # bit-identical
    assert matrix.sha256() == str(z["matrix_sha"])
    policy = dp_optimize(matrix, float(z["theta"]))
    assert tuple(a.value for a in policy.actions) == tuple(z["actions"])
    assert policy.sources == tuple(z["sources"])
    run = hybrid_decode(model, policy, int(z["budget"]), 3)
    assert np.array_equal(sets_of(run.selections), z["run_sets"])
    for t in range(3):  # REUSE layers share their source's selection object
        for l, src in enumerate(policy.sources):
            assert run.selections[t][l] is run.selections[t][src]
    for t in range(3):
        for l in range(6):
            assert rel(run.outputs[t, l, 0], z["outputs"][t, l, 0]) < 1e-3
    assert run.fidelity.aggregate == pytest.approx(1.1709555430500145, rel=1e-3)
    assert run.reuse_full_scans == 0
    assert run.full_score_computations == (policy.full_count,) * 3


def test_overlap_fixture_golden(golden_dir):
    """tests/test_synthetic.py golden adjacent overlap 0.9084821428571429 (L8 N256 k32 T4)."""
    z = load_npz(golden_dir / "fixture_overlap.npz")
    model = FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]))
    trace = run_full_trace(model, 4, int(z["budget"]))
    assert np.array_equal(sets_of(trace.topk), z["trace_sets"])
    m = build_similarity_matrix(trace)
    assert np.array_equal(m.values, z["matrix"])
    assert float(np.mean([m.values[j, j - 1] for j in range(1, 8)])) == \
        pytest.approx(0.9084821428571429, rel=1e-12)


def test_multi_head_layer_wide_selection(golden_dir):
    """H=2 heads sharing one set per layer (sel_group = Hkv, engine.py:177-183)."""
    z = load_npz(golden_dir / "mha_reference.npz")
    model = FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]))
    run = hybrid_decode(model, policy_from_actions(tuple(z["actions"])), int(z["budget"]), 2)
    assert np.array_equal(sets_of(run.selections), z["run_sets"])
    assert max(rel(run.outputs[t, l, h], z["outputs"][t, l, h]) for t in range(2)
               for l in range(4) for h in range(2)) < 1e-3
    assert run.fidelity.aggregate == pytest.approx(float(z["aggregate"]), rel=1e-3)


def test_config1_against_reference_outputs(golden_dir):
    """BASELINE config 1 (fp32, GQA 8/2, d64, N2048, k128): the reference's own outputs."""
    cfg = CONFIGS["cfg1"]
    q, k, v = generate_numpy(cfg)
    z = load_npz(golden_dir / "cfg1_reference.npz")
    dec = HybridDecoder(cfg.actions, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                        cfg.budget, q_heads=cfg.q_heads)
    res = dec.step(torch.from_numpy(q).cuda(), cfg.context)
    torch.cuda.synchronize()
    out = res.outputs.double().cpu().numpy()
    assert max(rel(out[l, 0, h], z["outputs"][l, 0, h]) for l in range(cfg.layers)
               for h in range(cfg.q_heads)) < 1e-3
    sel = res.selections.cpu().numpy()
    assert np.array_equal(sel, z["sets"])


def _check_rows(cfg, q, k, v, res, rows, n):
    """Oracle (float64 on the exact stored values) for sampled (layer, b, kv head) rows."""
    G = cfg.group
    for (l, b, h) in rows:
        qn = q[l, b].double().cpu().numpy()
        kn = k[l, b, h, :n].double().cpu().numpy()
        vn = v[l, b, h, :n].double().cpu().numpy()
        slot = res.slot_of_layer[l]
        src = cfg.full_layers[slot]
        got = res.selections[slot, b, h].cpu().numpy()
        if src == l:
            sc = np.zeros(n)
            for g in range(G):
                sc += kn @ qn[h * G + g] / np.sqrt(cfg.head_dim)
            want = orc.topk_of_logits(sc, cfg.budget)
            assert np.array_equal(got, want), (l, b, h)
        for g in range(G):
            hq = h * G + g
            if src == l:
                ref, _ = orc.full_attention(qn[hq], kn, vn)
            else:
                ref = orc.subset_attention(qn[hq], kn, vn, got)
            assert rel(res.outputs[l, b, hq].double().cpu().numpy(), ref) < 2e-2


@pytest.mark.parametrize("name,batch", [("cfg2", 1), ("cfg3", 1), ("cfg4", 2)])
def test_full_size_configs_sampled_rows(name, batch):
    cfg = CONFIGS[name].with_(batch=batch)
    q, k, v = generate_torch(cfg, "cuda")
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    res = dec.step(q, cfg.context)
    torch.cuda.synchronize()
    dec.check_flags()
    sel = res.selections
    # every set: k distinct ascending indices in range
    assert sel.shape[-1] == cfg.budget
    assert bool((sel[..., 1:] > sel[..., :-1]).all())
    assert int(sel.min()) >= 0 and int(sel.max()) < cfg.context
    rng = np.random.default_rng(1)
    layers = [cfg.full_layers[0], cfg.full_layers[-1], cfg.full_layers[0] + 1
              if cfg.actions[cfg.full_layers[0] + 1] == "reuse" else 3, cfg.layers - 2]
    rows = [(l, int(rng.integers(batch)), int(rng.integers(cfg.kv_heads))) for l in layers]
    _check_rows(cfg, q, k, v, res, rows, cfg.context)
    del q, k, v, dec, res
    torch.cuda.empty_cache()


def test_full_budget_reuse_equals_full_attention():
    """Acceptance criterion 04: a budget covering the cache makes REUSE exact."""
    cfg = CONFIGS["cfg2"].with_(layers=4, full_layers=(0,), context=4096, budget=4096, batch=2)
    q, k, v = generate_torch(cfg, "cuda")
    res = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads).step(q, 4096)
    full = HybridDecoder(("full",) * 4, k, v, cfg.budget, q_heads=cfg.q_heads).step(q, 4096)
    a = res.outputs.double().cpu().numpy()
    b = full.outputs.double().cpu().numpy()
    assert max(rel(a[l, bb, h], b[l, bb, h]) for l in range(4) for bb in range(2)
               for h in range(cfg.q_heads)) < 2e-3


def test_config5_profile_policy_matches_oracle():
    """BASELINE config 5: all-FULL profiling pass at 32K over 32 layers x 8 KV heads, GPU
    overlap matrix -> per-KV-head reference fold -> merge -> DP. The policy must equal the
    one planned from the float64 oracle's own index sets on the same seed."""
    cfg = CONFIGS["cfg5"]
    T = 2
    q, k, v = generate_torch(cfg, "cuda")
    g = torch.Generator(device="cuda").manual_seed(99)
    qs = [q, (q.float() + 0.5 * torch.randn(q.shape, generator=g, device="cuda")).to(q.dtype)]
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    idx = torch.empty((T, cfg.layers, cfg.kv_heads, cfg.budget), dtype=torch.int32, device="cuda")
    for t in range(T):
        res = dec.step(qs[t], cfg.context)
        idx[t].copy_(res.selections[:, 0])
    counts = overlap_counts(idx, cfg.context).cpu().numpy()  # [T, Hkv, L, L]
    mats = [similarity_from_counts(counts[:, h], cfg.budget) for h in range(cfg.kv_heads)]
    gpu_matrix = merge_similarity_matrices(mats)
    # oracle: float64 sets of every (layer, kv head) on the same stored values
    oracle_sets = np.zeros((T, cfg.layers, cfg.kv_heads, cfg.budget), dtype=np.int64)
    for t in range(T):
        qn = qs[t].double().cpu().numpy()
        for l in range(cfg.layers):
            kl = k[l, 0].double().cpu().numpy()
            sc = orc.group_scores(qn[l], kl[None], cfg.context, cfg.group, 1)
            for h in range(cfg.kv_heads):
                oracle_sets[t, l, h] = orc.topk_of_logits(sc[0, h], cfg.budget)
    assert np.array_equal(idx.cpu().numpy(), oracle_sets)
    omats = [orc.similarity_fold(orc.overlap_counts([[oracle_sets[t, l, h]
                                                      for l in range(cfg.layers)]
                                                     for t in range(T)]), cfg.budget)
             for h in range(cfg.kv_heads)]
    omerged = orc.merge_fold(omats)
    assert np.array_equal(gpu_matrix.values, omerged)
    for theta in (0.3, 0.5, 0.7, 0.9):
        p = dp_optimize(gpu_matrix, theta)
        from paper_2602_00777_b200 import SimilarityMatrix
        po = dp_optimize(SimilarityMatrix(values=omerged, budget=cfg.budget), theta)
        assert p.actions == po.actions and p.sources == po.sources
        assert p.cum_similarity == po.cum_similarity


def test_sink_and_recent_augmentation(golden_dir):
    """tests/test_engine.py:146-158: REUSE sets = selection | first sinks | last recent;
    FULL layers untouched (engine.py:122-126,187-188)."""
    z = load_npz(golden_dir / "fixture_engine.npz")
    model = FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]))
    pol = policy_from_actions(("full", "reuse", "reuse", "full", "reuse", "reuse"))
    plain = hybrid_decode(model, pol, 8, 2)
    aug = hybrid_decode(model, pol, 8, 2, include_sinks=4, include_recent=4)
    for t in range(2):
        n_t = int(z["context_len"]) + t
        for l in (1, 2, 4, 5):
            base = set(plain.selections[t][l].indices)
            want = base | set(range(4)) | set(range(n_t - 4, n_t))
            assert set(aug.selections[t][l].indices) == want
            assert aug.reuse_gathered_rows[t][l] == len(want)
            # the oracle on the augmented set
            qn = np.asarray(z["queries"][t][l, 0])
            kn = np.asarray(z["keys"][l, 0, :n_t])
            vn = np.asarray(z["values"][l, 0, :n_t])
            ref = orc.subset_attention(qn, kn, vn, sorted(want))
            assert rel(aug.outputs[t, l, 0], ref) < 1e-3
        for l in (0, 3):
            np.testing.assert_array_equal(plain.outputs[t, l], aug.outputs[t, l])
