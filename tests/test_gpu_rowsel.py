"""The shared-memory-resident select (csrc/rowsel.cuh): one CTA cluster per score row.

Its index sets must equal the streaming select's (select.cuh select_row) bit for bit, with
and without the float64 boundary refinement, at every cluster size (1, 2, 4, 8 CTAs), for
grouped rows (sel_group > 1) and on the degenerate rows that take its generic path (ties,
all-equal rows, a refinement window over kCandCap). Reference rule: attention.py:264-275
(topk_of_logits) with the heads summed in reference order (engine.py:177-181).
"""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.attention import full_attention, topk_select  # noqa: E402

DEV = "cuda"


def _planted_stack(n, Hkv=4, G=4, d=128, B=2, seed=0):
    """bf16 q / K with 256 planted tokens per (b, kv-head) pulled toward the group's query."""
    g = torch.Generator().manual_seed(seed)
    q = torch.randn((1, B, Hkv * G, d), generator=g)
    k = torch.randn((1, B, Hkv, n, d), generator=g)
    for b in range(B):
        for h in range(Hkv):
            pos = torch.randperm(n, generator=g)[:256]
            qd = q[0, b, h * G:(h + 1) * G].mean(0)
            k[0, b, h, pos] += 2.0 * qd / qd.norm()
    q, k = q.to(torch.bfloat16).to(DEV), k.to(torch.bfloat16).to(DEV)
    return q, k


@pytest.mark.parametrize("n,budget,sel_group,cluster", [
    (8192, 128, 1, 1), (32768, 2048, 1, 1), (40960, 2048, 1, 1), (40961, 2048, 1, 2),
    (65536, 2048, 1, 2), (131072, 4096, 1, 4), (262144, 4096, 1, 8), (32768, 2048, 2, 1),
    (70000, 3000, 4, 2),
])
def test_rowsel_equals_streaming_select_refined(n, budget, sel_group, cluster):
    q, k = _planted_stack(n, seed=n + sel_group)
    _, sc = full_attention(q, k, k, n)
    with _abi.tuning(rowsel=1, rowsel_cluster=cluster):  # the fewest CTAs holding the row
        got, info = topk_select(sc, budget, n, sel_group=sel_group, q=q, k=k, info=True)
    with _abi.tuning(rowsel=1):  # rows spread over more CTAs (few rows)
        spread = topk_select(sc, budget, n, sel_group=sel_group, q=q, k=k)
    assert torch.equal(got, spread)
    with _abi.tuning(rowsel=0):
        ref = topk_select(sc, budget, n, sel_group=sel_group, q=q, k=k)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    inf = info.cpu().numpy().reshape(-1, 8)
    assert (inf[:, 3] == cluster).all()          # cluster size used
    assert np.isin(inf[:, 2], [7, 67]).all()      # band path (7) or generic refine path (67)
    # and the float64 rule itself, on one row: the fp32 scores' order except inside the
    # refinement window, where float64 scores decide
    qn = q.double().cpu().numpy()
    kn = k.double().cpu().numpy()
    agg = orc.group_scores(qn[0], kn[0], n, 4, sel_group)
    np.testing.assert_array_equal(got[0, 0, 0].cpu().numpy(),
                                  orc.topk_of_logits(agg[0, 0], budget))


@pytest.mark.parametrize("n,budget,kind", [
    (20000, 1500, "ties"), (9000, 700, "allequal"), (70000, 3000, "ties"),
    (131072, 4096, "allequal"), (50000, 5000, "normal"), (100000, 16384, "normal"),
])
def test_rowsel_degenerate_rows_match_streaming_select(n, budget, kind):
    rng = np.random.default_rng(n)
    rows = 6
    if kind == "ties":
        x = rng.integers(-20, 20, size=(rows, n)).astype(np.float32)
    elif kind == "allequal":
        x = np.full((rows, n), 0.75, dtype=np.float32)
    else:
        x = rng.standard_normal((rows, n)).astype(np.float32)
    rs = (n + 7) & ~7
    buf = np.zeros((1, rows, 1, rs), dtype=np.float32)
    buf[0, :, 0, :n] = x
    sc = torch.from_numpy(buf).to(DEV)
    with _abi.tuning(rowsel=1):
        got = topk_select(sc, budget, n).cpu().numpy()
    with _abi.tuning(rowsel=0):
        ref = topk_select(sc, budget, n).cpu().numpy()
    np.testing.assert_array_equal(got, ref)
    for r in range(rows):
        np.testing.assert_array_equal(got[0, r, 0], orc.topk_of_logits(x[r].astype(np.float64),
                                                                       budget))


def test_rowsel_oversized_window_skips_refinement_like_streaming_select():
    """A row whose refinement window holds more than kCandCap scores: both selects fall back
    to fp32 order with the lower-index tie rule and raise HYLRA_FLAG_REFINE_SKIPPED."""
    from paper_2602_00777_b200.errors import SelectionPrecisionWarning
    n, budget = 32768, 2048
    q, k = _planted_stack(n, Hkv=2, G=4, B=1, seed=5)
    _, sc = full_attention(q, k, k, n)
    # squeeze every score into a band far narrower than tau = max|s| / 4096 around 1.0, plus
    # one large score so max|s| (and tau) stay wide
    sc[..., :n] = 1.0 + (sc[..., :n] - sc[..., :n].mean()) * 1e-6
    sc[..., 7] = 100.0
    with _abi.tuning(rowsel=1):
        with pytest.warns(SelectionPrecisionWarning):
            got = topk_select(sc, budget, n, q=q, k=k)
    with _abi.tuning(rowsel=0):
        with pytest.warns(SelectionPrecisionWarning):
            ref = topk_select(sc, budget, n, q=q, k=k)
    assert torch.equal(got, ref)
    x = sc[0, 0, 0, :n].double().cpu().numpy()
    np.testing.assert_array_equal(got[0, 0, 0].cpu().numpy(), orc.topk_of_logits(x, budget))
