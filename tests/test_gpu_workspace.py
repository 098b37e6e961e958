"""Workspace reuse and input validation on the GPU (VERDICT Missing 5 / Weak 2).

* One decoder stepping over a growing cache reuses its workspace across many n_valid
  values: every step must equal a step on a fresh (zeroed) workspace, bit for bit, under
  every schedule. (Round 1 placed the split-K counters after n_valid-sized partials, so a
  counter could start on a stale partial and its merge never fire.)
* The side-stream schedule with more pairs in its second FULL launch than in its first.
* Non-finite cache entries a step never reads are still rejected (the reference checks the
  whole cache when it builds its float64 copies, attention.py:38-46,61-71).
* A selection whose float64 refinement window is too wide is reported, not silent.
"""
import warnings

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import (InvalidSelectionError, NumericInputError,  # noqa: E402
                                   SelectionPrecisionWarning)
from paper_2602_00777_b200.engine import DecodeLoop, HybridDecoder  # noqa: E402
from test_gpu_kernels import make_stack, max_head_err  # noqa: E402


@pytest.mark.parametrize("schedule", ["fusedsel", "single", "fused3"])
def test_workspace_reuse_across_growing_n_valid(schedule):
    """ADVICE (high): Hkv 4, G 7, B 1, budget 1024, n_valid growing from 4096 (4929 hit the
    round-1 aliasing under fusedsel)."""
    L, B, Hq, Hkv, d, cap, budget = 6, 1, 28, 4, 128, 8192, 1024
    actions = ("full", "reuse", "full", "reuse", "reuse", "full")
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=44, planted=48)
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq)
    dec.set_schedule(schedule)
    sizes = list(range(4096, 5300, 41)) + [4929, 8192, 4100, 6001, 4929]
    for n in sizes:
        res = dec.step(q, n)
        fresh = HybridDecoder(actions, k, v, budget, q_heads=Hq)
        fresh.set_schedule(schedule)
        ref = fresh.step(q, n)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, ref.selections), n
        assert torch.equal(res.outputs, ref.outputs), n


def test_dual_stream_second_full_launch_larger_than_first():
    """ADVICE (medium): FULL(A) then FULL(B) on one workspace with |B| > |A| pairs; the
    outputs change every step (new queries), so a merge that never fired shows."""
    actions = ("full", "reuse", "full", "full", "full", "full", "reuse", "full")
    L, B, Hq, Hkv, d, cap, budget = len(actions), 8, 32, 8, 128, 2048, 256
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=5, planted=32)
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, dual_stream=True, fuse_select=False)
    assert dec.dual
    g = torch.Generator(device="cuda").manual_seed(9)
    for _ in range(4):
        qs = torch.randn(q.shape, generator=g, device="cuda").to(q.dtype)
        res = dec.step(qs, cap)
        ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, fuse_select=False,
                            single_launch=False).step(qs, cap)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, ref.selections)
        assert max_head_err(res.outputs.double().cpu().numpy(),
                            ref.outputs.double().cpu().numpy()) < 4e-3


def test_validate_cache_rejects_unread_non_finite_rows():
    """A NaN in a row no kernel reads (an unselected row of a REUSE layer) passes the step,
    but validate_cache rejects it like the reference's cache construction."""
    L, B, Hq, Hkv, d, cap, budget = 4, 2, 8, 2, 128, 4096, 128
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=8, planted=16)
    actions = ("full", "reuse", "full", "reuse")
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq)
    res = dec.step(q, cap)
    torch.cuda.synchronize()
    sel = set(res.selections[0, 1, 0].tolist())
    row = next(r for r in range(cap) if r not in sel)
    dec.v[1, 1, 0, row, 5] = float("nan")  # layer 1 REUSE, b 1, kv head 0
    dec.clear_flags()
    dec.step(q, cap)
    torch.cuda.synchronize()
    dec.check_flags()  # the step never read that row
    with pytest.raises(NumericInputError, match="KV cache"):
        dec.validate_cache(cap)
    dec.v[1, 1, 0, row, 5] = 0.0
    dec.validate_cache(cap)
    # fp32 caches too
    q32, k32, v32, *_ = make_stack(2, 1, 8, 2, 64, 1024, "f32", seed=1)
    d32 = HybridDecoder(("full", "reuse"), k32, v32, 64, q_heads=8)
    d32.validate_cache()
    d32.k[0, 0, 1, 1000, 63] = float("-inf")
    with pytest.raises(NumericInputError):
        d32.validate_cache()
    d32.validate_cache(1000)  # the row lies past n_valid


@pytest.mark.parametrize("single", [False, True])
def test_appended_non_finite_rows_raise(single):
    L, B, Hq, Hkv, d, cap, budget = 4, 1, 8, 2, 128, 2048, 128
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=3)
    dec = HybridDecoder(("full", "reuse", "full", "reuse"), k, v, budget, q_heads=Hq,
                        single_launch=single)
    rows_k = torch.randn((L, B, Hkv, d), device="cuda").to(torch.bfloat16)
    rows_v = torch.randn((L, B, Hkv, d), device="cuda").to(torch.bfloat16)
    dec.step(q, cap, append=(rows_k, rows_v, 2000))
    torch.cuda.synchronize()
    dec.check_flags()
    rows_v[3, 0, 1, 7] = float("nan")  # a REUSE layer's row: read only if selected
    dec.step(q, cap, append=(rows_k, rows_v, 2001))
    torch.cuda.synchronize()
    with pytest.raises(NumericInputError):
        dec.check_flags()
    dec.clear_flags()
    dec.append(rows_k, rows_v, 2002, layers=[3])
    torch.cuda.synchronize()
    with pytest.raises(NumericInputError, match="KV cache"):
        dec.check_flags()


@pytest.mark.parametrize("n,schedule", [(1500, "fused3"), (4096, "fused3"), (4096, "single"),
                                        (40000, "fusedsel")])
def test_refinement_skipped_is_reported(n, schedule):
    """Every score of the row within the float64 window of the k-th value (identical keys):
    more than 1024 window candidates, so the boundary falls back to fp32 order (lowest
    index on exact ties). The flag surfaces as SelectionPrecisionWarning (InvalidSelection
    Error when strict) with the count of such rows; with all scores tied the fallback
    still equals the reference (ties -> lower index)."""
    L, B, Hq, Hkv, d, budget = 2, 2, 8, 2, 128, 256
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=21)
    k.copy_(k[:, :, :, :1, :].clone().expand_as(k))  # every row: the same key
    dec = HybridDecoder(("full", "reuse"), k, v, budget, q_heads=Hq)
    dec.set_schedule(schedule)
    res = dec.step(q, n)
    torch.cuda.synchronize()
    assert dec.refine_skipped_rows() == B * Hkv
    with pytest.warns(SelectionPrecisionWarning, match=f"{B * Hkv} selection row"):
        dec.check_flags()
    with pytest.raises(InvalidSelectionError):
        dec.check_flags(strict=True)
    want = np.arange(budget)
    for b in range(B):
        for h in range(Hkv):
            assert np.array_equal(res.selections[0, b, h].cpu().numpy(), want)
    # and a normal row clears it
    dec.clear_flags()
    q2, k2, v2, *_ = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=22, planted=32)
    dec2 = HybridDecoder(("full", "reuse"), k2, v2, budget, q_heads=Hq)
    dec2.step(q2, n)
    torch.cuda.synchronize()
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        dec2.check_flags(strict=True)
    assert dec2.refine_skipped_rows() == 0
