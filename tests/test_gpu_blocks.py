"""Block-level selection (paper §3.5; reference engine.py:212-286) on the GPU."""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import policy_from_actions  # noqa: E402
from paper_2602_00777_b200.attention import block_select, full_attention, topk_select  # noqa: E402
from paper_2602_00777_b200.engine import (HybridDecoder, hybrid_decode,  # noqa: E402
                                          hybrid_decode_blocks)
from refmodel import FixtureModel, load_npz  # noqa: E402
from test_gpu_kernels import make_stack, max_head_err  # noqa: E402


def rel(x, r):
    return float(np.linalg.norm(x - r) / np.linalg.norm(r))


def test_block_fixture_golden(golden_dir):
    """BLOCK_FIXTURE: 2 blocks of 128, static_jump_policy(5, 2), golden aggregate
    0.4524886792120594 (tests/test_engine.py:34-38,196-206)."""
    z = load_npz(golden_dir / "block_reference.npz")
    model = FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]))
    run = hybrid_decode_blocks(model, policy_from_actions(tuple(z["actions"])),
                               int(z["block_budget"]), int(z["block_size"]), 2)
    got = np.array([[list(s.block_indices) for s in row] for row in run.selections])
    assert np.array_equal(got, z["blocks"])
    for t in range(2):
        for l in range(5):
            assert rel(run.outputs[t, l].ravel(), z["outputs"][t, l].ravel()) < 1e-3
            want = int(z["gathered"][t][l])
            assert run.reuse_gathered_rows[t][l] == (None if want < 0 else want)
    assert run.fidelity.aggregate == pytest.approx(0.4524886792120594, rel=1e-3)


def test_block_size_one_equals_token_mode(golden_dir):
    """hybrid_decode_blocks(..., block_size=1) == hybrid_decode (tests/test_engine.py:183-193)."""
    z = load_npz(golden_dir / "fixture_engine.npz")
    model = FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]))
    pol = policy_from_actions(tuple(z["actions"]))
    tok = hybrid_decode(model, pol, 12, 3)
    blk = hybrid_decode_blocks(model, pol, 12, 1, 3)
    assert np.allclose(tok.outputs, blk.outputs, rtol=1e-5, atol=1e-6)
    for t in range(3):
        for l in range(6):
            n_t = int(z["context_len"]) + t
            assert blk.selections[t][l].token_coverage(n_t).tolist() == \
                list(tok.selections[t][l].indices)


@pytest.mark.parametrize("n,bb,bs,kind,sg", [
    (4000, 16, 128, "normal", 1), (4000, 40, 64, "ties", 1), (32768, 16, 128, "normal", 1),
    (1000, 3, 300, "normal", 1), (4001, 10, 4, "normal", 1), (5003, 7, 32, "ties", 1),
    (777, 5, 8, "normal", 2), (3001, 20, 16, "ties", 2), (3000, 20, 2, "ties", 1),
    (70001, 9, 128, "normal", 2), (65, 2, 64, "normal", 1)])
def test_block_select_matches_oracle(n, bb, bs, kind, sg):
    rng = np.random.default_rng(n + bb)
    S, B, H = 2, 2, 4
    x = (rng.standard_normal((S, B, H, n)) if kind == "normal"
         else rng.integers(-5, 5, size=(S, B, H, n))).astype(np.float32)
    x[0, 0, 0, -5:] += 9.0  # make the truncated final block win somewhere
    buf = np.zeros((S, B, H, (n + 7) & ~7), dtype=np.float32)
    buf[..., :n] = x
    buf[..., n:] = 1e9  # padding past n must never be pooled
    blocks, tokens, counts = block_select(torch.from_numpy(buf).cuda(), bb, bs, n, sel_group=sg)
    blocks, tokens, counts = blocks.cpu().numpy(), tokens.cpu().numpy(), counts.cpu().numpy()
    for s in range(S):
        for b in range(B):
            for grp in range(H // sg):
                agg = np.zeros(n, dtype=np.float32)
                for h in range(grp * sg, (grp + 1) * sg):
                    agg += x[s, b, h]  # fp32 head-order sum, as the pooling kernel adds
                want = orc.topk_of_logits(orc.block_max_of_logits(agg.astype(np.float64), bs), bb)
                assert np.array_equal(blocks[s, b, grp], want)
                cov = orc.block_coverage(want, bs, n)
                assert counts[s, b, grp] == cov.shape[0]
                assert np.array_equal(tokens[s, b, grp, :cov.shape[0]], cov)


@pytest.mark.parametrize("n,k", [(2048, 100), (2049, 100), (300, 17), (64, 63), (1500, 1)])
def test_small_row_select_ties_and_refinement(n, k):
    """Rows of <= 2048 scores take the sorted small-row path: exact (score desc, index asc)
    without refinement; with q/k the float64 re-score decides near-ties."""
    rng = np.random.default_rng(n * 7 + k)
    x = rng.integers(-3, 3, size=(1, 2, 2, n)).astype(np.float32)
    buf = np.zeros((1, 2, 2, (n + 7) & ~7), dtype=np.float32)
    buf[..., :n] = x
    idx = topk_select(torch.from_numpy(buf).cuda(), k, n).cpu().numpy()
    for b in range(2):
        for h in range(2):
            assert np.array_equal(idx[0, b, h], orc.topk_of_logits(x[0, b, h].astype(np.float64), k))
    # refinement on real scores: GPU FULL scores + refined select == float64 oracle sets
    L, B, Hq, Hkv, d = 1, 2, 8, 2, 64
    q, kk, v, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=n + k, planted=min(k, 8))
    _, sc = full_attention(q, kk, v, n)
    got = topk_select(sc, k, n, q=q, k=kk).cpu().numpy()
    sc64 = orc.group_scores(qn[0], kn[0], n, Hq // Hkv, 1)
    for b in range(B):
        for h in range(Hkv):
            assert np.array_equal(got[0, b, h], orc.topk_of_logits(sc64[b, h], k))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_block_decode_step_matches_oracle(dtype):
    L, B, Hq, Hkv, d, cap, n_valid, bb, bs = 5, 2, 16, 4, 128, 4200, 4100, 8, 128
    q, k, v, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, cap, dtype, seed=17, planted=48)
    actions = ("full", "reuse", "full", "reuse", "reuse")
    dec = HybridDecoder(actions, k, v, bb, q_heads=Hq, block_size=bs)
    res = dec.step(q, n_valid)
    torch.cuda.synchronize()
    dec.check_flags()
    ref_out, ref_blocks = orc.hybrid_step_blocks(qn, kn, vn, n_valid, actions, bb, bs)
    sel = res.selections.cpu().numpy()
    for l in range(L):
        assert np.array_equal(sel[res.slot_of_layer[l]], ref_blocks[l])
    tol = 2e-2 if dtype == "bf16" else 1e-3
    assert max_head_err(res.outputs.double().cpu().numpy(), ref_out) < tol


@pytest.mark.parametrize("n,bs,bb", [(4096, 64, 8), (3000, 16, 5)])
def test_block_refinement_all_tied(n, bs, bb):
    """Every key identical: all blocks tie, every token qualifies for the float64 re-score
    (more than the filtered list holds at n=4096), and ties go to the lowest blocks."""
    L, B, Hq, Hkv, d = 2, 1, 8, 2, 128
    q, k, v, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=5)
    k[:] = k[:, :, :, :1, :]
    kn[:] = kn[:, :, :, :1, :]
    actions = ("full", "reuse")
    dec = HybridDecoder(actions, k, v, bb, q_heads=Hq, block_size=bs)
    res = dec.step(q, n)
    torch.cuda.synchronize()
    dec.check_flags()
    ref_out, ref_blocks = orc.hybrid_step_blocks(qn, kn, vn, n, actions, bb, bs)
    sel = res.selections.cpu().numpy()
    assert np.array_equal(sel[res.slot_of_layer[0]], ref_blocks[0])
    assert list(ref_blocks[0][0, 0]) == list(range(bb))
    assert max_head_err(res.outputs.double().cpu().numpy(), ref_out) < 2e-2


@pytest.mark.parametrize("bs,bb,n_valid", [(128, 8, 4100), (64, 12, 4096), (192, 6, 3900)])
def test_block_reuse_tiles_equal_row_gather(bs, bb, n_valid, monkeypatch):
    """Block-mode REUSE by TMA tiles of the selected blocks (block_size a multiple of 64)
    reads the same rows in the same order as the row-by-row coverage gather: identical
    outputs and selections (HYLRA_BLOCK_TILES=0 forces the gather). A ragged last block
    (n_valid not a multiple of block_size) is masked by the coverage count."""
    L, B, Hq, Hkv, d, cap = 5, 2, 16, 4, 128, 4200
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=23, planted=48)
    # plant the final token so the ragged last block is selected
    k[:, :, :, n_valid - 1, :] = 4.0 * q.float().view(L, B, Hkv, Hq // Hkv, d).mean(3).to(k.dtype)
    actions = ("full", "reuse", "full", "reuse", "reuse")
    monkeypatch.setenv("HYLRA_BLOCK_TILES", "0")
    ref = HybridDecoder(actions, k, v, bb, q_heads=Hq, block_size=bs,
                        single_launch=False).step(q, n_valid)
    torch.cuda.synchronize()
    R, S = ref.outputs.clone(), ref.selections.clone()
    nb = -(-n_valid // bs)
    assert bool((S == nb - 1).any(-1).all()), "the ragged last block must be selected"
    monkeypatch.setenv("HYLRA_BLOCK_TILES", "1")
    dec = HybridDecoder(actions, k, v, bb, q_heads=Hq, block_size=bs, single_launch=False)
    res = dec.step(q, n_valid)
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(res.selections, S)
    assert torch.equal(res.outputs, R)


@pytest.mark.parametrize("bs,bb,n_valid,B", [(128, 8, 4100, 2), (64, 12, 4096, 1), (16, 40, 3001, 2),
                                             (12, 30, 2000, 3)])
def test_block_single_launch_equals_multi_launch(bs, bb, n_valid, B):
    """hylra_decode_step_blocks_ex fuse_select=2: the final CTA of each FULL pair pools the
    token scores into blocks, selects them and writes the coverage, REUSE items gather it
    after their row's ready flag: bit-identical to the multi-launch block step (pool kernel,
    block SELECT, expansion, REUSE), over repeated steps and graph replays. Ragged last
    blocks and block sizes that are not multiples of 4 included."""
    L, Hq, Hkv, d, cap = 6, 16, 4, 128, 4200
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=29, planted=48)
    actions = ("full", "reuse", "full", "reuse", "reuse", "full")
    ref = HybridDecoder(actions, k, v, bb, q_heads=Hq, block_size=bs, single_launch=False)
    r = ref.step(q, n_valid)
    torch.cuda.synchronize()
    R, S = r.outputs.clone(), r.selections.clone()
    dec = HybridDecoder(actions, k, v, bb, q_heads=Hq, block_size=bs, single_launch=True)
    assert dec.single and dec.kernels_per_step == 1
    for _ in range(2):
        res = dec.step(q, n_valid)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, S)
        assert torch.equal(res.outputs, R)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, n_valid)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, n_valid)
    for _ in range(3):
        dec.out.zero_()
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(dec.out, R)


@pytest.mark.parametrize("single", [True, False])
def test_block_decode_loop_appends_in_step(single):
    """DecodeLoop over a block-mode decoder (zero copy): the step's new K/V rows ride the
    step's append option (hylra_decode_step_blocks_ex append_*) — written inside the
    single-launch kernel, or appended ahead of the multi-launch step — queries and outputs
    in pinned host memory. Equal to an eager step over a cache holding the same rows."""
    from paper_2602_00777_b200.engine import DecodeLoop
    L, B, Hq, Hkv, d, cap, bs, bb = 6, 2, 16, 4, 128, 4200, 64, 12
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=37, planted=48)
    actions = ("full", "reuse", "full", "reuse", "reuse", "full")
    dec = HybridDecoder(actions, k.clone(), v.clone(), bb, q_heads=Hq, block_size=bs,
                        single_launch=single)
    assert dec.single == single
    pos = 3999
    loop = DecodeLoop(dec, pos, q_copy=False)
    assert loop.zero_copy
    g = torch.Generator().manual_seed(5)
    for _ in range(3):
        qh = torch.randn((L, B, Hq, d), generator=g).to(torch.bfloat16)
        kh = torch.randn((L, B, Hkv, d), generator=g).to(torch.bfloat16)
        vh = torch.randn((L, B, Hkv, d), generator=g).to(torch.bfloat16)
        loop.q_host.copy_(qh)
        loop.k_host.copy_(kh)
        loop.v_host.copy_(vh)
        out = loop.run().clone()
        dec.check_flags()
        k2, v2 = k.clone(), v.clone()
        k2[:, :, :, pos] = kh.cuda()
        v2[:, :, :, pos] = vh.cuda()
        assert torch.equal(dec.k, k2) and torch.equal(dec.v, v2)
        ref = HybridDecoder(actions, k2, v2, bb, q_heads=Hq, block_size=bs,
                            single_launch=False).step(qh.cuda(), pos + 1)
        torch.cuda.synchronize()
        assert torch.equal(dec.idx[..., :ref.selections.shape[-1]], ref.selections)
        assert torch.equal(out, ref.outputs.cpu())
