"""Block-level selection (paper §3.5; reference engine.py:212-286) on the GPU."""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import policy_from_actions  # noqa: E402
from paper_2602_00777_b200.attention import block_select  # noqa: E402
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


@pytest.mark.parametrize("n,bb,bs,kind", [(4000, 16, 128, "normal"), (4000, 40, 64, "ties"),
                                          (32768, 16, 128, "normal"), (1000, 3, 300, "normal")])
def test_block_select_matches_oracle(n, bb, bs, kind):
    rng = np.random.default_rng(n + bb)
    S, B, H = 2, 2, 2
    x = (rng.standard_normal((S, B, H, n)) if kind == "normal"
         else rng.integers(-5, 5, size=(S, B, H, n))).astype(np.float32)
    x[0, 0, 0, -5:] += 9.0  # make the truncated final block win somewhere
    buf = np.zeros((S, B, H, (n + 7) & ~7), dtype=np.float32)
    buf[..., :n] = x
    blocks, tokens, counts = block_select(torch.from_numpy(buf).cuda(), bb, bs, n)
    blocks, tokens, counts = blocks.cpu().numpy(), tokens.cpu().numpy(), counts.cpu().numpy()
    for s in range(S):
        for b in range(B):
            for h in range(H):
                want = orc.topk_of_logits(orc.block_max_of_logits(x[s, b, h].astype(np.float64), bs),
                                          bb)
                assert np.array_equal(blocks[s, b, h], want)
                cov = orc.block_coverage(want, bs, n)
                assert counts[s, b, h] == cov.shape[0]
                assert np.array_equal(tokens[s, b, h, :cov.shape[0]], cov)


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
