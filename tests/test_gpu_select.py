"""The histogram-driven and cooperative selection paths (select.cuh hist_select / coop_*)
against the sampled path and the float64 oracle.

The FULL kernel emits a per-row histogram of the scores; the selects read it instead of
sampling the row ("fused3" / "fusedsel" / "single"), and the single-launch step with
cooperative selects ("singlecoop", fuse_select = 3) spreads each row's classification over
the splits of its pair. Every path must give bit-identical outputs and selections, with the
histogram / records re-zeroed for the next step (repeated steps, graph replays).
"""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from test_gpu_kernels import make_stack  # noqa: E402

SHAPES = [
    # actions, B, Hq, Hkv, d, n, budget
    (("full", "reuse", "full", "full", "reuse", "reuse", "full", "reuse"), 2, 16, 4, 128, 8192, 512),
    (("full", "full", "reuse", "reuse"), 1, 32, 8, 128, 32768, 2048),
    (("full", "reuse", "reuse"), 3, 28, 4, 128, 20000, 1000),     # G = 7, ragged n
    (("full", "reuse", "full", "reuse"), 2, 16, 4, 64, 4100, 300),  # d = 64
    (("full", "reuse"), 1, 8, 2, 128, 1500, 128),                 # short rows: sorted path
    (("full", "reuse"), 1, 8, 2, 128, 3000, 3000),                # budget covers the cache
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("refine", [True, False])
def test_schedules_bit_identical_with_histogram_and_coop(shape, refine):
    actions, B, Hq, Hkv, d, n, budget = shape
    q, k, v, qn, kn, vn = make_stack(len(actions), B, Hq, Hkv, d, n, "bf16", seed=61, planted=96)
    ref = None
    for name in ("fused3", "fusedsel", "single", "singlecoop"):
        dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, refine=refine)
        dec.set_schedule(name)
        for rep in range(3):  # the histograms / coop records reset themselves
            res = dec.step(q, n)
            torch.cuda.synchronize()
            dec.check_flags()
            got = (res.outputs.clone(), res.selections.clone())
            if ref is None:
                ref = got
            assert torch.equal(got[1], ref[1]), (name, rep)
            assert torch.equal(got[0], ref[0]), (name, rep)
    if refine:  # and the oracle's sets
        _, sets, _ = orc.hybrid_step(qn, kn, vn, n, actions, budget)
        sel = ref[1].cpu().numpy()
        slot = 0
        for l, a in enumerate(actions):
            if a == "full":
                assert np.array_equal(sel[slot], sets[l]), l
                slot += 1


def test_singlecoop_graph_replay_and_growing_rows():
    actions = ("full", "reuse", "full", "reuse", "reuse", "full")
    L, B, Hq, Hkv, d, cap, budget = len(actions), 2, 32, 8, 128, 16384, 1024
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=71, planted=64)
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq)
    dec.set_schedule("singlecoop")
    for n in (9000, 16384, 12345, 16384):
        res = dec.step(q, n)
        ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, single_launch=False,
                            fuse_select=False).step(q, n)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, ref.selections), n
        assert torch.equal(res.outputs, ref.outputs), n
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cap)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, cap)
    want_o, want_i = dec.out.clone(), dec.idx.clone()
    for _ in range(4):
        dec.out.zero_()
        dec.idx.zero_()
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(dec.out, want_o) and torch.equal(dec.idx, want_i)


def test_singlecoop_non_finite_row_falls_back_and_flags():
    from paper_2602_00777_b200 import NumericInputError
    actions = ("full", "reuse")
    q, k, v, *_ = make_stack(2, 1, 8, 2, 128, 8192, "bf16", seed=5)
    k[0, 0, 1, 4000, 3] = float("inf")
    dec = HybridDecoder(actions, k, v, 256, q_heads=8)
    dec.set_schedule("singlecoop")
    dec.step(q, 8192)
    torch.cuda.synchronize()
    with pytest.raises(NumericInputError):
        dec.check_flags()
    # the next clean step is unaffected (records and histograms were reset)
    k[0, 0, 1, 4000, 3] = 0.0
    dec.clear_flags()
    res = dec.step(q, 8192)
    ref = HybridDecoder(actions, k, v, 256, q_heads=8, single_launch=False,
                        fuse_select=False).step(q, 8192)
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(res.selections, ref.selections)
    assert torch.equal(res.outputs, ref.outputs)
