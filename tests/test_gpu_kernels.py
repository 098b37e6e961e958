"""GPU parity: each CUDA kernel (through the C ABI) against the float64 oracle.

Tolerances (north_star): outputs within 1e-3 relative L2 per (b, head) for fp32 inputs and
2e-2 for bf16 inputs, against the float64 reference on the same (rounded) values; index
sets exactly equal (the f64 boundary refinement makes ties at fp32 resolution irrelevant;
only float64-level ties could differ and the seeded inputs have none).
"""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import (InvalidInputError, InvalidSelectionError,  # noqa: E402
                                   full_attention, sparse_attention, topk_select)
from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402

DEV = "cuda"


def make_stack(L, B, Hq, Hkv, d, cap, dtype, seed=0, planted=0):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn((L, B, Hq, d), generator=g)
    k = torch.randn((L, B, Hkv, cap, d), generator=g)
    v = torch.randn((L, B, Hkv, cap, d), generator=g)
    if planted:
        G = Hq // Hkv
        qm = q.view(L, B, Hkv, G, d).mean(3)
        qh = qm / qm.norm(dim=-1, keepdim=True)
        pos = torch.randperm(cap, generator=g)[:planted]
        k[:, :, :, pos, :] += 2.0 * qh[:, :, :, None, :]
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, k, v = q.to(dt), k.to(dt), v.to(dt)
    return q.to(DEV), k.to(DEV), v.to(DEV), q.double().numpy(), k.double().numpy(), v.double().numpy()


def rel_err(x, ref):
    return np.linalg.norm(x - ref) / np.linalg.norm(ref)


def max_head_err(out, ref):
    L, B, H, _ = ref.shape
    return max(rel_err(out[l, b, h], ref[l, b, h]) for l in range(L) for b in range(B)
               for h in range(H) if np.isfinite(ref[l, b, h]).all())


@pytest.mark.parametrize("dtype,d,Hq,Hkv,cap,n_valid", [
    ("bf16", 128, 32, 8, 4096, 4096),
    ("bf16", 128, 28, 4, 2048, 1999),   # G = 7, ragged tail
    ("bf16", 64, 8, 2, 1024, 777),
    ("bf16", 128, 16, 1, 512, 512),     # G = 16 (both fragment row halves)
    ("bf16", 128, 12, 1, 640, 600),     # G = 12
    ("bf16", 128, 8, 8, 300, 257),      # G = 1
    ("f32", 64, 8, 2, 2048, 2048),
    ("f32", 128, 32, 8, 1024, 1000),
    ("f32", 32, 4, 4, 96, 96),
    ("bf16", 32, 4, 2, 200, 131),       # SIMT bf16 path (d = 32)
])
def test_full_attention_matches_oracle(dtype, d, Hq, Hkv, cap, n_valid):
    q, k, v, qn, kn, vn = make_stack(2, 2, Hq, Hkv, d, cap, dtype, seed=d + Hq + cap)
    out, sc = full_attention(q, k, v, n_valid)
    torch.cuda.synchronize()
    out = out.double().cpu().numpy()
    sc = sc.double().cpu().numpy()
    G = Hq // Hkv
    ref = np.zeros_like(out)
    for l in range(2):
        for b in range(2):
            for h in range(Hq):
                ref[l, b, h], _ = orc.full_attention(qn[l, b, h], kn[l, b, h // G, :n_valid],
                                                     vn[l, b, h // G, :n_valid])
        refsc = orc.group_scores(qn[l], kn[l], n_valid, G, 1)
        np.testing.assert_allclose(sc[l, :, :, :n_valid], refsc, atol=2e-4 * np.abs(refsc).max())
    tol = 2e-2 if dtype == "bf16" else 1e-3
    assert max_head_err(out, ref) < tol


@pytest.mark.parametrize("n,budget,kind", [
    (2048, 128, "normal"), (32768, 2048, "normal"), (131072, 4096, "normal"),
    (5000, 4999, "normal"), (5000, 5000, "normal"), (4000, 1, "normal"),
    (20000, 1500, "ties"), (9000, 700, "allequal"), (70000, 3000, "ties"),
    (300, 17, "ties"), (65536, 2048, "planted"),
])
def test_topk_select_exact(n, budget, kind):
    rng = np.random.default_rng(n + budget)
    S, B, H = 2, 2, 2
    if kind == "normal":
        x = rng.standard_normal((S, B, H, n)).astype(np.float32)
    elif kind == "ties":
        x = rng.integers(-20, 20, size=(S, B, H, n)).astype(np.float32)
    elif kind == "allequal":
        x = np.full((S, B, H, n), 1.5, dtype=np.float32)
    else:
        x = rng.standard_normal((S, B, H, n)).astype(np.float32)
        x[..., rng.choice(n, 512, replace=False)] += 8.0
    rs = (n + 7) & ~7
    buf = np.zeros((S, B, H, rs), dtype=np.float32)
    buf[..., :n] = x
    idx = topk_select(torch.from_numpy(buf).to(DEV), budget, n)
    got = idx.cpu().numpy()
    for s in range(S):
        for b in range(B):
            for h in range(H):
                want = orc.topk_of_logits(x[s, b, h].astype(np.float64), budget)
                np.testing.assert_array_equal(got[s, b, h], want)


@pytest.mark.parametrize("rows,n,budget,kind", [
    (200, 32768, 2048, "normal"),    # 512-thread CTAs (149..296 rows)
    (320, 32768, 2048, "normal"),    # 256-thread CTAs (> 296 rows)
    (320, 20000, 1500, "ties"),
    (200, 9000, 700, "allequal"),
    (320, 65536, 2048, "planted"),
    (2, 262144, 16384, "normal"),    # longest supported row (bitmap 32 KB)
    (300, 262144, 4096, "planted"),
])
@pytest.mark.parametrize("impl", ["rowsel", "stream"])
def test_topk_select_exact_all_cta_widths(rows, n, budget, kind, impl):
    """The streaming SELECT's CTA width follows the row count (1024 / 512 / 256 threads) and
    the shared-memory-resident select (rowsel.cuh) covers rows up to 8 x 40960 tokens on CTA
    clusters: every width and cluster size returns the reference's exact sets, including at
    the maximum row length."""
    from paper_2602_00777_b200 import _abi
    rng = np.random.default_rng(rows * 7 + n)
    if kind == "normal":
        x = rng.standard_normal((rows, n)).astype(np.float32)
    elif kind == "ties":
        x = rng.integers(-20, 20, size=(rows, n)).astype(np.float32)
    elif kind == "allequal":
        x = np.full((rows, n), -0.25, dtype=np.float32)
    else:
        x = rng.standard_normal((rows, n)).astype(np.float32)
        for r in range(rows):
            x[r, rng.choice(n, 512, replace=False)] += 8.0
    rs = (n + 7) & ~7
    buf = np.zeros((1, rows, 1, rs), dtype=np.float32)
    buf[0, :, 0, :n] = x
    with _abi.tuning(rowsel=1 if impl == "rowsel" else 0):
        got = topk_select(torch.from_numpy(buf).to(DEV), budget, n).cpu().numpy()
    for r in range(rows):
        want = orc.topk_of_logits(x[r].astype(np.float64), budget)
        np.testing.assert_array_equal(got[0, r, 0], want)


def test_topk_select_group_sum_matches_layer_wide_rule():
    # sel_group = Hkv: one set per layer from the head-order sum (engine.py:177-183)
    rng = np.random.default_rng(3)
    S, B, H, n = 1, 2, 4, 3000
    x = rng.standard_normal((S, B, H, n)).astype(np.float32)
    idx = topk_select(torch.from_numpy(x.copy()).to(DEV), 100, n, sel_group=4)
    got = idx.cpu().numpy()
    for b in range(B):
        agg = np.zeros(n, dtype=np.float32)
        for h in range(H):
            agg = agg + x[0, b, h]
        np.testing.assert_array_equal(got[0, b, 0], orc.topk_of_logits(agg.astype(np.float64), 100))


@pytest.mark.parametrize("dtype,d,Hq,Hkv,cap,k", [
    ("bf16", 128, 32, 8, 4096, 1000), ("bf16", 64, 14, 2, 1024, 64), ("f32", 64, 8, 2, 2048, 128),
    ("bf16", 128, 16, 2, 512, 500), ("f32", 32, 2, 2, 99, 12),
])
def test_sparse_attention_matches_oracle(dtype, d, Hq, Hkv, cap, k):
    q, k_, v, qn, kn, vn = make_stack(2, 2, Hq, Hkv, d, cap, dtype, seed=k + d)
    rng = np.random.default_rng(k)
    idx = np.stack([np.stack([np.stack([np.sort(rng.choice(cap, k, replace=False))
                                        for _ in range(Hkv)]) for _ in range(2)])
                    for _ in range(2)]).astype(np.int32)
    out = sparse_attention(q, k_, v, torch.from_numpy(idx).to(DEV), cap).double().cpu().numpy()
    G = Hq // Hkv
    ref = np.zeros_like(out)
    for l in range(2):
        for b in range(2):
            for h in range(Hq):
                ref[l, b, h] = orc.subset_attention(qn[l, b, h], kn[l, b, h // G],
                                                    vn[l, b, h // G], idx[l, b, h // G])
    tol = 2e-2 if dtype == "bf16" else 1e-3
    assert max_head_err(out, ref) < tol


def test_sparse_attention_rejects_out_of_range():
    q, k, v, *_ = make_stack(1, 1, 4, 2, 64, 256, "bf16")
    idx = torch.tensor([[[[0, 5, 300]] * 2]], dtype=torch.int32, device=DEV)
    with pytest.raises(InvalidSelectionError):
        sparse_attention(q, k, v, idx, 256)
    # unchecked call: the device flag catches it
    with pytest.raises(InvalidSelectionError):
        sparse_attention(q, k, v, idx, 256, check=False)


def test_overlap_counts_exact():
    from paper_2602_00777_b200 import overlap_counts
    rng = np.random.default_rng(11)
    T, L, R, k, n = 3, 9, 4, 300, 70000
    sets = np.stack([np.stack([np.stack([np.sort(rng.choice(n, k, replace=False))
                                         for _ in range(R)]) for _ in range(L)])
                     for _ in range(T)]).astype(np.int32)
    sets[:, 1] = sets[:, 0]  # identical layers
    c = overlap_counts(torch.from_numpy(sets).to(DEV), n).cpu().numpy()
    for r in range(R):
        ref = orc.overlap_counts([[sets[t, l, r] for l in range(L)] for t in range(T)])
        np.testing.assert_array_equal(c[:, r], ref)


@pytest.mark.parametrize("dtype,refine,actions", [
    ("bf16", True, ("full", "reuse", "reuse", "full", "reuse", "full")),
    ("f32", True, ("full", "reuse", "reuse", "full", "reuse", "full")),
    ("bf16", False, ("full", "reuse", "reuse", "full", "reuse", "full")),
    # many more REUSE than FULL (layer, b, head) pairs: disjoint split-K workspaces
    ("bf16", True, ("full",) + ("reuse",) * 13),
])
def test_decode_step_matches_oracle(dtype, refine, actions):
    L, B, Hq, Hkv, d, cap, n_valid, budget = len(actions), 2, 16, 4, 128, 3000, 2900, 256
    q, k, v, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, cap, dtype, seed=5, planted=64)
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq)
    dec.refine = refine
    res = dec.step(q, n_valid)
    torch.cuda.synchronize()
    dec.check_flags()
    ref_out, ref_sets, _ = orc.hybrid_step(qn, kn, vn, n_valid, actions, budget)
    got_out = res.outputs.double().cpu().numpy()
    tol = 2e-2 if dtype == "bf16" else 1e-3
    assert max_head_err(got_out, ref_out) < tol
    sel = res.selections.cpu().numpy()
    for l in range(L):
        np.testing.assert_array_equal(sel[res.slot_of_layer[l]], ref_sets[l])


def test_decode_step_graph_replay_equals_eager():
    L, B, Hq, Hkv, d, cap = 4, 1, 8, 2, 128, 4096
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=9, planted=32)
    dec = HybridDecoder(("full", "reuse", "full", "reuse"), k, v, 128, q_heads=Hq)
    res = dec.step(q, cap)
    eager_out = res.outputs.clone()
    eager_idx = res.selections.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cap)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        dec.step(q, cap)
    dec.out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(dec.out, eager_out)
    assert torch.equal(dec.idx[..., :128], eager_idx)


def test_policy_must_start_full():
    q, k, v, *_ = make_stack(2, 1, 4, 2, 64, 128, "bf16")
    with pytest.raises(InvalidInputError):
        HybridDecoder(("reuse", "full"), k, v, 8, q_heads=4)


@pytest.mark.parametrize("schedule", ["pipelined", "sequential", "sequential-noprefetch"])
def test_pipelined_schedules_match_fused(schedule):
    from paper_2602_00777_b200.engine import LayerwiseDecoder, PipelinedDecoder
    L, B, Hq, Hkv, d, cap, budget = 8, 2, 16, 4, 128, 4096, 256
    q, k, v, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=21, planted=64)
    actions = ("full", "reuse", "full", "full", "reuse", "reuse", "full", "reuse")
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq).step(q, cap)
    ref_out, ref_idx = ref.outputs.clone(), ref.selections.clone()
    if schedule.startswith("sequential"):
        dec = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq,
                               prefetch=schedule == "sequential")
    else:
        dec = PipelinedDecoder(actions, k, v, budget, q_heads=Hq, schedule=schedule)
    res = dec.step(q, cap)
    torch.cuda.synchronize()
    assert torch.equal(res.selections, ref_idx)
    # two bf16 evaluations with different split-K merges: each is ~1e-3 from float64
    o, r = res.outputs.double().cpu().numpy(), ref_out.double().cpu().numpy()
    assert max_head_err(o, r) < 4e-3
    # graph capture of the two-stream DAG
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cap)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, cap)
    dec.out.zero_()
    dec.idx.zero_()
    gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(dec.idx[..., :budget], ref_idx)
    assert max_head_err(dec.out.double().cpu().numpy(), r) < 4e-3


@pytest.mark.parametrize("zero_copy,single,q_copy", [
    (False, "auto", "auto"), (True, "auto", False), (True, "auto", True), (True, True, False),
    (True, True, True), (True, True, "auto")])
def test_decode_loop_host_io_graph(zero_copy, single, q_copy):
    """DecodeLoop: H2D (q + new K/V row) -> append -> step -> D2H in one graph launch;
    zero_copy=True: rows appended and queries read from pinned host memory in place,
    outputs stored by the kernels straight into pinned host memory."""
    from paper_2602_00777_b200.engine import DecodeLoop
    L, B, Hq, Hkv, d, cap, budget = 9, 2, 8, 2, 128, 2048, 128
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=13, planted=16)
    actions = ("full", "reuse", "full", "reuse", "reuse", "full", "reuse", "reuse", "reuse")
    dec = HybridDecoder(actions, k.clone(), v.clone(), budget, q_heads=Hq, single_launch=single)
    assert dec.single == (single is True)
    pos = 1500
    loop = DecodeLoop(dec, pos, zero_copy=zero_copy, q_copy=q_copy)
    g = torch.Generator().manual_seed(3)
    for step in range(3):
        qh = torch.randn((L, B, Hq, d), generator=g).to(torch.bfloat16)
        kh = torch.randn((L, B, Hkv, d), generator=g).to(torch.bfloat16)
        vh = torch.randn((L, B, Hkv, d), generator=g).to(torch.bfloat16)
        loop.q_host.copy_(qh)
        loop.k_host.copy_(kh)
        loop.v_host.copy_(vh)
        out = loop.run().clone()
        # eager reference on a separate cache with the same appended row
        k2, v2 = k.clone(), v.clone()
        k2[:, :, :, pos] = kh.cuda()
        v2[:, :, :, pos] = vh.cuda()
        assert torch.equal(dec.k[:, :, :, pos].cpu(), kh) and torch.equal(dec.v, v2)
        ref = HybridDecoder(actions, k2, v2, budget, q_heads=Hq).step(qh.cuda(), pos + 1)
        torch.cuda.synchronize()
        assert torch.equal(dec.idx, ref.selections)
        assert torch.equal(out, ref.outputs.cpu())
        # the per-layer index sets reach the pinned host buffer in the same launch(es)
        assert torch.equal(loop.sel_host, ref.selections.cpu())


@pytest.mark.parametrize("actions", [
    ("full", "reuse", "full", "full", "reuse", "reuse", "full", "reuse", "full", "full"),
    ("full", "full", "reuse", "reuse"),
])
def test_dual_stream_step_matches_single_stream(actions):
    """hylra_decode_step_ex with a side stream (no fusion): FULL(A) -> FULL(B) -> REUSE on the
    caller's stream, SELECT(A) / SELECT(B) on the side stream. Same selections; outputs
    within split-K rounding of the one-stream step; also under CUDA-graph capture."""
    L = len(actions)
    B, Hq, Hkv, d, cap, budget = 2, 16, 4, 128, 4096, 256
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=31, planted=64)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq).step(q, cap)
    ref_out, ref_idx = ref.outputs.clone(), ref.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, dual_stream=True, fuse_select=False)
    assert dec.dual
    res = dec.step(q, cap)
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(res.selections, ref_idx)
    r = ref_out.double().cpu().numpy()
    assert max_head_err(res.outputs.double().cpu().numpy(), r) < 4e-3
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, cap)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, cap)
    dec.out.zero_()
    dec.idx.zero_()
    gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(dec.idx[..., :budget], ref_idx)
    assert max_head_err(dec.out.double().cpu().numpy(), r) < 4e-3


@pytest.mark.parametrize("actions,d,refine,n", [
    (("full", "reuse", "full", "full", "reuse", "reuse", "full", "reuse", "full", "full"), 128, True, 4096),
    (("full", "full", "reuse", "reuse"), 64, True, 3001),
    (("full", "reuse", "full", "reuse"), 128, False, 4096),   # every FULL layer feeds REUSE
    (("full", "full", "reuse", "full", "reuse"), 128, True, 70000),  # 3 bitmap chunks/row
    (("full", "reuse", "full", "reuse"), 128, True, 1500),    # small-row (sorting) path
    (("full", "reuse", "reuse"), 64, True, 200),              # budget >= rows: every index
])
def test_fused_select_step_equals_unfused(actions, d, refine, n):
    """hylra_decode_step_ex fuse_select: the FULL kernel selects the rows of the layers that
    feed REUSE layers itself (last CTA of each pair), the other selections run on the side
    stream under REUSE. Same launches and split-K partitions as the plain step, so outputs
    and selections are bit-identical — eager and under CUDA-graph capture."""
    L = len(actions)
    B, Hq, Hkv, budget = 2, 16, 4, 256
    cap = n
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=41, planted=64)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, refine=refine,
                        fuse_select=False).step(q, n)
    ref_out, ref_idx = ref.outputs.clone(), ref.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, refine=refine, fuse_select=True,
                        single_launch=False)
    assert dec.fused
    res = dec.step(q, n)
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(res.selections, ref_idx)
    assert torch.equal(res.outputs, ref_out)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, n)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, n)
    dec.out.zero_()
    dec.idx.zero_()
    gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(dec.idx[..., :budget], ref_idx)
    assert torch.equal(dec.out, ref_out)


@pytest.mark.parametrize("actions,d,refine,n,B,Hq,Hkv", [
    (("full", "reuse", "full", "full", "reuse", "reuse", "full", "reuse", "full", "full"), 128, True, 4096, 2, 16, 4),
    (("full", "full", "reuse", "reuse"), 64, True, 3001, 2, 16, 4),
    (("full", "reuse", "full", "reuse"), 128, False, 4096, 1, 16, 4),
    (("full", "full", "reuse", "full", "reuse"), 128, True, 70000, 1, 16, 4),
    (("full", "reuse", "full", "reuse"), 128, True, 1500, 3, 16, 4),
    (("full", "reuse", "reuse"), 64, True, 200, 2, 16, 4),
    (("full", "full", "full"), 128, True, 2048, 2, 16, 4),            # no REUSE layer
    (("full",) + ("reuse",) * 15, 128, True, 8192, 4, 16, 4),         # one source, many waiters
    (("full", "reuse", "full", "reuse"), 128, True, 3000, 2, 16, 1),   # G = 16 (both halves)
    (("full", "reuse", "reuse"), 64, True, 2500, 3, 12, 1),            # G = 12, d = 64
])
def test_single_launch_step_equals_unfused(actions, d, refine, n, B, Hq, Hkv):
    """hylra_decode_step_ex fuse_select=2: FULL items (every select fused) and REUSE items
    (waiting on per-row ready flags) in one grid. Same split-K partitions as the plain
    3-launch step, so outputs and selections are bit-identical; repeated eager steps and
    CUDA-graph replays check that the ticket / ready flags reset themselves."""
    L = len(actions)
    budget = 256
    cap = n
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=43, planted=64)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, refine=refine,
                        fuse_select=False).step(q, n)
    ref_out, ref_idx = ref.outputs.clone(), ref.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, refine=refine, single_launch=True)
    assert dec.single and dec.kernels_per_step == 1
    for _ in range(3):
        dec.out.zero_()
        dec.idx.zero_()
        res = dec.step(q, n)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, ref_idx)
        assert torch.equal(res.outputs, ref_out)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.step(q, n)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        dec.step(q, n)
    for _ in range(5):
        dec.out.zero_()
        dec.idx.zero_()
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(dec.idx[..., :budget], ref_idx)
        assert torch.equal(dec.out, ref_out)
    # the synchronisation words and the split-K counters (the fixed region right after the
    # 256-byte flag header: ticket / done + ready flags + group counters, then the FULL and
    # REUSE counter regions of 64 slots x B x Hkv ints each) are back at zero after every step
    n_ready = len(dec.full_layers) * B * Hkv
    sync_end = 256 + -(-(256 + 8 * n_ready) // 256) * 256
    ctr = -(-(4 * 64 * B * Hkv) // 256) * 256
    fixed = dec.ws[256:sync_end + 2 * ctr].view(torch.int32)
    assert int(fixed.abs().sum()) == 0


def test_schedules_bit_identical_at_config2_scale():
    """Regression test for a pipeline-stage release race. The consumer warps released a
    stage (mbarrier arrive) before their last V ldmatrix reads had completed, so the
    producer could refill it early. It showed only at config-2 scale, when a CTA running a
    fused select shared the SM with streaming CTAs: V columns 96..127 of a tile were then
    read from the next tile. Every schedule must reproduce the plain 3-launch step bit for
    bit, on repeated steps."""
    from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch
    cfg = CONFIGS["cfg2"].with_(batch=8, layers=17, full_layers=(0, 1, 2, 8, 15, 16))
    q, k, v = generate_torch(cfg, DEV)
    ref = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads, fuse_select=False)
    ref.step(q, cfg.context)
    torch.cuda.synchronize()
    R, I = ref.out.clone(), ref.idx.clone()
    for kw in ({"fuse_select": True, "single_launch": False}, {"single_launch": True},
               {"fuse_select": False}):
        dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads, **kw)
        for _ in range(3):
            dec.step(q, cfg.context)
            torch.cuda.synchronize()
            assert torch.equal(dec.idx, I), kw
            bad = [l for l in range(cfg.layers) if not torch.equal(dec.out[l], R[l])]
            assert not bad, (kw, bad)
    del q, k, v, ref, dec
    torch.cuda.empty_cache()


def test_autotune_keeps_results_bit_identical():
    """HybridDecoder.autotune times single / singlecoop / fusedsel / dual / fused3 as graph
    replays and keeps the fastest; whichever it keeps, the step's outputs and selections are
    unchanged."""
    L, B, Hq, Hkv, d, cap, budget = 6, 2, 16, 4, 128, 4096, 256
    actions = ("full", "reuse", "full", "full", "reuse", "reuse")
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=47, planted=32)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, fuse_select=False).step(q, cap)
    R, I = ref.outputs.clone(), ref.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq)
    times = dec.autotune(q, cap, reps=3)
    assert set(times) == {"single", "singlecoop", "fusedsel", "dual", "fused3"}
    assert all(t > 0 for t in times.values())
    assert dec.schedule == min(times, key=times.get)
    res = dec.step(q, cap)
    torch.cuda.synchronize()
    assert torch.equal(res.selections, I) and torch.equal(res.outputs, R)
    for name in ("single", "fusedsel", "fused3"):
        dec.set_schedule(name)
        res = dec.step(q, cap)
        torch.cuda.synchronize()
        assert torch.equal(res.selections, I) and torch.equal(res.outputs, R), name
    f32 = HybridDecoder(actions, k.float(), v.float(), budget, q_heads=Hq)
    # fp32 caches run the CUDA-core kernels: the 3-launch step, or the two-stream one
    assert f32.autotune(q.float(), cap, reps=2).keys() == {"dual", "fused3"}


@pytest.mark.parametrize("schedule", ["single", "fusedsel", "fused3"])
def test_step_append_option_equals_separate_append(schedule):
    """hylra_step_options append_*: the step's new K/V rows written inside the step (by the
    single-launch kernel itself: each FULL pair's own row by the split that streams it, the
    REUSE layers' rows by the FULL pair they inherit from; by the append kernel otherwise)
    give the same cache, selections and outputs as hylra_append_kv followed by the step. The
    new row's key is aligned with the queries so every selection contains it."""
    L, B, Hq, Hkv, d, cap, budget = 7, 2, 16, 4, 128, 3000, 192
    actions = ("full", "reuse", "reuse", "full", "full", "reuse", "reuse")
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=53, planted=32)
    pos = 2500
    g = torch.Generator().manual_seed(9)
    qm = q.float().view(L, B, Hkv, Hq // Hkv, d).mean(3)
    k_new = (4.0 * qm / qm.norm(dim=-1, keepdim=True)
             + 0.1 * torch.randn((L, B, Hkv, d), generator=g).cuda()).to(torch.bfloat16)
    v_new = torch.randn((L, B, Hkv, d), generator=g).to(torch.bfloat16)
    k_pinned, v_pinned = k_new.cpu().pin_memory(), v_new.pin_memory()
    k1, v1 = k.clone(), v.clone()
    ref = HybridDecoder(actions, k1, v1, budget, q_heads=Hq, fuse_select=False)
    ref.append(k_pinned, v_pinned, pos)
    r = ref.step(q, pos + 1)
    torch.cuda.synchronize()
    R, I = r.outputs.clone(), r.selections.clone()
    assert bool((I == pos).any(-1).all()), "the new row must be selected everywhere"
    k2, v2 = k.clone(), v.clone()
    dec = HybridDecoder(actions, k2, v2, budget, q_heads=Hq)
    dec.set_schedule(schedule)
    res = dec.step(q, pos + 1, append=(k_pinned, v_pinned, pos))
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(k2, k1) and torch.equal(v2, v1)
    assert torch.equal(res.selections, I) and torch.equal(res.outputs, R)


def test_step_layer_events_chunks_reuse():
    """hylra_decode_step_events: per-layer completion events split the REUSE launch into
    chunks; selections identical, outputs within split-K rounding; events fire."""
    L, B, Hq, Hkv, d, cap, budget = 9, 2, 8, 2, 128, 2048, 128
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=14, planted=16)
    actions = ("full", "reuse", "full", "reuse", "reuse", "full", "reuse", "reuse", "reuse")
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq).step(q, cap)
    ref_out, ref_idx = ref.outputs.clone(), ref.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq)
    evs = [torch.cuda.Event() if l in (0, 1, 4, 7, 8) else None for l in range(L)]
    for e in evs:
        if e is not None:
            e.record()
    wait = torch.cuda.Event()
    wait.record()
    res = dec.step(q, cap, layer_events=evs, reuse_wait=wait)
    torch.cuda.synchronize()
    assert all(e.query() for e in evs if e is not None)
    assert torch.equal(res.selections, ref_idx)
    o, r = res.outputs.double().cpu().numpy(), ref_out.double().cpu().numpy()
    assert max_head_err(o, r) < 4e-3


def test_append_kv_from_device_and_pinned_host():
    """hylra_append_kv writes [L, B, Hkv, d] rows at cache row pos of the chosen layers."""
    L, B, Hq, Hkv, d, cap = 3, 2, 8, 2, 64, 100
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=5)
    dec = HybridDecoder(("full", "reuse", "full"), k, v, 8, q_heads=Hq)
    k0, v0 = k.clone(), v.clone()
    rows_k = torch.randn((L, B, Hkv, d)).to(torch.bfloat16)
    rows_v = torch.randn((L, B, Hkv, d)).to(torch.bfloat16)
    dec.append(rows_k.cuda(), rows_v.cuda(), 7, layers=[1])
    dec.append(rows_k.pin_memory(), rows_v.pin_memory(), 99, layers=[0, 2])
    torch.cuda.synchronize()
    k0[1, :, :, 7] = rows_k[1].cuda()
    v0[1, :, :, 7] = rows_v[1].cuda()
    k0[[0, 2], :, :, 99] = rows_k[[0, 2]].cuda()
    v0[[0, 2], :, :, 99] = rows_v[[0, 2]].cuda()
    assert torch.equal(k, k0) and torch.equal(v, v0)
    with pytest.raises(InvalidInputError):
        dec.append(rows_k.cuda(), rows_v.cuda(), cap)


@pytest.mark.parametrize("where", ["k", "v", "q"])
def test_non_finite_inputs_raise_numeric_error(where):
    """Non-finite cache or query values -> NumericInputError (attention.py:43-44,205-206)."""
    from paper_2602_00777_b200 import NumericInputError
    L, B, Hq, Hkv, d, cap = 2, 1, 8, 2, 128, 1024
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=2)
    {"k": k, "v": v}.get(where, q).view(-1)[777] = float("nan") if where != "k" else float("inf")
    dec = HybridDecoder(("full", "reuse"), k, v, 64, q_heads=Hq)
    dec.step(q, cap)
    torch.cuda.synchronize()
    with pytest.raises(NumericInputError):
        dec.check_flags()


def _embed(rows, d=32):
    """2-D reference fixtures embedded in d dims (zero padding keeps every dot product)."""
    x = torch.zeros((len(rows), d), dtype=torch.float32)
    x[:, :2] = torch.tensor(rows, dtype=torch.float64).float()
    return x


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_known_answers_on_gpu(dtype):
    """The reference's known-answer tests through the kernels (tests/test_attention.py:33-59,
    100-105, 192-200). The 2-D fixtures are zero-padded to d = 32 (f32) / 64 (bf16) and the
    query is scaled by sqrt(d / 2), so logits equal the reference's q.k / sqrt(2) (in bf16 up
    to the rounding of that scaled query, inside the 2e-3 tolerance)."""
    import math
    d = 32 if dtype == "f32" else 64
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    tol = 1e-6 if dtype == "f32" else 2e-3
    s = math.sqrt(d / 2)

    def attend(q2, keys, values):
        q = (_embed([q2], d) * s).to(dt).view(1, 1, 1, d).to(DEV)
        k = _embed(keys, d).to(dt).view(1, 1, 1, len(keys), d).to(DEV)
        v = _embed(values, d).to(dt).view(1, 1, 1, len(values), d).to(DEV)
        return q, k, v

    # single token: the output is its value row
    q, k, v = attend([0.5, 0.5], [[1.0, 2.0]], [[5.0, -3.0]])
    out, _ = full_attention(q, k, v)
    assert torch.allclose(out[0, 0, 0, :2].cpu(), torch.tensor([5.0, -3.0]), rtol=tol, atol=tol)
    # orthogonal query: uniform weights
    q, k, v = attend([0.0, 1.0], [[1.0, 0.0], [2.0, 0.0], [-1.0, 0.0]],
                     [[3.0, 0.0], [0.0, 3.0], [0.0, 0.0]])
    out, _ = full_attention(q, k, v)
    assert torch.allclose(out[0, 0, 0, :2].cpu(), torch.tensor([1.0, 1.0]), rtol=tol, atol=tol)
    # two-token fixture [[10, 0], [0, 0]]: logit 10 / sqrt(2), weight 1 / (1 + e^-l)
    q, k, v = attend([1.0, 0.0], [[10.0, 0.0], [0.0, 0.0]], [[1.0, 0.0], [0.0, 1.0]])
    out, sc = full_attention(q, k, v)
    w1 = 1.0 / (1.0 + math.exp(-10 / math.sqrt(2)))
    assert abs(float(sc[0, 0, 0, 0]) - 10 / math.sqrt(2)) < 10 * tol
    assert torch.allclose(out[0, 0, 0, :2].cpu().double(), torch.tensor([w1, 1 - w1],
                          dtype=torch.float64), rtol=tol, atol=tol)
    # subset fixture: selection {0, 2}, softmax renormalised over the subset
    keys = [[10.0, 0.0], [0.0, 0.0], [1.0, 1.0], [-2.0, 0.5]]
    values = [[1.0, 0.0], [0.0, 1.0], [2.0, 2.0], [3.0, -1.0]]
    q, k, v = attend([1.0, 0.0], keys, values)
    idx = torch.tensor([[[[0, 2]]]], dtype=torch.int32, device=DEV)
    got = sparse_attention(q, k, v, idx)
    l0, l2 = 10 / math.sqrt(2), 1 / math.sqrt(2)
    w0 = 1 / (1 + math.exp(l2 - l0))
    want = torch.tensor([w0 * 1 + (1 - w0) * 2, (1 - w0) * 2], dtype=torch.float64)
    assert torch.allclose(got[0, 0, 0, :2].cpu().double(), want, rtol=tol, atol=tol)
    # top-k ties and saturation
    for row, budget, want in (([3.0, 1.0, 2.0], 2, [0, 2]), ([5.0, 5.0, 5.0], 2, [0, 1]),
                              ([1.0, 2.0], 10, [0, 1])):
        buf = torch.zeros((1, 1, 1, 8), dtype=torch.float32)
        buf[0, 0, 0, :len(row)] = torch.tensor(row)
        got = topk_select(buf.to(DEV), budget, len(row))
        assert got[0, 0, 0].cpu().tolist() == want


@pytest.mark.parametrize("sinks,recent,n", [(4, 16, 4096), (0, 64, 3000), (8, 0, 2048),
                                            (3000, 3000, 2500)])
def test_single_launch_with_sinks_recent(sinks, recent, n):
    """Sink / recent augmentation (engine.py:122-126) inside the single-launch step: the
    final CTA of each FULL pair writes the augmented row after its select; identical to the
    multi-launch step with the augment kernel (including ranges that cover every token)."""
    L, B, Hq, Hkv, d, budget = 6, 2, 16, 4, 128, 256
    actions = ("full", "reuse", "full", "reuse", "reuse", "full")
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=61, planted=32)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, include_sinks=sinks,
                        include_recent=recent, fuse_select=False, single_launch=False)
    r = ref.step(q, n)
    torch.cuda.synchronize()
    R, S = r.outputs.clone(), r.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, include_sinks=sinks,
                        include_recent=recent, single_launch=True)
    assert dec.single and dec.kernels_per_step == 1
    for _ in range(2):
        res = dec.step(q, n)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, S)
        assert torch.equal(res.outputs, R)


def test_single_launch_at_the_longest_row():
    """The single-launch step at the longest supported row (262144 tokens: the fused select's
    bitmap, band list and candidates in the FULL kernel's drained ring) is bit-identical to
    the 3-launch step."""
    L, B, Hq, Hkv, d, n, budget = 3, 1, 8, 2, 128, 262144, 4096
    actions = ("full", "reuse", "reuse")
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=71, planted=256)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, fuse_select=False,
                        single_launch=False).step(q, n)
    torch.cuda.synchronize()
    R, S = ref.outputs.clone(), ref.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, single_launch=True)
    res = dec.step(q, n)
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(res.selections, S) and torch.equal(res.outputs, R)


@pytest.mark.parametrize("sel_group,Hkv,Hq,B", [(2, 4, 16, 2), (4, 4, 16, 1), (8, 8, 8, 1)])
def test_single_launch_with_selection_groups(sel_group, Hkv, Hq, B):
    """Selection rows that sum several KV heads (sel_group > 1; sel_group = Hkv is the
    reference's layer-wide set): in the single-launch step the last FULL pair of each group
    to finish selects (a self-resetting per-group counter); identical to the multi-launch
    step, over repeated steps."""
    L, d, n, budget = 5, 128, 3000, 192
    actions = ("full", "reuse", "full", "reuse", "reuse")
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=67, planted=32)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, sel_group=sel_group,
                        fuse_select=False, single_launch=False)
    r = ref.step(q, n)
    torch.cuda.synchronize()
    R, S = r.outputs.clone(), r.selections.clone()
    dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, sel_group=sel_group,
                        single_launch=True)
    assert dec.single and dec.kernels_per_step == 1
    for _ in range(3):
        res = dec.step(q, n)
        torch.cuda.synchronize()
        dec.check_flags()
        assert torch.equal(res.selections, S)
        assert torch.equal(res.outputs, R)


def test_layerwise_prefetch_matches_waiting_launches_across_steps():
    """LayerwiseDecoder's early loads (K/V and indices before griddepcontrol.wait) never read
    stale data: with queries alternating between steps (so every step's selections differ
    from the previous step's), the prefetching decoder equals the waiting one bit for bit,
    eagerly and as CUDA-graph replays."""
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    L, B, Hq, Hkv, d, cap, budget = 8, 2, 16, 4, 128, 8192, 512
    q1, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=5, planted=64)
    q2 = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=6, planted=64)[0]
    actions = ("full", "reuse", "reuse", "full", "full", "reuse", "reuse", "reuse")
    pre = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq, prefetch=True)
    wait = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq, prefetch=False)
    for qq in (q1, q2, q1, q2):
        a, b = pre.step(qq, cap), wait.step(qq, cap)
        torch.cuda.synchronize()
        assert torch.equal(a.outputs, b.outputs) and torch.equal(a.selections, b.selections)
    pre.check_flags(strict=True)
    qs = q1.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pre.step(qs, cap)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        pre.step(qs, cap)
    for qq in (q2, q1, q2):
        qs.copy_(qq)
        gr.replay()
        ref = wait.step(qq, cap)
        torch.cuda.synchronize()
        assert torch.equal(pre.out, ref.outputs)
        assert torch.equal(pre.idx[..., :budget], ref.selections)


@pytest.mark.parametrize("dtype,d,Hq,Hkv,cap,n_valid,budget,sel_group", [
    ("bf16", 128, 28, 4, 4096, 4000, 300, 1),   # G = 7 (Qwen), ragged rows
    ("bf16", 64, 16, 4, 2048, 2048, 128, 4),    # layer-wide sets (the reference's sel_group)
    ("f32", 64, 8, 2, 1024, 1000, 100, 1),      # CUDA-core path (no early loads)
    ("bf16", 128, 16, 1, 8192, 8192, 8192, 1),  # budget covers the cache
])
def test_layerwise_decoder_matches_oracle(dtype, d, Hq, Hkv, cap, n_valid, budget, sel_group):
    """LayerwiseDecoder (hylra_decode_layer per layer) against the float64 oracle's step
    (engine.py:167-197): exact index sets, outputs within the dtype tolerance."""
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    L, B = 6, 2
    q, k, v, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, cap, dtype, seed=d + Hq, planted=48)
    actions = ("full", "reuse", "full", "full", "reuse", "reuse")
    dec = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq, sel_group=sel_group)
    res = dec.step(q, n_valid)
    torch.cuda.synchronize()
    dec.check_flags(strict=True)
    ref_out, ref_sets, _ = orc.hybrid_step(qn, kn, vn, n_valid, actions, budget,
                                           sel_group=sel_group)
    sel = res.selections.cpu().numpy()
    for l in range(L):
        np.testing.assert_array_equal(sel[res.slot_of_layer[l]], ref_sets[l])
    tol = 2e-2 if dtype == "bf16" else 1e-3
    assert max_head_err(res.outputs.double().cpu().numpy(), ref_out) < tol


@pytest.mark.parametrize("d,Hq,Hkv,cap,k", [(128, 32, 8, 4096, 1000), (64, 14, 2, 2048, 333),
                                            (128, 28, 4, 8192, 2048), (128, 16, 16, 512, 64)])
def test_reuse_tma_gather_equals_cp_async_gather(d, Hq, Hkv, cap, k):
    """The REUSE gather by TMA row gathers (tile::gather4 over 2-D row views of the cache)
    returns exactly the cp.async gather's outputs: same rows, same swizzled tile layout,
    ragged last tiles zero-filled."""
    from paper_2602_00777_b200 import _abi
    q, k_, v, *_ = make_stack(3, 2, Hq, Hkv, d, cap, "bf16", seed=k)
    rng = np.random.default_rng(d + k)
    idx = np.stack([np.stack([np.stack([np.sort(rng.choice(cap, k, replace=False))
                                        for _ in range(Hkv)]) for _ in range(2)])
                    for _ in range(3)]).astype(np.int32)
    it = torch.from_numpy(idx).to(DEV)
    with _abi.tuning(gather_tma=0):
        ref = sparse_attention(q, k_, v, it, cap)
    with _abi.tuning(gather_tma=1):
        got = sparse_attention(q, k_, v, it, cap)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


def test_layerwise_decoder_with_model_dependence():
    """A model's decode: layer l+1's query is computed from layer l's output by the model's
    own (torch) kernel on the same stream, between LayerwiseDecoder.layer calls. The GPU step
    must use the queries as they are when each layer runs: the float64 oracle, given the
    final query stack, reproduces every index set and output. (Were a layer to read its query
    before the model kernel wrote it, it would see the initial values, far from the final
    ones.)"""
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    L, B, Hq, Hkv, d, cap, budget = 6, 2, 16, 4, 128, 4096, 256
    q0, k, v, _, kn, vn = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=31, planted=64)
    actions = ("full", "reuse", "reuse", "full", "reuse", "full")
    dec = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq)
    for _ in range(2):  # the second step runs on warm, non-zero workspaces / buffers
        q = q0.clone()
        for l in range(L):
            if l > 0:
                # the "model": the next query mixes the previous layer's output in
                q[l] = (0.25 * q0[l].float() + 8.0 * dec.out[l - 1]).to(torch.bfloat16)
            dec.layer(l, q, cap)
        dec.finish()
        torch.cuda.synchronize()
    dec.check_flags(strict=True)
    assert (q[1:].float() - q0[1:].float()).abs().mean() > 0.3  # the chain really moved q
    ref_out, ref_sets, _ = orc.hybrid_step(q.double().cpu().numpy(), kn, vn, cap, actions,
                                           budget)
    sel = dec.idx[..., :budget].cpu().numpy()
    for l in range(L):
        np.testing.assert_array_equal(sel[dec.slot_of_layer[l]], ref_sets[l])
    assert max_head_err(dec.out.double().cpu().numpy(), ref_out) < 2e-2


def test_layerwise_decoder_growing_rows_and_flags():
    """LayerwiseDecoder across steps with a growing cache (n_valid 3000 -> 4096: workspaces
    grow, splits change) equals HybridDecoder's selections at every step, refinement off;
    a non-finite score raises NumericInputError from check_flags, whichever of its
    workspaces holds the flag, and clear_flags resets them."""
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    from paper_2602_00777_b200.errors import NumericInputError
    L, B, Hq, Hkv, d, cap, budget = 5, 2, 16, 4, 128, 4096, 300
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=77, planted=40)
    actions = ("full", "reuse", "full", "reuse", "full")
    lw = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq, refine=False)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, refine=False)
    for n in (3000, 3500, 4096, 3001):
        a, r = lw.step(q, n), ref.step(q, n)
        torch.cuda.synchronize()
        assert torch.equal(a.selections, r.selections), n
    lw.check_flags(strict=True)
    q_bad = q.clone()
    q_bad[2, 1, 5, 7] = float("nan")
    lw.step(q_bad, cap)
    torch.cuda.synchronize()
    with pytest.raises(NumericInputError):
        lw.check_flags()
    lw.clear_flags()
    lw.step(q, cap)
    torch.cuda.synchronize()
    lw.check_flags(strict=True)


@pytest.mark.parametrize("B,Hq,Hkv,cap,budget", [(1, 32, 8, 32768, 2048), (2, 28, 4, 16384, 1024),
                                                 (1, 16, 2, 8192, 333)])
def test_bulk_merge_equals_l2_merge(B, Hq, Hkv, cap, budget):
    """The split-K final merge staging a pair's partials by cp.async.bulk (bulk_merge=1, the
    default) returns exactly the L2-load merge's outputs, for one-layer FULL launches (~37
    splits per pair at B=1, partials up to 74 KB; G=7 too large for the staging area at some
    split counts, so the fallback is covered) and REUSE launches, layer-sequential."""
    from paper_2602_00777_b200 import _abi
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    L = 4
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, 128, cap, "bf16", seed=cap + budget, planted=64)
    actions = ("full", "reuse", "full", "reuse")
    outs = {}
    for m in ((0, 0), (1, 0), (0, 1), (1, 1)):
        with _abi.tuning(bulk_merge=m[0], cluster_merge=m[1]):
            dec = LayerwiseDecoder(actions, k, v, budget, q_heads=Hq)
            res = dec.step(q, cap)
            torch.cuda.synchronize()
            dec.check_flags(strict=True)
            outs[m] = (res.outputs.clone(), res.selections.clone())
    for m in outs:
        assert torch.equal(outs[m][0], outs[(0, 0)][0]), m
        assert torch.equal(outs[m][1], outs[(0, 0)][1]), m


@pytest.mark.parametrize("d,Hq,Hkv,cap,k,L,B", [(128, 32, 8, 32768, 2048, 1, 1),
                                                (128, 32, 8, 8192, 1000, 2, 2),
                                                (64, 14, 2, 4096, 333, 1, 1),
                                                (128, 28, 4, 16384, 2048, 1, 3),
                                                (128, 64, 4, 4096, 700, 1, 1),
                                                (128, 32, 8, 16384, 4096, 1, 1),
                                                (64, 16, 2, 4096, 1000, 1, 1)])
def test_reuse_cluster_merge_equals_global_merge(d, Hq, Hkv, cap, k, L, B):
    """A REUSE launch split 2-8 ways under one wave merges its splits through the CTA
    cluster's distributed shared memory (cluster_merge=1, the default): bit-identical to
    the global split-K merge, for d 64 / 128, G 4 / 7 / 16, ragged selections, clusters of
    2 to 16 (non-portable) CTAs."""
    from paper_2602_00777_b200 import _abi
    q, k_, v, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=k + B)
    rng = np.random.default_rng(d + k + B)
    idx = np.stack([np.stack([np.stack([np.sort(rng.choice(cap, k, replace=False))
                                        for _ in range(Hkv)]) for _ in range(B)])
                    for _ in range(L)]).astype(np.int32)
    it = torch.from_numpy(idx).to(DEV)
    with _abi.tuning(cluster_merge=0):
        ref = sparse_attention(q, k_, v, it, cap)
    with _abi.tuning(cluster_merge=1):
        got = sparse_attention(q, k_, v, it, cap)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


def test_fused_fine_splits_keep_selections():
    """Tuning knob fused_fine_splits: the fused-select FULL launch over few pairs takes finer
    split-K partitions. Selections stay bit-identical; outputs move only at bf16 level (P
    is rounded to bf16 against another running max) and stay deterministic."""
    from paper_2602_00777_b200 import _abi
    actions = ("full", "reuse", "full", "full", "reuse", "reuse")
    L, B, Hq, Hkv, d, n, budget = len(actions), 1, 32, 8, 128, 32768, 2048
    q, k, v, *_ = make_stack(L, B, Hq, Hkv, d, n, "bf16", seed=77, planted=64)
    ref = HybridDecoder(actions, k, v, budget, q_heads=Hq, fuse_select=True,
                        single_launch=False).step(q, n)
    ref_out, ref_idx = ref.outputs.clone(), ref.selections.clone()
    with _abi.tuning(fused_fine_splits=1):
        dec = HybridDecoder(actions, k, v, budget, q_heads=Hq, fuse_select=True,
                            single_launch=False)
        a = dec.step(q, n)
        a_out = a.outputs.clone()
        b = dec.step(q, n)
        torch.cuda.synchronize()
        dec.check_flags(strict=True)
    assert torch.equal(a.selections, ref_idx)
    assert torch.equal(b.outputs, a_out)
    scale = ref_out.abs().amax(dim=-1, keepdim=True).clamp_min(1e-30)
    assert float(((a_out - ref_out).abs() / scale).max()) < 2e-2
