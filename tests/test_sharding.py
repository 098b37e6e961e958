"""Multi-GPU partitioning, exercised on CPU with the gloo backend (world size 2).

Each rank computes the outputs of its shard only (here with the float64 oracle standing
in for the kernels: the test is about the partition and the once-per-step gather, which
are identical code on NCCL), all-gathers them, and the result must equal the unsharded
oracle step bit for bit; index sets stay shard-local.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hylra_oracle as orc
from paper_2602_00777_b200.errors import ConfigurationError
from paper_2602_00777_b200.sharding import gather_outputs, plan_shards, shard_slices


def test_plan_kvhead_and_batch():
    plans = plan_shards(8, 32, 4, 8)
    assert [p.mode for p in plans] == ["kvhead"] * 8
    assert plans[3].kv_heads == (3, 4) and plans[3].q_heads == (12, 16)
    assert plans[3].batch == (0, 4)
    qwen = plan_shards(4, 28, 16, 8)
    assert all(p.mode == "batch" for p in qwen)
    assert qwen[5].batch == (10, 12) and qwen[5].kv_heads == (0, 4)
    with pytest.raises(ConfigurationError):
        plan_shards(4, 28, 6, 8)
    with pytest.raises(ConfigurationError):
        plan_shards(8, 32, 4, 3, mode="kvhead")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _make(seed=0):
    rng = np.random.default_rng(seed)
    L, B, Hq, Hkv, d, N = 3, 4, 8, 4, 16, 96
    q = rng.standard_normal((L, B, Hq, d))
    k = rng.standard_normal((L, B, Hkv, N, d))
    v = rng.standard_normal((L, B, Hkv, N, d))
    return q, k, v


ACTIONS = ("full", "reuse", "full")


def _step(q, k, v, blocks):
    """The oracle step standing in for the kernels: token mode (budget 10) or block mode
    (block budget 3 of 8-token blocks)."""
    if blocks:
        out, sets = orc.hybrid_step_blocks(q, k, v, k.shape[3], ACTIONS, 3, 8)
        return out, sets
    out, sets, _ = orc.hybrid_step(q, k, v, k.shape[3], ACTIONS, 10)
    return out, sets


def _worker(rank, world, port, mode, q, blocks=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        qn, kn, vn = _make()
        L, B, Hq, d = qn.shape
        plan = plan_shards(kn.shape[2], Hq, B, world, mode=mode)[rank]
        qs, ks, vs = shard_slices(plan, torch.from_numpy(qn), torch.from_numpy(kn),
                                  torch.from_numpy(vn))
        out, sets = _step(qs.numpy(), ks.numpy(), vs.numpy(), blocks)
        full = gather_outputs(torch.from_numpy(out), plan)
        q.put((rank, full.numpy(), {l: sets[l] for l in sets}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,blocks", [("kvhead", False), ("batch", False),
                                         ("kvhead", True)])
def test_gloo_two_rank_step_equals_unsharded(mode, blocks):
    """Token mode, and block mode (its block sets are per (b, kv-head) row too)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q, blocks))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (o, s)) for r, o, s in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    qn, kn, vn = _make()
    ref, ref_sets = _step(qn, kn, vn, blocks)
    for r in range(2):
        assert np.array_equal(res[r][0], ref)  # replicated, identical on both ranks
    # shard-local index sets equal the corresponding slices of the unsharded sets
    for r in range(2):
        plan = plan_shards(kn.shape[2], qn.shape[2], qn.shape[1], 2, mode=mode)[r]
        for l in range(3):
            b0, b1 = plan.batch
            h0, h1 = plan.kv_heads
            assert np.array_equal(res[r][1][l], ref_sets[l][b0:b1, h0:h1])


def _agree_worker(rank, world, port, q):
    from paper_2602_00777_b200.sharding import agree_schedule
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank's own autotune prefers a different schedule; singlecoop is missing on
        # rank 1 (a schedule a rank did not time)
        mine = [{"single": 1.50, "singlecoop": 1.40, "fusedsel": 1.55, "fused3": 1.60},
                {"single": 1.45, "fusedsel": 1.70, "fused3": 1.52}][rank]
        q.put((rank, agree_schedule(mine)))
    finally:
        dist.destroy_process_group()


def test_ranks_agree_on_one_schedule():
    """bench.py under torchrun: every rank must time the same schedule (the timed loops
    hold matching collectives; differing per-rank autotune picks deadlocked a 2-rank run).
    The agreed schedule is the fastest by its max over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    name, times = res[0]
    assert name == "single" and times == {"single": 1.50, "fusedsel": 1.70, "fused3": 1.60}
