"""The CUDA kernels under multi-GPU sharding, two ranks on one GPU.

Each rank is its own process with its own CUDA context (gloo process group: the ranks
share the device, and nothing on the attention path waits on another rank). Rank r
decodes only its shard — KV heads [r*Hkv/2, (r+1)*Hkv/2) with their query heads
(Llama-shaped, "kvhead"), or sequences [r*B/2, (r+1)*B/2) (Qwen-shaped, "batch") — through
the same HybridDecoder over strided views of the full cache (no copies), then the outputs
are all-gathered once. The gathered outputs and every shard-local index set must equal
the unsharded GPU step bit for bit. The shapes keep the split-K partition the same at
both pair counts (bit-equality needs identical partitions; 4 splits of 32 tiles per FULL
pair, 1 per REUSE pair: 4-tile selections stay unsplit at either pair count), which
bench.py's shard sizes do not need.
"""
import os
import socket

import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

import torch.multiprocessing as mp  # noqa: E402

ACTIONS = ("full", "full", "reuse", "full", "reuse", "reuse", "full", "reuse")
SHAPES = {"kvhead": dict(B=8, Hq=32, Hkv=8), "batch": dict(B=8, Hq=28, Hkv=4)}
N, BUDGET, D = 8192, 256, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data(mode):
    from paper_2602_00777_b200.synthetic import StackConfig, generate_torch
    sh = SHAPES[mode]
    cfg = StackConfig("shard", len(ACTIONS), sh["B"], sh["Hq"], sh["Hkv"], D, N, BUDGET, "bf16",
                      tuple(l for l, a in enumerate(ACTIONS) if a == "full"), 64, 0.9, seed=5)
    return cfg, generate_torch(cfg, "cuda")


def _worker(rank, world, port, mode, schedule, out_dir):
    import torch.distributed as dist

    from paper_2602_00777_b200.engine import HybridDecoder
    from paper_2602_00777_b200.sharding import gather_outputs, plan_shards, shard_slices
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, (q, k, v) = _data(mode)
        plan = plan_shards(cfg.kv_heads, cfg.q_heads, cfg.batch, world, mode=mode)[rank]
        qs, ks, vs = shard_slices(plan, q, k, v)
        dec = HybridDecoder(ACTIONS, ks, vs, BUDGET, q_heads=qs.shape[2])
        dec.set_schedule(schedule)
        res = dec.step(qs.contiguous(), N)
        torch.cuda.synchronize()
        dec.check_flags(strict=True)
        full = gather_outputs(res.outputs, plan)
        torch.save({"out": full.cpu(), "sel": res.selections.cpu(), "plan": plan},
                   os.path.join(out_dir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["kvhead", "batch"])
@pytest.mark.parametrize("schedule", ["single", "fused3"])
def test_two_rank_cuda_shards_equal_unsharded_step(mode, schedule, tmp_path):
    from paper_2602_00777_b200.engine import HybridDecoder
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, schedule, str(tmp_path)))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    cfg, (q, k, v) = _data(mode)
    dec = HybridDecoder(ACTIONS, k, v, BUDGET, q_heads=cfg.q_heads)
    dec.set_schedule(schedule)
    ref = dec.step(q, N)
    torch.cuda.synchronize()
    ref_out, ref_sel = ref.outputs.cpu(), ref.selections.cpu()
    for r in range(2):
        got = torch.load(tmp_path / f"rank{r}.pt", weights_only=False)
        assert torch.equal(got["out"], ref_out), f"rank {r}: gathered outputs differ"
        plan = got["plan"]
        b0, b1 = plan.batch
        h0, h1 = plan.kv_heads
        assert torch.equal(got["sel"], ref_sel[:, b0:b1, h0:h1]), f"rank {r}: index sets differ"
