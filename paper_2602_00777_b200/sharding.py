"""Multi-GPU partitioning of the hybrid decode step (one process per GPU).

SURVEY.md §8(e): every kernel is independent per (batch, KV head) and top-k reuse is
per-KV-head and shard-local, so the step shards with no exchange at all:

* "kvhead": rank p owns KV heads [p*Hkv/P, (p+1)*Hkv/P) and their query heads, for all
  layers and sequences (Llama-3-8B shape, Hkv = 8 >= P);
* "batch":  rank p owns sequences [p*B/P, (p+1)*B/P) (Qwen2.5-7B shape, Hkv = 4 < P).

The only collective is an optional all-gather of the per-shard outputs, once per step,
for callers that need them replicated (NCCL over NVLink; gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigurationError

__all__ = ["ShardPlan", "plan_shards", "shard_slices", "gather_outputs", "agree_schedule"]


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    mode: str            # "kvhead" or "batch"
    kv_heads: tuple      # [start, stop) of KV heads owned
    q_heads: tuple       # [start, stop) of query heads owned
    batch: tuple         # [start, stop) of sequences owned


def plan_shards(kv_heads: int, q_heads: int, batch: int, world: int,
                mode: str | None = None) -> list:
    """Partition plan for `world` ranks; prefers KV-head sharding when it divides."""
    if world < 1:
        raise ConfigurationError(f"world size must be >= 1, got {world}")
    if q_heads % kv_heads:
        raise ConfigurationError("q_heads must be a multiple of kv_heads")
    G = q_heads // kv_heads
    if mode is None:
        mode = "kvhead" if kv_heads % world == 0 else "batch"
    plans = []
    for r in range(world):
        if mode == "kvhead":
            if kv_heads % world:
                raise ConfigurationError(f"{kv_heads} KV heads do not split over {world} ranks")
            per = kv_heads // world
            kh = (r * per, (r + 1) * per)
            plans.append(ShardPlan(r, world, mode, kh, (kh[0] * G, kh[1] * G), (0, batch)))
        elif mode == "batch":
            if batch % world:
                raise ConfigurationError(f"batch {batch} does not split over {world} ranks")
            per = batch // world
            plans.append(ShardPlan(r, world, mode, (0, kv_heads), (0, q_heads),
                                   (r * per, (r + 1) * per)))
        else:
            raise ConfigurationError(f"unknown shard mode {mode!r}")
    return plans


def shard_slices(plan: ShardPlan, q, k, v):
    """Views of q [L,B,Hq,d] and k/v [L,B,Hkv,cap,d] owned by `plan` (no copies)."""
    b0, b1 = plan.batch
    h0, h1 = plan.kv_heads
    q0, q1 = plan.q_heads
    return q[:, b0:b1, q0:q1], k[:, b0:b1, h0:h1], v[:, b0:b1, h0:h1]


def gather_outputs(out_local, plan: ShardPlan, group=None):
    """All-gather per-shard outputs [L, B_local, Hq_local, d] into the full
    [L, B, Hq, d] tensor on every rank (one collective per step)."""
    import torch
    import torch.distributed as dist

    if plan.world == 1:
        return out_local
    src = out_local.contiguous()
    if src.is_cuda and dist.get_backend(group) == "nccl":
        buf = torch.empty((plan.world,) + tuple(src.shape), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(buf, src, group=group)
    else:  # gloo (CPU tests; ranks sharing a GPU in a functional check)
        host = src.cpu()
        parts = [torch.empty_like(host) for _ in range(plan.world)]
        dist.all_gather(parts, host, group=group)
        buf = torch.stack(parts).to(src.device)
    if plan.mode == "kvhead":
        # [P, L, B, Hq/P, d] -> [L, B, P*Hq/P, d]
        return buf.permute(1, 2, 0, 3, 4).reshape(
            out_local.shape[0], out_local.shape[1], -1, out_local.shape[3])
    # batch: [P, L, B/P, Hq, d] -> [L, P*B/P, Hq, d]
    return buf.permute(1, 0, 2, 3, 4).reshape(out_local.shape[0], -1, out_local.shape[2],
                                              out_local.shape[3])


SCHEDULES = ("single", "singlecoop", "fusedsel", "dual", "fused3")


def agree_schedule(times: dict, group=None, device="cpu"):
    """One step schedule for every rank: each rank autotunes its own shard
    (HybridDecoder.autotune -> {schedule: ms}), but a multi-rank step must run the same
    schedule everywhere — the timed loops hold matching collectives, and the slowest rank
    sets the step time. Returns (name, {schedule: max ms over ranks}): the schedule fastest
    by its max over ranks (a schedule a rank could not time counts as infinitely slow)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(times.get(n, float("inf"))) for n in SCHEDULES],
                     dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    best = int(torch.argmin(t).item())
    return SCHEDULES[best], {n: float(x) for n, x in zip(SCHEDULES, t.tolist())
                             if x != float("inf")}
