"""Seeded synthetic decode inputs with planted critical tokens (BASELINE.json configs 1-5).

The reference's own generator (pkg/src/layerreuse/synthetic.py:100-192, rho-blended rows)
is out of scope: the BASELINE configs specify a different distribution. Here Q, K, V are
N(0, 1); every layer has `planted` critical token positions, a fraction `keep` of which
is shared with the previous layer (75% for config 1, 90% = "10% drift" for configs 2-5),
and at those positions K is shifted by `shift * q_hat`, q_hat being the unit mean of the
group's queries, so those tokens dominate the selection score. Values are rounded to the
storage dtype before anyone (GPU or oracle) sees them, so both sides consume identical
numbers. Stand-in for the paper's model traces (LongBench v2 / PG-19 are not used).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

__all__ = ["StackConfig", "CONFIGS", "planted_positions", "generate_numpy", "generate_torch",
           "round_bf16"]


@dataclass(frozen=True)
class StackConfig:
    name: str
    layers: int
    batch: int
    q_heads: int
    kv_heads: int
    head_dim: int
    context: int
    budget: int
    dtype: str                 # "bf16" or "f32"
    full_layers: tuple         # FULL layers of the decode policy (the rest REUSE)
    planted: int
    keep: float
    shift: float = 2.0
    seed: int = 0

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads

    @property
    def actions(self) -> tuple:
        return tuple("full" if l in self.full_layers else "reuse" for l in range(self.layers))

    def with_(self, **kw) -> "StackConfig":
        return replace(self, **kw)


_LLAMA_FULL = (0, 1, 2, 8, 15, 16, 24, 31)
_QWEN_FULL = (0, 1, 2, 9, 15, 21, 27)

CONFIGS = {
    # config 1: CPU-reference-sized parity stack
    "cfg1": StackConfig("cfg1", 4, 1, 8, 2, 64, 2048, 128, "f32", (0, 2), 64, 0.75),
    # config 2: Llama-3-8B-shaped, 32K context (batch 1/4/8)
    "cfg2": StackConfig("cfg2", 32, 8, 32, 8, 128, 32768, 2048, "bf16", _LLAMA_FULL, 512, 0.9),
    # config 3: same stack at 128K context, batch 4, top-k 4096
    "cfg3": StackConfig("cfg3", 32, 4, 32, 8, 128, 131072, 4096, "bf16", _LLAMA_FULL, 512, 0.9),
    # config 4: Qwen2.5-7B-shaped, 64K context, batch 16
    "cfg4": StackConfig("cfg4", 28, 16, 28, 4, 128, 65536, 2048, "bf16", _QWEN_FULL, 512, 0.9),
    # config 5: offline profiling pass (all-FULL) on the Llama shape at 32K, batch 1
    "cfg5": StackConfig("cfg5", 32, 1, 32, 8, 128, 32768, 2048, "bf16", tuple(range(32)), 512, 0.9),
}


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bfloat16 (ties to even), returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def planted_positions(cfg: StackConfig) -> list:
    """Per-layer planted token positions (sorted int64), deterministic in cfg.seed."""
    rng = np.random.default_rng([cfg.seed, 0x91A7])
    n, p = cfg.context, min(cfg.planted, cfg.context)
    out = []
    cur = np.sort(rng.choice(n, size=p, replace=False))
    out.append(cur)
    n_keep = int(round(cfg.keep * p))
    for _ in range(1, cfg.layers):
        kept = rng.choice(cur, size=n_keep, replace=False)
        pool = np.setdiff1d(np.arange(n), kept, assume_unique=False)
        fresh = rng.choice(pool, size=p - n_keep, replace=False)
        cur = np.sort(np.concatenate([kept, fresh]))
        out.append(cur)
    return out


def _qhat(q: np.ndarray, G: int) -> np.ndarray:
    """Unit mean of each KV group's queries: q [..., Hq, d] -> [..., Hkv, d]."""
    sh = q.shape
    m = q.reshape(*sh[:-2], sh[-2] // G, G, sh[-1]).mean(axis=-2)
    return m / np.linalg.norm(m, axis=-1, keepdims=True)


def generate_numpy(cfg: StackConfig, capacity: int | None = None):
    """(q [L,B,Hq,d], k [L,B,Hkv,cap,d], v) float32 arrays holding dtype-rounded values.

    Rows [context, capacity) are zero. CPU-sized configs only (parity / oracle tests)."""
    cap = capacity or cfg.context
    rng = np.random.default_rng([cfg.seed, 0x5EED])
    L, B, Hq, Hkv, d, N = cfg.layers, cfg.batch, cfg.q_heads, cfg.kv_heads, cfg.head_dim, cfg.context
    rnd = round_bf16 if cfg.dtype == "bf16" else (lambda a: a.astype(np.float32))
    q = rnd(rng.standard_normal((L, B, Hq, d), dtype=np.float32))
    k = np.zeros((L, B, Hkv, cap, d), dtype=np.float32)
    v = np.zeros((L, B, Hkv, cap, d), dtype=np.float32)
    k[:, :, :, :N] = rng.standard_normal((L, B, Hkv, N, d), dtype=np.float32)
    v[:, :, :, :N] = rng.standard_normal((L, B, Hkv, N, d), dtype=np.float32)
    qh = _qhat(q.astype(np.float64), cfg.group).astype(np.float32)  # [L,B,Hkv,d]
    for l, pos in enumerate(planted_positions(cfg)):
        kl = k[l]  # view [B, Hkv, cap, d]
        kl[:, :, pos, :] += cfg.shift * qh[l][:, :, None, :]
    k = rnd(k)
    v = rnd(v)
    return q, k, v


def generate_torch(cfg: StackConfig, device="cuda", capacity: int | None = None):
    """Device tensors (q [L,B,Hq,d], k/v [L,B,Hkv,cap,d]) in the config's dtype, drawn
    with torch's Philox generator layer by layer (the full-size configs: 8.6-64 GB)."""
    import torch

    cap = capacity or cfg.context
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    L, B, Hq, Hkv, d, N = cfg.layers, cfg.batch, cfg.q_heads, cfg.kv_heads, cfg.head_dim, cfg.context
    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed * 1000003 + 17)
    q = torch.randn((L, B, Hq, d), generator=g, device=device, dtype=torch.float32).to(dt)
    k = torch.zeros((L, B, Hkv, cap, d), device=device, dtype=dt)
    v = torch.zeros((L, B, Hkv, cap, d), device=device, dtype=dt)
    G = cfg.group
    qm = q.float().view(L, B, Hkv, G, d).mean(dim=3)
    qhat = qm / qm.norm(dim=-1, keepdim=True)
    for l, pos in enumerate(planted_positions(cfg)):
        kl = torch.randn((B, Hkv, N, d), generator=g, device=device, dtype=torch.float32)
        pi = torch.as_tensor(pos, device=device)
        kl[:, :, pi, :] += cfg.shift * qhat[l][:, :, None, :]
        k[l, :, :, :N].copy_(kl)
        del kl
        v[l, :, :, :N].copy_(torch.randn((B, Hkv, N, d), generator=g, device=device,
                                         dtype=torch.float32))
    return q, k, v
