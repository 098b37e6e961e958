"""Device-tensor attention primitives over the C ABI (no CPU fallback).

Reference counterparts (pkg/src/layerreuse/attention.py):
  full_attention  (:210-226)  -> `full_attention`   (hylra_full_decode)
  topk_of_logits  (:264-275)  -> `topk_select`      (hylra_topk_select)
  sparse_attention(:244-261)  -> `sparse_attention` (hylra_reuse_decode)
  TopKSet         (:108-140)  -> `TopKSet` (same canonical-form checks)

Layout (see include/hylra.h): q [L, B, Hq, d]; k, v [L, B, Hkv, capacity, d] with
d-contiguous rows (any outer strides); outputs fp32 [L, B, Hq, d]. A single layer may be
passed without the leading L axis. All work is enqueued on the current CUDA stream.
"""
from __future__ import annotations

import torch

from . import _abi
from .errors import ConfigurationError, InvalidInputError, InvalidSelectionError
from .sets import BlockSet, TopKSet

__all__ = ["TopKSet", "BlockSet", "geometry", "full_attention", "topk_select", "block_select",
           "sparse_attention", "scores_row_stride"]


_DTYPES = {torch.bfloat16: _abi.HYLRA_BF16, torch.float32: _abi.HYLRA_F32}


def scores_row_stride(capacity: int) -> int:
    return (capacity + 7) & ~7


def _as_stack(t: torch.Tensor, dims: int) -> torch.Tensor:
    return t.unsqueeze(0) if t.dim() == dims - 1 else t


def geometry(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
             out: torch.Tensor | None = None) -> _abi.Geometry:
    """Build the ABI geometry from [L,B,Hq,d] queries and [L,B,Hkv,cap,d] caches."""
    if q.dim() != 4 or k.dim() != 5 or v.dim() != 5:
        raise ConfigurationError("expected q [L,B,Hq,d] and k/v [L,B,Hkv,cap,d]")
    if k.shape != v.shape or k.stride() != v.stride():
        raise ConfigurationError(f"keys {tuple(k.shape)} and values {tuple(v.shape)} differ")
    L, B, Hq, d = q.shape
    Lk, Bk, Hkv, cap, dk = k.shape
    if (Lk, Bk, dk) != (L, B, d):
        raise ConfigurationError(
            f"query shape {tuple(q.shape)} does not match cache shape {tuple(k.shape)}")
    if q.dtype != k.dtype or k.dtype != v.dtype or q.dtype not in _DTYPES:
        raise ConfigurationError("q, k, v must share dtype bfloat16 or float32")
    if not (k.is_cuda and v.is_cuda and (q.is_cuda or q.is_pinned())):
        raise ConfigurationError("k / v must be CUDA tensors, q a CUDA or pinned host tensor")
    if q.stride(3) != 1 or q.stride(2) != d or k.stride(4) != 1 or k.stride(3) != d:
        raise ConfigurationError("rows must be d-contiguous (q heads and KV rows packed)")
    g = _abi.Geometry()
    g.batch, g.q_heads, g.kv_heads, g.head_dim = B, Hq, Hkv, d
    g.capacity, g.dtype, g.num_layers = cap, _DTYPES[q.dtype], L
    g.q_stride_layer, g.q_stride_batch = q.stride(0), q.stride(1)
    g.kv_stride_layer, g.kv_stride_batch, g.kv_stride_head = k.stride(0), k.stride(1), k.stride(2)
    if out is not None:
        if out.dtype != torch.float32 or out.shape != q.shape or out.stride(3) != 1 \
                or out.stride(2) != d:
            raise ConfigurationError("out must be fp32 with q's shape and packed heads")
        g.out_stride_layer, g.out_stride_batch = out.stride(0), out.stride(1)
    return g


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def full_attention(q, k, v, n_valid: int | None = None, *, scores: bool = True,
                   layers=None):
    """FULL attention of every query head over rows [0, n_valid) of its KV head.

    Returns (out fp32 [L,B,Hq,d], scores fp32 [L,B,Hkv,row_stride] or None) where
    scores[l,b,h,n] = sum over the group's heads of q.k_n / sqrt(d) (engine.py:177-181).
    """
    single = q.dim() == 3
    q, k, v = _as_stack(q, 4), _as_stack(k, 5), _as_stack(v, 5)
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    g = geometry(q, k, v, out)
    n_valid = g.capacity if n_valid is None else int(n_valid)
    layer_ids = list(range(g.num_layers)) if layers is None else list(layers)
    ns = len(layer_ids)
    sc = None
    if scores:
        sc = torch.empty((ns, g.batch, g.kv_heads, scores_row_stride(g.capacity)),
                         dtype=torch.float32, device=q.device)
    ws_b = _abi.lib().hylra_attention_workspace_bytes(g, ns, n_valid)
    ws = _workspace(ws_b, q.device)
    _abi.check(_abi.lib().hylra_full_decode(
        g, q.data_ptr(), k.data_ptr(), v.data_ptr(), n_valid, ns, _abi.int32_array(layer_ids),
        out.data_ptr(), sc.data_ptr() if sc is not None else None, ws.data_ptr(), ws.numel(),
        _stream(q)))
    if single:
        out = out[0]
        sc = sc[0] if sc is not None else None
    return out, sc


def topk_select(scores, budget: int, n_valid: int, *, sel_group: int = 1, q=None, k=None,
                layers=None, info: bool = False):
    """Exact top-min(budget, n_valid) per (slot, b, group) row, ties to the lower index,
    ascending int32 [S, B, Hkv/sel_group, k_eff]. With q/k given, the k-th boundary is
    re-resolved in float64 from the original values (see select.cuh)."""
    single = scores.dim() == 3
    scores = _as_stack(scores, 4)
    if scores.dtype != torch.float32 or not scores.is_cuda or not scores.is_contiguous():
        raise ConfigurationError("scores must be a contiguous fp32 CUDA tensor")
    if budget < 1:
        raise InvalidInputError(f"budget must be >= 1, got {budget}")
    S, B, Hkv, rs = scores.shape
    if q is not None and k is not None:
        q4, k5 = _as_stack(q, 4), _as_stack(k, 5)
        g = geometry(q4, k5, k5)
        qp, kp = q4.data_ptr(), k5.data_ptr()
        layer_ids = list(range(S)) if layers is None else list(layers)
    else:
        g = _abi.Geometry()
        g.batch, g.q_heads, g.kv_heads, g.head_dim = B, Hkv, Hkv, 128
        g.dtype, g.num_layers = _abi.HYLRA_F32, S
        g.capacity = rs
        qp = kp = None
        layer_ids = list(range(S))
    if scores_row_stride(g.capacity) != rs:
        raise ConfigurationError(f"scores row stride {rs} does not match capacity {g.capacity}")
    k_eff = min(budget, n_valid)
    groups = Hkv // sel_group if sel_group >= 1 else 0
    idx = torch.empty((S, B, max(groups, 1), k_eff), dtype=torch.int32, device=scores.device)
    inf = torch.zeros((S, B, max(groups, 1), 8), dtype=torch.int32, device=scores.device)
    ws = _workspace(256, scores.device)
    _abi.check(_abi.lib().hylra_topk_select(
        g, scores.data_ptr(), S, int(n_valid), int(budget), int(sel_group), qp, kp,
        _abi.int32_array(layer_ids), idx.data_ptr(), k_eff, inf.data_ptr(), ws.data_ptr(),
        ws.numel(), _stream(scores)))
    _raise_flags(ws)
    if single:
        idx, inf = idx[0], inf[0]
    return (idx, inf) if info else idx


def block_select(scores, block_budget: int, block_size: int, n_valid: int, *,
                 sel_group: int = 1, q=None, k=None, layers=None, info: bool = False):
    """Block-level top-k (attention.py:287-313): per row, max-pool the token scores into
    blocks, keep the top min(block_budget, n_blocks) blocks (ties -> lower block,
    ascending) and expand them to their token coverage.

    Returns (blocks int32 [S,B,groups,bb], tokens int32 [S,B,groups,bb*block_size] (-1 past
    the coverage), counts int32 [S,B,groups])."""
    single = scores.dim() == 3
    scores = _as_stack(scores, 4)
    if scores.dtype != torch.float32 or not scores.is_cuda or not scores.is_contiguous():
        raise ConfigurationError("scores must be a contiguous fp32 CUDA tensor")
    if block_budget < 1:
        raise InvalidInputError(f"block_budget must be >= 1, got {block_budget}")
    if block_size < 1:
        raise InvalidInputError(f"block_size must be >= 1, got {block_size}")
    S, B, Hkv, rs = scores.shape
    if q is not None and k is not None:
        q4, k5 = _as_stack(q, 4), _as_stack(k, 5)
        g = geometry(q4, k5, k5)
        qp, kp = q4.data_ptr(), k5.data_ptr()
        layer_ids = list(range(S)) if layers is None else list(layers)
    else:
        g = _abi.Geometry()
        g.batch, g.q_heads, g.kv_heads, g.head_dim = B, Hkv, Hkv, 128
        g.dtype, g.num_layers, g.capacity = _abi.HYLRA_F32, S, rs
        qp = kp = None
        layer_ids = list(range(S))
    nb = -(-n_valid // block_size)
    bb = min(block_budget, nb)
    groups = Hkv // sel_group
    blocks = torch.empty((S, B, groups, bb), dtype=torch.int32, device=scores.device)
    tokens = torch.empty((S, B, groups, bb * block_size), dtype=torch.int32, device=scores.device)
    counts = torch.empty((S, B, groups), dtype=torch.int32, device=scores.device)
    inf = torch.zeros((S, B, groups, 8), dtype=torch.int32, device=scores.device)
    ws = _workspace(256 + 4 * S * B * groups * ((nb + 7) & ~7), scores.device)
    _abi.check(_abi.lib().hylra_block_select(
        g, scores.data_ptr(), S, int(n_valid), int(block_budget), int(block_size), int(sel_group),
        qp, kp, _abi.int32_array(layer_ids), blocks.data_ptr(), bb, tokens.data_ptr(),
        bb * block_size, counts.data_ptr(), inf.data_ptr(), ws.data_ptr(), ws.numel(),
        _stream(scores)))
    _raise_flags(ws)
    if single:
        blocks, tokens, counts, inf = blocks[0], tokens[0], counts[0], inf[0]
    return (blocks, tokens, counts, inf) if info else (blocks, tokens, counts)


def sparse_attention(q, k, v, idx, n_valid: int | None = None, *, sel_group: int = 1,
                     check: bool = True):
    """Attention over the selected rows only, softmax renormalised over the subset.

    idx: int32 [B, Hkv/sel_group, k] (one layer) or [L, B, Hkv/sel_group, k]; every row
    must be canonical (ascending, distinct, < n_valid) as TopKSet requires."""
    single = q.dim() == 3
    q, k, v = _as_stack(q, 4), _as_stack(k, 5), _as_stack(v, 5)
    idx = _as_stack(idx, 4)
    if idx.dtype != torch.int32 or not idx.is_cuda:
        raise ConfigurationError("idx must be an int32 CUDA tensor")
    idx = idx.contiguous()
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    g = geometry(q, k, v, out)
    n_valid = g.capacity if n_valid is None else int(n_valid)
    L = g.num_layers
    if idx.shape[0] not in (1, L):
        raise ConfigurationError("idx must hold one selection set per layer (or one shared)")
    k_eff = idx.shape[-1]
    if k_eff < 1:
        raise InvalidSelectionError("selection must contain at least one index")
    if check:
        if bool((idx[..., 1:] <= idx[..., :-1]).any()):
            raise InvalidSelectionError("token indices must be strictly ascending")
        if int(idx.min()) < 0:
            raise InvalidSelectionError("token indices must be non-negative")
        if int(idx.max()) >= n_valid:
            raise InvalidSelectionError(
                f"selection index {int(idx.max())} is out of range for cache length {n_valid}")
    src = [i if idx.shape[0] == L else 0 for i in range(L)]
    ws_b = _abi.lib().hylra_attention_workspace_bytes(g, L, k_eff)
    ws = _workspace(ws_b, q.device)
    _abi.check(_abi.lib().hylra_reuse_decode(
        g, q.data_ptr(), k.data_ptr(), v.data_ptr(), n_valid, L, _abi.int32_array(range(L)),
        _abi.int32_array(src), idx.data_ptr(), None, k_eff, k_eff, int(sel_group), out.data_ptr(),
        ws.data_ptr(), ws.numel(), _stream(q)))
    _raise_flags(ws)
    return out[0] if single else out


def _raise_flags(ws: torch.Tensor, strict: bool = False) -> None:
    """Synchronising check of the device flag words (eager API only; graphs skip it)."""
    _abi.raise_for_flags(ws[:8].view(torch.int32).tolist(), strict)
