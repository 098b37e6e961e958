"""Hybrid FULL/REUSE decoding (HyLRA Algorithm 2) on B200 through the C ABI.

Reference: pkg/src/layerreuse/engine.py:129-209 `hybrid_decode` and
synthetic.py:237-301 `run_full_trace`. Three entry points:

* `HybridDecoder` — tensor-native, stateful: fixed cache geometry + policy, one
  `hylra_decode_step` per decode step (3 kernels: all FULL layers, all selections, all
  REUSE layers), CUDA-graph capturable, buffers reused across steps.
* `decode_step(...)` — functional one-shot form of the same.
* `hybrid_decode(model, policy, budget, steps)` / `run_full_trace(model, steps, budget)` —
  drop-ins taking the reference's duck-typed model (config.{layers, heads, head_dim,
  context_len}, grown_arrays, queries) and returning reference-shaped results (float64
  outputs [T, L, H, d], per-step per-layer TopKSet tuples in which a REUSE layer's entry
  IS its source's object, fidelity table against an all-FULL baseline, counters).

Policy semantics follow the engine, not `policy.sources`: a REUSE layer uses the most
recent FULL layer's selection of the same step (engine.py:173,176,185-194).
"""
from __future__ import annotations

import ctypes
import time

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .attention import block_select, full_attention, geometry, topk_select
from .errors import ConfigurationError, InvalidInputError, InvalidSelectionError, NumericInputError
from .policy import Action, LayerPolicy, policy_from_actions
from .profiling import overlap_counts, similarity_from_counts
from .results import (CostModelReport, DecodeRunResult, DecodeTrace, FidelityReport,
                      FidelityTable, cost_model, fidelity_report, fidelity_tables)
from .sets import BlockSet, TopKSet

__all__ = ["HybridDecoder", "OffloadDecoder", "PipelinedDecoder", "DecodeLoop", "StepResult", "decode_step",
           "DecodeRunResult", "FidelityTable", "DecodeTrace", "hybrid_decode",
           "hybrid_decode_blocks", "run_full_trace", "trace_overlap_counts",
           "build_similarity_matrix", "CostModelReport", "cost_model", "FidelityReport",
           "fidelity_report"]


def _actions_of(policy) -> tuple:
    if isinstance(policy, LayerPolicy):
        return policy.actions
    return policy_from_actions(policy).actions


@dataclass
class StepResult:
    """outputs: fp32 [L, B, Hq, d]; selections: int32 [n_full, B, groups, k_eff];
    slot_of_layer[l] = selection slot layer l used (its own for FULL, its source's for
    REUSE)."""

    outputs: torch.Tensor
    selections: torch.Tensor
    slot_of_layer: tuple
    full_layers: tuple

    def selection(self, layer: int) -> torch.Tensor:
        return self.selections[self.slot_of_layer[layer]]


class HybridDecoder:
    """Stateful hybrid decode driver for one cache geometry and one policy.

    k_cache / v_cache: [L, B, Hkv, capacity, d] (bf16 or fp32) resident in HBM; queries
    come per step as [L, B, Hq, d] in the same dtype. `step(q, n_valid)` enqueues one
    decode step on the current stream and returns views of the decoder's own output
    buffers (overwritten by the next step).
    """

    def __init__(self, policy, k_cache: torch.Tensor, v_cache: torch.Tensor, budget: int, *,
                 q_heads: int, sel_group: int = 1, refine: bool = True, block_size: int = 1,
                 include_sinks: int = 0, include_recent: int = 0, dual_stream: bool = False,
                 fuse_select: bool = True, single_launch="auto"):
        self.actions = _actions_of(policy)
        if len(self.actions) != k_cache.shape[0]:
            raise ConfigurationError(
                f"policy covers {len(self.actions)} layers, cache has {k_cache.shape[0]}")
        if self.actions[0] is not Action.FULL:
            raise InvalidInputError("the first layer of a policy must run full attention")
        if budget < 1:
            raise InvalidInputError(f"budget must be >= 1, got {budget}")
        self.k, self.v = k_cache, v_cache
        L, B, Hkv, cap, d = k_cache.shape
        self.budget, self.sel_group, self.refine = int(budget), int(sel_group), bool(refine)
        if sel_group < 1 or Hkv % sel_group:
            raise ConfigurationError(f"sel_group {sel_group} does not divide kv_heads {Hkv}")
        self.full_layers = tuple(l for l, a in enumerate(self.actions) if a is Action.FULL)
        slots, cur = [], -1
        for a in self.actions:
            if a is Action.FULL:
                cur += 1
            slots.append(cur)
        self.slot_of_layer = tuple(slots)
        self.q_heads = q_heads
        self.out = torch.empty((L, B, q_heads, d), dtype=torch.float32, device=k_cache.device)
        if block_size < 1:
            raise InvalidInputError(f"block_size must be >= 1, got {block_size}")
        if include_sinks < 0 or include_recent < 0:
            raise InvalidInputError("include_sinks and include_recent must be >= 0")
        if block_size > 1 and (include_sinks or include_recent):
            raise ConfigurationError("sink/recent augmentation applies to token selection only")
        self.block_size = int(block_size)
        self.sinks, self.recent = int(include_sinks), int(include_recent)
        # token mode: k indices per row; block mode: budget counts blocks
        self.k_stride = (min(self.budget, -(-cap // block_size)) if block_size > 1
                         else min(self.budget, cap))
        self.idx = torch.zeros((len(self.full_layers), B, Hkv // sel_group, self.k_stride),
                               dtype=torch.int32, device=k_cache.device)
        self._acts = _abi.uint8_array(1 if a is Action.FULL else 0 for a in self.actions)
        self.ws = torch.zeros(256, dtype=torch.uint8, device=k_cache.device)
        has_reuse = len(self.full_layers) < L
        # dual stream (token mode): the FULL layers that feed REUSE layers are scored first,
        # then the other FULL layers, then the REUSE launch, on the caller's stream; the
        # selects run on a high-priority side stream under the next streaming launch
        # (hylra_decode_step_ex)
        feeds = [l for l in self.full_layers if l + 1 < L and self.actions[l + 1] is Action.REUSE]
        self._dual_ok = (block_size == 1 and not (include_sinks or include_recent)
                         and 0 < len(feeds) < len(self.full_layers))
        self.dual = bool(dual_stream) and self._dual_ok
        # fused selects (token mode): the FULL kernel selects the rows of the FULL layers that
        # feed REUSE layers itself; the other FULL layers' SELECT runs on the side stream
        # under the REUSE launch (hylra_decode_step_ex fuse_select; tensor-core path only)
        self.fused = (bool(fuse_select) and block_size == 1 and not (include_sinks or include_recent)
                      and len(feeds) > 0 and sel_group == 1 and k_cache.dtype == torch.bfloat16
                      and d in (64, 128))
        if self.fused:
            self.dual = False
        # single-launch step (hylra_decode_step_ex fuse_select=2): FULL items with every
        # select fused, then the REUSE items, in one grid; REUSE items wait on per-row ready
        # flags. Same eligibility as the fused selects, any policy.
        # "auto": where it measured faster on B200 (scripts/ab_schedules.py,
        # profiles/r01_schedule_matrix.txt): enough FULL (layer, b, kv-head) pairs that the
        # fused selects of the last FULL pairs overlap REUSE items instead of delaying them
        # (cfg2 B>=4, cfg3 B=4, cfg4 B>=8; not B=1, cfg2 B=2, cfg4 B=4)
        # Block mode: always (its fused block selects are short; cfg2 B=1 229 vs 232 us,
        # B=8 1.44 vs 1.52 ms, scripts/block_single_ab.py).
        auto_rule = single_launch == "auto"
        if single_launch == "auto":
            # round 2 (scripts/dual_ab.py, profiles/r02_schedules_dual.txt): the single
            # launch from 192 FULL pairs, and from 128 at rows under 64K tokens (cfg2 B=2:
            # 396 vs 397 / 411 / 414 us); below that, long rows keep the fused selects (cfg3
            # B=1: fusedsel 730 vs 763 us) and short rows the two-stream step (below)
            pairs = len(self.full_layers) * B * Hkv
            single_launch = (bool(fuse_select) and not dual_stream and len(feeds) > 0
                             and (pairs >= 192 or block_size > 1
                                  or (pairs >= 128 and cap < 65536)))
        # token or block mode (hylra_decode_step_blocks_ex: the FULL pairs' final CTAs pool,
        # select blocks and write the coverage)
        self._single_ok = (not (block_size > 1 and (include_sinks or include_recent
                                                     or sel_group > 1))
                           and k_cache.dtype == torch.bfloat16 and d in (64, 128))
        self.single = bool(single_launch) and self._single_ok
        self.coop = False  # single-launch step with cooperative selects ("singlecoop")
        if self.single:
            self.dual = self.fused = False
        elif auto_rule and self.fused and cap < 65536:
            # short rows, few pairs: the two-stream step, whose selects run compact on a side
            # stream under the next streaming launch (cfg2 B=1: dual 218 vs fused3 224 vs
            # fusedsel 222 us, scripts/dual_ab.py), else the 3-launch step
            self.fused = False
            self.dual = self._dual_ok
        self._feeds_all = len(feeds) == len(self.full_layers)
        self._has_reuse = has_reuse
        # schedules this decoder can switch between (autotune): the fused-select and
        # single-launch variants need the tensor-core path, token mode, sel_group 1
        self._fused_ok = (block_size == 1 and not (include_sinks or include_recent)
                          and len(feeds) > 0 and sel_group == 1
                          and k_cache.dtype == torch.bfloat16 and d in (64, 128))
        self._count_kernels()
        if self.dual or self._fused_ok or self._dual_ok:
            # high priority: select CTAs are dispatched ahead of the queued FULL / REUSE CTAs
            self._side = torch.cuda.Stream(device=k_cache.device, priority=-8)
            self._events = [torch.cuda.Event() for _ in range(4)]
            for e in self._events:  # torch creates events lazily
                e.record(torch.cuda.current_stream(k_cache.device))

    def _count_kernels(self):
        aug = self._has_reuse and bool(self.sinks or self.recent)
        self.kernels_per_step = ((2 + self._has_reuse + aug) if self.block_size == 1
                                 else (3 + 2 * self._has_reuse)) + 2 * self.dual \
            - (self.fused and self._feeds_all)
        if self.single:
            self.kernels_per_step = 1

    @property
    def schedule(self) -> str:
        return (("singlecoop" if self.coop else "single") if self.single else
                "fusedsel" if self.fused else "dual" if self.dual else "fused3")

    def set_schedule(self, name: str) -> None:
        """Switch between the step schedules ("single", "singlecoop", "fusedsel", "dual",
        "fused3"; block mode: "single", "fused3"); every one gives bit-identical outputs and
        selections, only the launch structure differs. "singlecoop": the single-launch step
        whose FULL splits select cooperatively (hylra_step_options fuse_select = 3; token
        mode, sel_group 1). "dual": FULL(A) -> FULL(B) -> REUSE with the selects on a
        high-priority side stream under the next streaming launch (token mode, some but not
        all FULL layers feeding REUSE layers)."""
        if name not in ("single", "singlecoop", "fusedsel", "dual", "fused3"):
            raise ConfigurationError(f"unknown schedule {name!r}")
        if name == "dual" and not self._dual_ok:
            raise ConfigurationError("schedule 'dual' needs token mode without sinks / recent "
                                     "and some, but not all, FULL layers feeding REUSE layers")
        if name == "singlecoop" and not (self._single_ok and self._fused_ok):
            raise ConfigurationError("schedule 'singlecoop' needs token mode, sel_group 1 and "
                                     "the tensor-core path")
        if (name == "fusedsel" and not self._fused_ok) or (name == "single" and not self._single_ok):
            raise ConfigurationError(f"schedule {name!r} needs the tensor-core path (bf16, "
                                     "head_dim 64/128) and sel_group 1"
                                     + (", token mode and no sinks / recent"
                                        if name == "fusedsel" else ""))
        self.single = name in ("single", "singlecoop")
        self.coop = name == "singlecoop"
        self.fused, self.dual = name == "fusedsel", name == "dual" 
        self._count_kernels()

    def autotune(self, q: torch.Tensor, n_valid: int | None = None, reps: int = 10) -> dict:
        """Time the schedules this decoder can run on these inputs (CUDA-graph replays, CUDA
        events on the current stream) and keep the fastest. Returns {schedule: ms}. The
        measured steps overwrite `out` / the selections (the next step rewrites them)."""
        names = ([n for n, ok in (("single", self._single_ok),
                                  ("singlecoop", self._single_ok and self._fused_ok),
                                  ("fusedsel", self._fused_ok),
                                  ("dual", self._dual_ok)) if ok] + ["fused3"])
        times = {}
        cur = torch.cuda.current_stream(self.k.device)
        for name in names:
            self.set_schedule(name)
            side = torch.cuda.Stream(device=self.k.device)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                for _ in range(2):
                    self.step(q, n_valid)
            cur.wait_stream(side)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                self.step(q, n_valid)
            gr.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                gr.replay()
            e1.record()
            e1.synchronize()
            times[name] = e0.elapsed_time(e1) / reps
            del gr
        self.set_schedule(min(times, key=times.get))
        return times

    def _geometry(self, q):
        return geometry(q, self.k, self.v, self.out)

    def workspace_bytes(self, q, n_valid: int) -> int:
        g = self._geometry(q)
        return int(_abi.lib().hylra_decode_step_workspace_bytes(
            g, self._acts, int(n_valid), self.budget, self.sel_group, self.sinks, self.recent))

    def step(self, q: torch.Tensor, n_valid: int | None = None, *, layer_events=None,
             reuse_wait=None, out: torch.Tensor | None = None, append=None,
             idx_out: torch.Tensor | None = None) -> StepResult:
        """Enqueue one decode step. layer_events (optional, L torch.cuda.Event or None):
        event l is recorded once out[l] is final, REUSE layers being launched in chunks
        that end at the evented layers; reuse_wait (optional event): the REUSE launches
        wait on it (hylra_decode_step_ex). Token mode only. out (optional): fp32
        [L, B, Hq, d] destination instead of the decoder's own buffer — device memory or
        pinned host memory, which the kernels then write across the link directly.
        append (optional): (k_rows, v_rows, pos) — this step's new K/V rows
        [L, B, Hkv, d] (device or pinned host, cache dtype), written at cache row pos
        (< n_valid) before they are read; the single-launch step writes them inside its one
        kernel (hylra_step_options append_*).
        idx_out (optional): int32 tensor shaped like the decoder's selections
        [n_full, B, groups, k_stride], device or pinned host memory, that receives a second
        copy of every selection as the selecting CTAs write it (hylra_step_options
        idx_mirror): the per-layer index sets reach the host with no copy after the step."""
        if idx_out is not None:
            if idx_out.shape != self.idx.shape or idx_out.dtype != torch.int32 \
                    or not idx_out.is_contiguous() or not (idx_out.is_cuda or idx_out.is_pinned()):
                raise ConfigurationError("idx_out must be a contiguous int32 tensor shaped like "
                                         "the selections, on the device or pinned on the host")
        if out is not None:
            if out.shape != self.out.shape or out.dtype != torch.float32 \
                    or not out.is_contiguous() or not (out.is_cuda or out.is_pinned()):
                raise ConfigurationError("out must be a contiguous fp32 [L, B, Hq, d] device "
                                         "or pinned host tensor")
            own = self.out
            self.out = out
            try:
                return self.step(q, n_valid, layer_events=layer_events, reuse_wait=reuse_wait,
                                 append=append, idx_out=idx_out)
            finally:
                self.out = own
        g = self._geometry(q)
        n_valid = g.capacity if n_valid is None else int(n_valid)
        lib = _abi.lib()
        st = torch.cuda.current_stream(self.k.device).cuda_stream
        if self.block_size == 1:
            if layer_events is not None and len(layer_events) != len(self.actions):
                raise ConfigurationError(
                    f"{len(layer_events)} layer events for {len(self.actions)} layers")
            need = int(lib.hylra_decode_step_workspace_bytes(
                g, self._acts, n_valid, self.budget, self.sel_group, self.sinks, self.recent))
            self._grow_ws(need)
            opt = _abi.StepOptions()
            if self.single:
                opt.fuse_select = 3 if self.coop else 2
            if self.dual or self.fused:
                opt.fuse_select = int(self.fused)
                opt.side_stream = self._side.cuda_stream
                (opt.fork_event, opt.select_event, opt.full_event,
                 opt.join_event) = (e.cuda_event for e in self._events)
            if reuse_wait is not None:
                opt.reuse_wait_event = reuse_wait.cuda_event
            self._append_option(opt, append)
            if idx_out is not None:
                opt.idx_mirror = idx_out.data_ptr()
            evs = None
            if layer_events is not None:
                evs = _abi.pointer_array(e.cuda_event if e is not None else None
                                         for e in layer_events)
                opt.layer_events = ctypes.cast(evs, ctypes.c_void_p)
            _abi.check(lib.hylra_decode_step_ex(
                g, q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(), n_valid, self._acts,
                self.budget, self.sel_group, int(self.refine), self.sinks, self.recent,
                self.out.data_ptr(), self.idx.data_ptr(), self.k_stride, self.ws.data_ptr(),
                self.ws.numel(), st, ctypes.byref(opt)))
            k_eff = min(self.budget, n_valid)
            return StepResult(self.out, self.idx[..., :k_eff], self.slot_of_layer,
                              self.full_layers)
        if layer_events is not None or reuse_wait is not None:
            raise ConfigurationError("per-layer events apply to token selection only")
        if self.block_size > 1:
            need = int(lib.hylra_decode_step_blocks_workspace_bytes(
                g, self._acts, n_valid, self.budget, self.block_size, self.sel_group))
            self._grow_ws(need)
            opt = _abi.StepOptions()
            opt.fuse_select = 2 if self.single else 0
            self._append_option(opt, append)
            if idx_out is not None:
                opt.idx_mirror = idx_out.data_ptr()
            _abi.check(lib.hylra_decode_step_blocks_ex(
                g, q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(), n_valid, self._acts,
                self.budget, self.block_size, self.sel_group, int(self.refine),
                self.out.data_ptr(), self.idx.data_ptr(), self.k_stride, self.ws.data_ptr(),
                self.ws.numel(), st, ctypes.byref(opt)))
            bb = min(self.budget, -(-n_valid // self.block_size))
            return StepResult(self.out, self.idx[..., :bb], self.slot_of_layer,
                              self.full_layers)

    def _grow_ws(self, need: int) -> None:
        """Grow the (zero-filled) workspace to `need` bytes, keeping the flag words."""
        if self.ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device=self.ws.device)
            ws[:8].copy_(self.ws[:8])
            self.ws = ws

    def _append_option(self, opt, append) -> None:
        """hylra_step_options append_* from step(append=(k_rows, v_rows, pos))."""
        if append is None:
            return
        k_rows, v_rows, pos = append
        L, B, Hkv, cap, d = self.k.shape
        for t in (k_rows, v_rows):
            if t.shape != (L, B, Hkv, d) or t.dtype != self.k.dtype or not t.is_contiguous() \
                    or not (t.is_cuda or t.is_pinned()):
                raise ConfigurationError("new rows must be contiguous [L, B, Hkv, d] device or "
                                         "pinned host tensors of the cache dtype")
        opt.append_k_rows, opt.append_v_rows = k_rows.data_ptr(), v_rows.data_ptr()
        opt.append_pos = int(pos)

    def append(self, k_rows: torch.Tensor, v_rows: torch.Tensor, pos: int, layers=None) -> None:
        """Write one step's new K/V rows [L, B, Hkv, d] (device or pinned host tensors, the
        cache dtype) at cache row `pos` of the given layers (default all), on the current
        stream (hylra_append_kv; host rows are read across the link in place)."""
        L, B, Hkv, cap, d = self.k.shape
        for t in (k_rows, v_rows):
            if t.shape != (L, B, Hkv, d) or t.dtype != self.k.dtype or not t.is_contiguous() \
                    or not (t.is_cuda or t.is_pinned()):
                raise ConfigurationError("new rows must be contiguous [L, B, Hkv, d] device or "
                                         "pinned host tensors of the cache dtype")
        ids = list(range(L)) if layers is None else list(layers)
        # the new rows are validated as they are written (a NaN / inf sets the cache flag,
        # raised by check_flags as NumericInputError, attention.py:43-44)
        _abi.check(_abi.lib().hylra_append_kv_checked(
            self._cache_geometry(), self.k.data_ptr(), self.v.data_ptr(), k_rows.data_ptr(),
            v_rows.data_ptr(), int(pos), len(ids), _abi.int32_array(ids), self.ws.data_ptr(),
            torch.cuda.current_stream(self.k.device).cuda_stream))

    def _cache_geometry(self):
        L, B, Hkv, cap, d = self.k.shape
        g = _abi.Geometry()
        g.batch, g.q_heads, g.kv_heads, g.head_dim = B, self.q_heads, Hkv, d
        g.capacity, g.num_layers = cap, L
        g.dtype = _abi.HYLRA_BF16 if self.k.dtype == torch.bfloat16 else _abi.HYLRA_F32
        g.kv_stride_layer, g.kv_stride_batch, g.kv_stride_head = self.k.stride()[:3]
        return g

    def validate_cache(self, n_valid: int | None = None) -> None:
        """Reject a cache holding NaN / inf in rows [0, n_valid) of any layer, as the
        reference does when it builds its float64 caches (attention.py:38-46,61-71):
        NumericInputError. One streaming pass over the cache (hylra_check_cache; ~5 ms for
        config 2 at B=8), synchronising; appended rows are checked as they are written."""
        L, B, Hkv, cap, d = self.k.shape
        n = cap if n_valid is None else int(n_valid)
        flags = torch.zeros(64, dtype=torch.int32, device=self.k.device)
        _abi.check(_abi.lib().hylra_check_cache(
            self._cache_geometry(), self.k.data_ptr(), self.v.data_ptr(), n, L, None,
            flags.data_ptr(), torch.cuda.current_stream(self.k.device).cuda_stream))
        _abi.raise_for_flags(flags[:2].tolist())

    def flags(self) -> int:
        """Device flag word (synchronises)."""
        return int(self.ws[:4].view(torch.int32).item())

    def refine_skipped_rows(self) -> int:
        """Selection rows, since the last clear_flags, whose k-th boundary followed fp32
        order because the float64 refinement window held too many scores (synchronises)."""
        return int(self.ws[4:8].view(torch.int32).item())

    def check_flags(self, strict: bool = False) -> None:
        """Raise the reference exception a kernel flagged (out-of-range index:
        InvalidSelectionError, non-finite input: NumericInputError). A selection whose
        float64 refinement was skipped warns (SelectionPrecisionWarning), or raises
        InvalidSelectionError with strict=True."""
        _abi.raise_for_flags(self.ws[:8].view(torch.int32).tolist(), strict)

    def clear_flags(self) -> None:
        self.ws[:8].zero_()


class OffloadDecoder(HybridDecoder):
    """Index-guided offload (the offload mirror of engine.py:314-368): the
    FULL layers' K/V stay in HBM, the REUSE layers' K/V live in page-locked host memory and
    each step the REUSE kernel reads only the selected rows of them across the link
    (hylra_decode_step_offload; same three kernels as HybridDecoder).

    k_full / v_full: [n_full, B, Hkv, cap, d] CUDA tensors (FULL layers in layer order);
    k_reuse / v_reuse: [n_reuse, B, Hkv, cap, d] pinned CPU tensors (REUSE layers in layer
    order) — or CUDA tensors. Use `split_cache` to build them from one [L, ...] cache.
    Token selection only (optionally with sinks / recent)."""

    def __init__(self, policy, k_full, v_full, k_reuse, v_reuse, budget: int, *, q_heads: int,
                 sel_group: int = 1, refine: bool = True, include_sinks: int = 0,
                 include_recent: int = 0):
        actions = _actions_of(policy)
        n_full = sum(a is Action.FULL for a in actions)
        n_reuse = len(actions) - n_full
        if k_full.shape[0] != n_full or (n_reuse and k_reuse.shape[0] != n_reuse):
            raise ConfigurationError(
                f"policy has {n_full} FULL / {n_reuse} REUSE layers, caches hold "
                f"{k_full.shape[0]} / {0 if k_reuse is None else k_reuse.shape[0]}")
        if n_reuse:
            for t in (k_reuse, v_reuse):
                if t.shape[1:] != k_full.shape[1:] or t.stride()[1:] != k_full.stride()[1:] \
                        or t.dtype != k_full.dtype:
                    raise ConfigurationError("offloaded and resident caches must share a layout")
                if not t.is_cuda and not t.is_pinned():
                    raise ConfigurationError("an offloaded cache must be in pinned host memory")
        # the base class sees an L-layer cache view only for shapes; kernels get the split
        full_view = k_full[:1].expand((len(actions),) + tuple(k_full.shape[1:]))
        super().__init__(actions, full_view, full_view, budget, q_heads=q_heads,
                         sel_group=sel_group, refine=refine, include_sinks=include_sinks,
                         include_recent=include_recent, dual_stream=False, fuse_select=False)
        self.k_full, self.v_full, self.k_reuse, self.v_reuse = k_full, v_full, k_reuse, v_reuse
        self.reuse_layers = tuple(l for l, a in enumerate(actions) if a is Action.REUSE)

    @staticmethod
    def split_cache(policy, k_cache, v_cache, device="cuda"):
        """[L, B, Hkv, cap, d] cache -> (k_full, v_full) on `device`, (k_reuse, v_reuse)
        pinned on the host."""
        actions = _actions_of(policy)
        fl = [l for l, a in enumerate(actions) if a is Action.FULL]
        rl = [l for l, a in enumerate(actions) if a is Action.REUSE]
        kf = k_cache[fl].to(device).contiguous()
        vf = v_cache[fl].to(device).contiguous()
        kr = k_cache[rl].cpu().contiguous().pin_memory() if rl else None
        vr = v_cache[rl].cpu().contiguous().pin_memory() if rl else None
        return kf, vf, kr, vr

    def _geometry(self, q):
        g = geometry(q, self.k, self.v, self.out)
        g.kv_stride_layer = self.k_full.stride(0) if self.k_full.shape[0] > 1 else \
            self.k_full.stride(1) * self.k_full.shape[1]
        return g

    def step(self, q: torch.Tensor, n_valid: int | None = None) -> StepResult:
        g = self._geometry(q)
        n_valid = g.capacity if n_valid is None else int(n_valid)
        lib = _abi.lib()
        st = torch.cuda.current_stream(self.k_full.device).cuda_stream
        need = int(lib.hylra_decode_step_workspace_bytes(
            g, self._acts, n_valid, self.budget, self.sel_group, self.sinks, self.recent))
        self._grow_ws(need)
        kr = self.k_reuse.data_ptr() if self.k_reuse is not None else None
        vr = self.v_reuse.data_ptr() if self.v_reuse is not None else None
        _abi.check(lib.hylra_decode_step_offload(
            g, q.data_ptr(), self.k_full.data_ptr(), self.v_full.data_ptr(), kr, vr, n_valid,
            self._acts, self.budget, self.sel_group, int(self.refine), self.sinks, self.recent,
            self.out.data_ptr(), self.idx.data_ptr(), self.k_stride, self.ws.data_ptr(),
            self.ws.numel(), st))
        k_eff = min(self.budget, n_valid)
        return StepResult(self.out, self.idx[..., :k_eff], self.slot_of_layer, self.full_layers)


class PipelinedDecoder(HybridDecoder):
    """Same step as HybridDecoder, scheduled as a two-stream DAG of per-layer launches.

    Every FULL layer is independent of every other once the queries are known, so the
    FULL kernels stream back to back on the main stream while, on a side stream, each
    FULL layer's SELECT and then the REUSE layers that inherit its selection run as soon
    as that layer's scores exist. The latency-bound SELECT and the REUSE gathers overlap
    the HBM-bound FULL stream; only the last FULL layer's selection is exposed. Captured
    into a CUDA graph the whole step is one replay.

    The layer-sequential order a real model's decode imposes (layer l+1's query depends on
    layer l's output) is LayerwiseDecoder.
    """

    def __init__(self, policy, k_cache, v_cache, budget, *, q_heads, sel_group=1,
                 refine=True, schedule="pipelined"):
        super().__init__(policy, k_cache, v_cache, budget, q_heads=q_heads,
                         sel_group=sel_group, refine=refine, dual_stream=False,
                         fuse_select=False)
        if schedule != "pipelined":
            raise ConfigurationError(f"unknown schedule {schedule!r} (the layer-sequential "
                                     "schedule is LayerwiseDecoder)")
        self.pipe_schedule = schedule
        L, B, Hkv, cap, d = k_cache.shape
        from .attention import scores_row_stride
        self.scores = torch.empty((len(self.full_layers), B, Hkv, scores_row_stride(cap)),
                                  dtype=torch.float32, device=k_cache.device)
        self.side = torch.cuda.Stream(device=k_cache.device)
        self._events = [torch.cuda.Event() for _ in range(len(self.full_layers) + 2)]
        # REUSE layers grouped by the FULL slot they inherit from
        self.reuse_groups = [[l for l in range(L) if self.actions[l] is Action.REUSE
                              and self.slot_of_layer[l] == s]
                             for s in range(len(self.full_layers))]
        self._ws = {}
        n_reuse_launch = (sum(1 for g in self.reuse_groups if g) if schedule == "pipelined"
                          else sum(len(g) for g in self.reuse_groups))
        self.kernels_per_step = len(self.full_layers) * 2 + n_reuse_launch

    @property
    def schedule(self) -> str:
        return self.pipe_schedule

    def _buf(self, key, nbytes):
        t = self._ws.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=self.k.device)
            self._ws[key] = t
        return t

    def step(self, q: torch.Tensor, n_valid: int | None = None) -> StepResult:
        lib = _abi.lib()
        g = self._geometry(q)
        n_valid = g.capacity if n_valid is None else int(n_valid)
        k_eff = min(self.budget, n_valid)
        B, Hkv = g.batch, g.kv_heads
        groups = Hkv // self.sel_group
        sc_slot = self.scores[0].numel()
        idx_slot = self.idx[0].numel()
        main = torch.cuda.current_stream(self.k.device)
        side = self.side if self.pipe_schedule == "pipelined" else main
        ws_f = self._buf("full", lib.hylra_attention_workspace_bytes(g, 1, n_valid))
        sizes = {len(x) if self.pipe_schedule == "pipelined" else 1 for x in self.reuse_groups if x}
        ws_r = self._buf("reuse", max([lib.hylra_attention_workspace_bytes(g, n, k_eff)
                                       for n in sizes] or [256]))
        flags = self.ws if self.ws.numel() >= 256 else self._buf("flags", 256)
        if self.ws.numel() < 256:
            self.ws = flags
        qp, kp, vp = q.data_ptr(), self.k.data_ptr(), self.v.data_ptr()
        outp = self.out.data_ptr()
        refine_q = qp if self.refine else None
        refine_k = kp if self.refine else None
        if side is not main:
            side.wait_stream(main)
        for s, f in enumerate(self.full_layers):
            ids = _abi.int32_array([f])
            _abi.check(lib.hylra_full_decode(
                g, qp, kp, vp, n_valid, 1, ids, outp, self.scores.data_ptr() + 4 * s * sc_slot,
                ws_f.data_ptr(), ws_f.numel(), main.cuda_stream))
            if side is not main:
                self._events[s].record(main)
                side.wait_event(self._events[s])
            _abi.check(lib.hylra_topk_select(
                g, self.scores.data_ptr() + 4 * s * sc_slot, 1, n_valid, self.budget,
                self.sel_group, refine_q, refine_k, ids, self.idx.data_ptr() + 4 * s * idx_slot,
                self.k_stride, None, flags.data_ptr(), flags.numel(), side.cuda_stream))
            rg = self.reuse_groups[s]
            # pipelined: one launch for the whole chain; sequential: one launch per layer
            launches = [rg] if (rg and self.pipe_schedule == "pipelined") else [[l] for l in rg]
            for grp in launches:
                _abi.check(lib.hylra_reuse_decode(
                    g, qp, kp, vp, n_valid, len(grp), _abi.int32_array(grp),
                    _abi.int32_array([0] * len(grp)), self.idx.data_ptr() + 4 * s * idx_slot, None,
                    self.k_stride, k_eff, self.sel_group, outp, ws_r.data_ptr(), ws_r.numel(),
                    side.cuda_stream))
        if side is not main:
            main.wait_stream(side)
        return StepResult(self.out, self.idx[..., :k_eff], self.slot_of_layer, self.full_layers)


class LayerwiseDecoder(HybridDecoder):
    """Layer-sequential decode: the reference's per-layer loop (engine.py:174-194) one layer
    at a time, for callers whose layer l+1 query depends on layer l's output (a model's
    decode). `layer(l, q)` enqueues layer l on the current stream (hylra_decode_layer):

    * FULL layer feeding REUSE layers: FULL attention + score emission, then its selection
      (the shared-memory-resident select for few rows), both on the stream — the next REUSE
      layer needs the indices;
    * FULL layer no REUSE layer reads: FULL attention on the stream, its selection on a
      high-priority side stream (joined by `finish()`): only the step's output waits for it;
    * REUSE layer: the gather over its source FULL layer's selection.

    Every launch uses programmatic dependent launch with early loads: the producer warps
    of layer l+1 start streaming K/V (REUSE: the indices and gathered rows) while layer l
    drains, and only the reads of q wait for it — except the first REUSE layer after a
    selection and the step's first layer (whose inputs the previous launch may have
    written). Consecutive layers alternate between two workspaces. Selections are
    bit-identical to HybridDecoder.step's; outputs agree within bf16 rounding (a one-layer
    launch partitions its rows into more split-K splits than the batched step's)."""

    def __init__(self, policy, k_cache, v_cache, budget, *, q_heads, sel_group=1,
                 refine=True, prefetch=True):
        super().__init__(policy, k_cache, v_cache, budget, q_heads=q_heads,
                         sel_group=sel_group, refine=refine, dual_stream=False,
                         fuse_select=False, single_launch=False)
        L, B, Hkv, cap, d = k_cache.shape
        from .attention import scores_row_stride
        self.prefetch = bool(prefetch)
        self.scores = torch.empty((len(self.full_layers), B, Hkv, scores_row_stride(cap)),
                                  dtype=torch.float32, device=k_cache.device)
        # does some REUSE layer inherit FULL slot s?
        self.feeds = [any(self.actions[l] is Action.REUSE and self.slot_of_layer[l] == s
                          for l in range(L)) for s in range(len(self.full_layers))]
        self.side = torch.cuda.Stream(device=k_cache.device, priority=-8)
        n_side = sum(1 for f in self.feeds if not f)
        self._ev = [(torch.cuda.Event(), torch.cuda.Event()) for _ in range(max(n_side, 1))]
        self._wsl = [torch.zeros(256, dtype=torch.uint8, device=k_cache.device)
                     for _ in range(2)]
        self._side_ws = torch.zeros(256, dtype=torch.uint8, device=k_cache.device)
        self._turn = 0       # workspace of the next launch
        self._prev = None    # what the previous launch on the stream wrote: "sel" / other
        self._pending = []   # side-stream selections to join
        self.kernels_per_step = L + len(self.full_layers)

    @property
    def schedule(self) -> str:
        return "sequential"

    def _ws_for(self, need: int) -> torch.Tensor:
        t = self._wsl[self._turn]
        if t.numel() < need:
            t2 = torch.zeros(need, dtype=torch.uint8, device=t.device)
            t2[:8].copy_(t[:8])
            self._wsl[self._turn] = t = t2
        self._turn ^= 1
        return t

    def layer(self, l: int, q: torch.Tensor, n_valid: int | None = None) -> torch.Tensor:
        """Enqueue layer l (q: the [L, B, Hq, d] query stack; layer l's rows are read) on
        the current stream; returns out[l] (final once the stream reaches it)."""
        lib = _abi.lib()
        g = self._geometry(q)
        n_valid = g.capacity if n_valid is None else int(n_valid)
        k_eff = min(self.budget, n_valid)
        main = torch.cuda.current_stream(self.k.device)
        st = main.cuda_stream
        s = self.slot_of_layer[l]
        first = l == 0
        if self.actions[l] is Action.FULL:
            ws = self._ws_for(int(lib.hylra_attention_workspace_bytes(g, 1, n_valid)))
            sc = self.scores[s]
            sel_here = self.feeds[s]
            _abi.check(lib.hylra_decode_layer(
                g, q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(), n_valid, l, 1, s,
                self.budget, self.sel_group, int(self.refine),
                int(self.prefetch and not first), self.out.data_ptr(), sc.data_ptr(),
                self.idx.data_ptr() if sel_here else None, self.k_stride, ws.data_ptr(),
                ws.numel(), st))
            if sel_here:
                self._prev = "sel"
            else:
                # the selection only feeds the step's output: off the critical path
                e_fork, e_join = self._ev[len(self._pending)]
                e_fork.record(main)
                self.side.wait_event(e_fork)
                # compact: the select shares the GPU with the next FULL layer's streaming
                _abi.check(lib.hylra_topk_select_ex(
                    g, sc.data_ptr(), 1, n_valid, self.budget, self.sel_group,
                    q.data_ptr() if self.refine else None,
                    self.k.data_ptr() if self.refine else None, _abi.int32_array([l]),
                    self.idx[s].data_ptr(), self.k_stride, None, self._side_ws.data_ptr(),
                    self._side_ws.numel(), self.side.cuda_stream, _abi.SELECT_COMPACT))
                e_join.record(self.side)
                self._pending.append(e_join)
                self._prev = "full"
        else:
            ws = self._ws_for(int(lib.hylra_attention_workspace_bytes(g, 1, k_eff)))
            early = self.prefetch and not first and self._prev != "sel"
            _abi.check(lib.hylra_decode_layer(
                g, q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(), n_valid, l, 0, s,
                self.budget, self.sel_group, int(self.refine), int(early),
                self.out.data_ptr(), None, self.idx.data_ptr(), self.k_stride, ws.data_ptr(),
                ws.numel(), st))
            self._prev = "reuse"
        return self.out[l]

    def finish(self) -> None:
        """Join the side-stream selections into the current stream (end of a step)."""
        main = torch.cuda.current_stream(self.k.device)
        for e in self._pending:
            main.wait_event(e)
        self._pending = []
        self._prev = None

    def step(self, q: torch.Tensor, n_valid: int | None = None) -> StepResult:
        g = self._geometry(q)
        n_valid = g.capacity if n_valid is None else int(n_valid)
        self._prev = None
        for l in range(len(self.actions)):
            self.layer(l, q, n_valid)
        self.finish()
        k_eff = min(self.budget, n_valid)
        return StepResult(self.out, self.idx[..., :k_eff], self.slot_of_layer, self.full_layers)

    def _flag_words(self):
        """[flag word OR-ed over the workspaces, refine-skipped rows summed] (synchronises)."""
        w = torch.stack([t[:8].view(torch.int32)[:2] for t in (*self._wsl, self._side_ws)])
        words = w.cpu().tolist()
        flag = 0
        for f, _ in words:
            flag |= f
        return [flag, sum(n for _, n in words)]

    def flags(self) -> int:
        return self._flag_words()[0]

    def refine_skipped_rows(self) -> int:
        return self._flag_words()[1]

    def check_flags(self, strict: bool = False) -> None:
        _abi.raise_for_flags(self._flag_words(), strict)

    def clear_flags(self) -> None:
        for t in (*self._wsl, self._side_ws):
            t[:8].zero_()


def _runs(layers):
    """Ascending layer ids -> [(first, last + 1)] runs of consecutive layers."""
    runs = []
    for l in layers:
        if runs and runs[-1][1] == l:
            runs[-1][1] = l + 1
        else:
            runs.append([l, l + 1])
    return [tuple(r) for r in runs]


class DecodeLoop:
    """One decode step with host I/O as a single CUDA-graph launch.

    Per step: the query [L, B, Hq, d] and the new token's key/value rows [L, B, Hkv, d]
    come from pinned host buffers (`q_host`, `k_host`, `v_host`), the K/V rows are
    appended at cache row `pos`, the hybrid step runs over `pos + 1` rows, the fp32
    outputs land in the pinned `out_host` and the per-layer top-k index sets in the pinned
    `sel_host` ([n_full, B, groups, k]; a REUSE layer's set is its source slot's,
    `slot_of_layer`). Fill the host buffers, call `run()`; it returns `out_host` after the
    step completed.

    zero_copy=True (HybridDecoder): no copy operations at all — hylra_append_kv
    reads the new rows from pinned host memory in place (the FULL layers' rows before the
    FULL kernel, the REUSE layers' on a side stream under it, waited on by the REUSE
    launch), the attention kernels read each (layer, KV head)'s queries across the link
    when their CTAs start and store the outputs straight into `out_host`. zero_copy=False: H2D copies, append, step,
    D2H copy, serialised (the reference point).
    """

    def __init__(self, decoder: HybridDecoder, pos: int, *, zero_copy: bool = True,
                 q_copy="auto"):
        k = decoder.k
        L, B, Hkv, cap, d = k.shape
        if not 0 <= pos < cap:
            raise InvalidInputError(f"pos {pos} outside the cache capacity {cap}")
        self.dec, self.pos = decoder, int(pos)
        dt = k.dtype
        Hq = decoder.q_heads
        self.q_host = torch.zeros((L, B, Hq, d), dtype=dt).pin_memory()
        self.k_host = torch.zeros((L, B, Hkv, d), dtype=dt).pin_memory()
        self.v_host = torch.zeros((L, B, Hkv, d), dtype=dt).pin_memory()
        self.out_host = torch.zeros((L, B, Hq, d), dtype=torch.float32).pin_memory()
        self.sel_host = torch.zeros(tuple(decoder.idx.shape), dtype=torch.int32).pin_memory()
        self.graph = None
        self.h2d_bytes = (self.q_host.numel() + 2 * self.k_host.numel()) * self.q_host.element_size()
        # outputs + the index sets (k_eff of each selection row's k_stride entries)
        n_sel = decoder.idx[..., 0].numel()
        k_eff = (min(decoder.budget, pos + 1) if decoder.block_size == 1
                 else min(decoder.budget, -(-(pos + 1) // decoder.block_size)))
        self.d2h_bytes = self.out_host.numel() * 4 + n_sel * k_eff * 4
        self.zero_copy = bool(zero_copy) and type(decoder) is HybridDecoder
        if not self.zero_copy:
            self.q_dev = torch.zeros((L, B, Hq, d), dtype=dt, device=k.device)
            self.kv_dev = torch.zeros((2, L, B, Hkv, d), dtype=dt, device=k.device)
        acts = decoder.actions
        self.full_layers = [l for l in range(L) if acts[l] is Action.FULL]
        self.reuse_layers = [l for l in range(L) if acts[l] is Action.REUSE]
        # zero_copy q_copy: the queries come over in one H2D copy on a side stream, under the
        # append, instead of being read across the link by every CTA as it starts (costly
        # when the whole step is one wave: +20 us at cfg2 B=1, +14 us at B=8 where the copy
        # itself takes longer). "auto": capture() times both and keeps the faster.
        if q_copy not in ("auto", True, False):
            raise ConfigurationError(f"q_copy must be 'auto', True or False, got {q_copy!r}")
        self.q_copy = q_copy if self.zero_copy else False
        if self.zero_copy:
            self.side = torch.cuda.Stream(device=k.device)
            self.q_dev = torch.zeros((L, B, Hq, d), dtype=dt, device=k.device)
            # the REUSE layers' new rows are appended on a side stream under the FULL kernel;
            # the REUSE launch waits on them (hylra_decode_step_ex reuse_wait_event)
            self.ev_rows = torch.cuda.Event()
            self.ev_rows.record()  # torch creates events lazily
            # the query copy on the side stream: the step waits for it (ev_q), the REUSE
            # rows' append behind it on the same side stream does not hold the step up
            self.ev_q = torch.cuda.Event()
            self.ev_q.record()

    def _body(self, q_copy: bool = False):
        dec, pos = self.dec, self.pos
        if self.zero_copy:
            main = torch.cuda.current_stream(dec.k.device)
            q = self.q_host
            if q_copy:
                self.side.wait_stream(main)
                with torch.cuda.stream(self.side):
                    self.q_dev.copy_(self.q_host, non_blocking=True)
                    self.ev_q.record(self.side)
                q = self.q_dev
            io = dict(out=self.out_host, idx_out=self.sel_host)
            if dec.single or dec.block_size > 1:
                # the step's append option: the single-launch kernel writes the new rows
                # itself (one launch); the block-mode multi-launch step appends them first
                if q_copy:
                    main.wait_event(self.ev_q)
                dec.step(q, pos + 1, append=(self.k_host, self.v_host, pos), **io)
                return
            if not self.reuse_layers:
                dec.append(self.k_host, self.v_host, pos)
                if q_copy:
                    main.wait_event(self.ev_q)
                dec.step(q, pos + 1, **io)
                return
            if not q_copy:
                self.side.wait_stream(main)
            with torch.cuda.stream(self.side):
                dec.append(self.k_host, self.v_host, pos, self.reuse_layers)
                self.ev_rows.record(self.side)
            dec.append(self.k_host, self.v_host, pos, self.full_layers)
            if q_copy:
                # every kernel of the step reads the queries: the step waits for their copy
                # (the REUSE rows' append queued behind it keeps overlapping the FULL launch)
                main.wait_event(self.ev_q)
            dec.step(q, pos + 1, reuse_wait=self.ev_rows, **io)
            main.wait_stream(self.side)
            return
        self.q_dev.copy_(self.q_host, non_blocking=True)
        self.kv_dev[0].copy_(self.k_host, non_blocking=True)
        self.kv_dev[1].copy_(self.v_host, non_blocking=True)
        dec.append(self.kv_dev[0], self.kv_dev[1], pos)
        dec.step(self.q_dev, pos + 1)
        self.out_host.copy_(dec.out, non_blocking=True)
        self.sel_host.copy_(dec.idx, non_blocking=True)

    def _graph(self, q_copy: bool):
        s = torch.cuda.Stream(device=self.dec.k.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self._body(q_copy)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._body(q_copy)
        return g

    def capture(self, reps: int = 10):
        """Warm up and capture the step (host copies included) into a CUDA graph; with
        q_copy="auto" both query paths are captured and timed, the faster is kept."""
        if self.q_copy != "auto":
            self.graph = self._graph(bool(self.q_copy))
            return self
        times = {}
        for qc in (False, True):
            g = self._graph(qc)
            g.replay()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                g.replay()
                torch.cuda.current_stream().synchronize()
            times[qc] = (time.perf_counter() - t0) / reps
            del g
        self.q_copy = min(times, key=times.get)
        self.graph = self._graph(self.q_copy)
        return self

    def run(self) -> torch.Tensor:
        if self.graph is None:
            self.capture()
        self.graph.replay()
        torch.cuda.current_stream().synchronize()
        return self.out_host


def decode_step(policy, k_cache, v_cache, q, budget: int, n_valid: int | None = None, *,
                sel_group: int = 1, refine: bool = True) -> StepResult:
    """One hybrid decode step (functional form of HybridDecoder.step)."""
    dec = HybridDecoder(policy, k_cache, v_cache, budget, q_heads=q.shape[2],
                        sel_group=sel_group, refine=refine)
    res = dec.step(q, n_valid)
    dec.check_flags()
    return res


# --------------------------------------------------------------------------- drop-ins
def _model_tensors(model, steps: int, device):
    """Reference model arrays -> fp32 device tensors in the ABI layout.

    keys/values [L, H, N+T, d] -> [L, 1, H, cap, d]; queries [T, L, H, d] -> [T, L, 1, H, d].
    """
    keys, values = model.grown_arrays(steps)
    queries = model.queries(steps)
    L, H, NT, d = keys.shape
    cap = (NT + 63) // 64 * 64
    k = torch.zeros((L, 1, H, cap, d), dtype=torch.float32, device=device)
    v = torch.zeros((L, 1, H, cap, d), dtype=torch.float32, device=device)
    k[:, 0, :, :NT] = torch.as_tensor(np.asarray(keys, dtype=np.float32), device=device)
    v[:, 0, :, :NT] = torch.as_tensor(np.asarray(values, dtype=np.float32), device=device)
    q = torch.as_tensor(np.asarray(queries, dtype=np.float32), device=device).unsqueeze(2)
    return q.contiguous(), k, v


def _check_model_args(model, actions, steps: int, budget: int) -> None:
    cfg = model.config
    if len(actions) != cfg.layers:
        raise ConfigurationError(f"policy covers {len(actions)} layers, model has {cfg.layers}")
    if actions[0] is not Action.FULL:
        raise InvalidInputError("the first layer of a policy must run full attention")
    if steps < 1:
        raise InvalidInputError(f"steps must be >= 1, got {steps}")
    if budget < 1:
        raise InvalidInputError(f"budget must be >= 1, got {budget}")


def _run(model, actions, budget: int, steps: int, device, refine: bool, sinks: int = 0,
         recent: int = 0):
    cfg = model.config
    q, k, v = _model_tensors(model, steps, device)
    H = cfg.heads
    dec = HybridDecoder(actions, k, v, budget, q_heads=H, sel_group=H, refine=refine,
                        include_sinks=sinks, include_recent=recent)
    dec.validate_cache()  # attention.py:38-46: non-finite K/V -> NumericInputError
    outs, sels = [], []
    for t in range(steps):
        n_t = cfg.context_len + t
        res = dec.step(q[t], n_t)
        dec.check_flags()
        outs.append(res.outputs[:, 0].double().cpu().numpy())
        sels.append(res.selections[:, 0, 0].cpu().numpy())
    return np.stack(outs), sels, dec


def hybrid_decode(model, policy, budget: int, steps: int, *, include_sinks: int = 0,
                  include_recent: int = 0, device="cuda", refine: bool = True) -> DecodeRunResult:
    """Drop-in for the reference `hybrid_decode` (engine.py:129-209) on the GPU.

    The model's heads are MHA heads sharing one layer-wide selection (sel_group = H), the
    reference's aggregation rule. Compute runs in fp32 on the device; the selection
    boundary is re-resolved in float64 (refine=True)."""
    actions = _actions_of(policy)
    pol = policy if isinstance(policy, LayerPolicy) else policy_from_actions(actions)
    _check_model_args(model, actions, steps, budget)
    if include_sinks < 0 or include_recent < 0:
        raise InvalidInputError("include_sinks and include_recent must be >= 0")
    cfg = model.config
    outputs, sel_arrays, _ = _run(model, actions, budget, steps, device, refine,
                                  include_sinks, include_recent)
    baseline = run_full_trace(model, steps, min(budget, cfg.context_len), device=device,
                              refine=refine)
    L = cfg.layers
    selections, full_counts, gathered = [], [], []
    for t in range(steps):
        n_t = cfg.context_len + t
        step_sel, step_g, cur = [], [], None
        for l, a in enumerate(actions):
            if a is Action.FULL:
                slot = sum(1 for x in actions[:l] if x is Action.FULL)
                cur = TopKSet(tuple(int(i) for i in sel_arrays[t][slot]), budget)
                step_g.append(None)
            else:
                if include_sinks or include_recent:  # engine.py:122-126,187-188
                    extra = set(range(min(include_sinks, n_t))) | \
                        set(range(max(n_t - include_recent, 0), n_t))
                    merged = tuple(sorted(set(cur.indices) | extra))
                    if merged != cur.indices or cur.budget != len(merged):
                        cur = TopKSet(merged, len(merged))
                step_g.append(cur.size)
            step_sel.append(cur)
        selections.append(tuple(step_sel))
        gathered.append(tuple(step_g))
        full_counts.append(pol.full_count)
    outputs.setflags(write=False)
    return DecodeRunResult(
        policy=pol, budget=budget, block_size=1, outputs=outputs,
        selections=tuple(selections),
        fidelity=fidelity_tables(baseline.outputs, outputs),
        full_score_computations=tuple(full_counts), reuse_full_scans=0,
        reuse_gathered_rows=tuple(gathered))


def hybrid_decode_blocks(model, policy, block_budget: int, block_size: int, steps: int, *,
                         device="cuda", refine: bool = True) -> DecodeRunResult:
    """Drop-in for the reference `hybrid_decode_blocks` (engine.py:212-286): FULL layers keep
    the top min(block_budget, n_blocks) blocks of block_size tokens (max-pooled summed
    logits), REUSE layers attend over the inherited blocks' token coverage."""
    actions = _actions_of(policy)
    pol = policy if isinstance(policy, LayerPolicy) else policy_from_actions(actions)
    _check_model_args(model, actions, steps, block_budget)
    if block_size < 1:
        raise InvalidInputError(f"block_size must be >= 1, got {block_size}")
    cfg = model.config
    q, k, v = _model_tensors(model, steps, device)
    H = cfg.heads
    dec = HybridDecoder(actions, k, v, block_budget, q_heads=H, sel_group=H, refine=refine,
                        block_size=block_size)
    dec.validate_cache()  # attention.py:38-46: non-finite K/V -> NumericInputError
    outs, sels = [], []
    for t in range(steps):
        res = dec.step(q[t], cfg.context_len + t)
        dec.check_flags()
        outs.append(res.outputs[:, 0].double().cpu().numpy())
        sels.append(res.selections[:, 0, 0].cpu().numpy())
    outputs = np.stack(outs)
    baseline_budget = min(max(block_budget * block_size, 1), cfg.context_len)
    baseline = run_full_trace(model, steps, baseline_budget, device=device, refine=refine)
    L = cfg.layers
    selections, full_counts, gathered = [], [], []
    for t in range(steps):
        n_t = cfg.context_len + t
        step_sel, step_g, cur = [], [], None
        for l, a in enumerate(actions):
            if a is Action.FULL:
                slot = sum(1 for x in actions[:l] if x is Action.FULL)
                cur = BlockSet(tuple(int(i) for i in sels[t][slot]), block_size)
                step_g.append(None)
            else:
                step_g.append(int(cur.token_coverage(n_t).shape[0]))
            step_sel.append(cur)
        selections.append(tuple(step_sel))
        gathered.append(tuple(step_g))
        full_counts.append(pol.full_count)
    outputs.setflags(write=False)
    return DecodeRunResult(
        policy=pol, budget=block_budget, block_size=block_size, outputs=outputs,
        selections=tuple(selections),
        fidelity=fidelity_tables(baseline.outputs, outputs),
        full_score_computations=tuple(full_counts), reuse_full_scans=0,
        reuse_gathered_rows=tuple(gathered))


def run_full_trace(model, steps: int, budget: int, block_size: int = 1, *, device="cuda",
                   refine: bool = True) -> DecodeTrace:
    """Drop-in for the reference `run_full_trace` (synthetic.py:237-301): every layer FULL;
    per (step, layer) one layer-wide TopKSet of `budget` tokens and one BlockSet of the top
    min(ceil(budget / block_size), n_blocks) blocks, both from the same FULL-kernel scores
    (summed over all heads). The int32 token sets stay on the device for the OVERLAP kernel
    (idx_device [T, L, 1, budget])."""
    cfg = model.config
    if steps < 1:
        raise InvalidInputError(f"steps must be >= 1, got {steps}")
    if budget < 1 or budget > cfg.context_len:
        raise InvalidInputError(
            f"budget must lie in [1, context_len={cfg.context_len}], got {budget}")
    if block_size < 1:
        raise InvalidInputError(f"block_size must be >= 1, got {block_size}")
    q, k, v = _model_tensors(model, steps, device)
    H, L = cfg.heads, cfg.layers
    block_budget = -(-budget // block_size)
    outs, topk, blocks = [], [], []
    idx_dev = torch.empty((steps, L, 1, budget), dtype=torch.int32, device=device)
    rq, rk = (q, k) if refine else (None, None)
    for t in range(steps):
        n_t = cfg.context_len + t
        out, sc = full_attention(q[t], k, v, n_t)
        idx = topk_select(sc, budget, n_t, sel_group=H, q=rq[t] if refine else None, k=rk)
        blk, _, _ = block_select(sc, block_budget, block_size, n_t, sel_group=H,
                                 q=rq[t] if refine else None, k=rk)
        idx_dev[t].copy_(idx[:, 0])
        outs.append(out[:, 0].double().cpu().numpy())
        sel, bsel = idx[:, 0, 0].cpu().numpy(), blk[:, 0, 0].cpu().numpy()
        topk.append(tuple(TopKSet(tuple(int(i) for i in sel[l]), budget) for l in range(L)))
        blocks.append(tuple(BlockSet(tuple(int(i) for i in bsel[l]), block_size)
                            for l in range(L)))
    outputs = np.stack(outs)
    outputs.setflags(write=False)
    queries = np.asarray(model.queries(steps))
    return DecodeTrace(cfg, budget, block_size, queries, outputs, tuple(topk), tuple(blocks),
                       idx_dev)


def trace_overlap_counts(trace: DecodeTrace) -> np.ndarray:
    """OVERLAP kernel over a GPU trace: int counts [T, L, L] (counts[t, j, i] = |S_i & S_j|)."""
    c = overlap_counts(trace.idx_device, trace.config.context_len + trace.steps, trace.budget)
    return c[:, 0].cpu().numpy()


def build_similarity_matrix(trace: DecodeTrace):
    """Drop-in for profiling.py:126-145: GPU counts + the reference's float64 fold."""
    return similarity_from_counts(trace_overlap_counts(trace), trace.budget)
