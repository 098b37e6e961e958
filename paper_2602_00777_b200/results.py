"""Host-side result types, fidelity measurement and the analytic cost model (no torch).

Reference: pkg/src/layerreuse/engine.py — `FidelityTable` (:47-57), `DecodeRunResult`
(:60-92), `_fidelity_tables` (:95-108), `CostModelReport` / `cost_model` (:289-368),
`FidelityReport` / `fidelity_report` (:371-424); `DecodeTrace` (synthetic.py:214-234).
The GPU drivers in engine.py fill these; formats.py reads and writes them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError
from .policy import LayerPolicy
from .profiling import relative_l2_error
from .sets import TopKSet

__all__ = [
    "FidelityTable", "DecodeRunResult", "DecodeTrace", "fidelity_tables", "CostModelReport",
    "cost_model", "FidelityReport", "fidelity_report",
]


@dataclass(frozen=True)
class FidelityTable:
    """Relative L2 error of hybrid outputs against the all-FULL baseline (engine.py:47-57):
    per_step_layer [T, L], per_layer (mean over steps), aggregate (mean of everything)."""

    per_step_layer: np.ndarray
    per_layer: np.ndarray
    aggregate: float


@dataclass(frozen=True)
class DecodeRunResult:
    """Outputs, selections, fidelity and counters of one hybrid run (engine.py:60-92).
    budget counts tokens in token mode and blocks in block mode."""

    policy: LayerPolicy
    budget: int
    block_size: int
    outputs: np.ndarray
    selections: tuple
    fidelity: FidelityTable
    full_score_computations: tuple
    reuse_full_scans: int
    reuse_gathered_rows: tuple

    @property
    def full_layer_count(self) -> int:
        return self.policy.full_count

    @property
    def reuse_layer_count(self) -> int:
        return self.policy.num_layers - self.policy.full_count

    @property
    def steps(self) -> int:
        return self.outputs.shape[0]


@dataclass(frozen=True)
class DecodeTrace:
    """All-FULL decode record (synthetic.py:214-234): queries/outputs [T, L, H, d],
    topk[t][l] (TopKSet of `budget` tokens) and blocks[t][l] (BlockSet of width block_size)
    per layer, both layer-wide over the summed head logits. idx_device keeps the int32
    token sets on the GPU ([T, L, 1, budget]) for the OVERLAP kernel, or is None."""

    config: object
    budget: int
    block_size: int
    queries: np.ndarray
    outputs: np.ndarray
    topk: tuple
    blocks: tuple = ()
    idx_device: object = None

    @property
    def steps(self) -> int:
        return self.queries.shape[0]


def fidelity_tables(baseline_outputs, hybrid_outputs) -> FidelityTable:
    """Per (step, layer) relative L2 error over the flattened [H, d] outputs (engine.py:95-108)."""
    base = np.asarray(baseline_outputs)
    hyb = np.asarray(hybrid_outputs)
    steps, layers = hyb.shape[0], hyb.shape[1]
    table = np.empty((steps, layers))
    for t in range(steps):
        for l in range(layers):
            table[t, l] = relative_l2_error(hyb[t, l].ravel(), base[t, l].ravel())
    table.setflags(write=False)
    per_layer = table.mean(axis=0)
    per_layer.setflags(write=False)
    return FidelityTable(per_step_layer=table, per_layer=per_layer,
                         aggregate=float(table.mean()))


# ----------------------------------------------------------------------------- cost model
@dataclass(frozen=True)
class CostModelReport:
    """Analytic KV traffic of one decode step under a policy (engine.py:289-311). Byte
    counts are exact integers; the HBM/link seconds scale them by the given bandwidths."""

    kv_bytes_full: int
    kv_bytes_hybrid: int
    bytes_ratio: float
    link_bytes_full: int
    link_bytes_offload: int
    predicted_speedup: float
    tokens_covered: int
    hbm_seconds_full: float
    hbm_seconds_hybrid: float
    link_seconds_full: float
    link_seconds_offload: float


def cost_model(policy: LayerPolicy, context_len: int, budget: int, *, block_size: int = 1,
               bytes_per_elem: int = 8, head_dim: int = 64, link_bandwidth: float = 32e9,
               hbm_bandwidth: float = 2e12) -> CostModelReport:
    """Price one step's KV reads (engine.py:314-368): a FULL layer reads context_len rows,
    a REUSE layer min(budget * block_size, context_len) rows, each 2 * head_dim *
    bytes_per_elem bytes (head_dim = the whole per-layer KV width). In the offload mirror
    the REUSE layers' caches sit across the link, so link bytes follow the same split.

    bench.py checks its algorithmic HBM bytes against kv_bytes_hybrid x batch."""
    if context_len < 1:
        raise InvalidInputError(f"context_len must be >= 1, got {context_len}")
    if budget < 1:
        raise InvalidInputError(f"budget must be >= 1, got {budget}")
    if block_size < 1:
        raise InvalidInputError(f"block_size must be >= 1, got {block_size}")
    if bytes_per_elem < 1:
        raise InvalidInputError(f"bytes_per_elem must be >= 1, got {bytes_per_elem}")
    if head_dim < 1:
        raise InvalidInputError(f"head_dim must be >= 1, got {head_dim}")
    if not link_bandwidth > 0 or not hbm_bandwidth > 0:
        raise InvalidInputError("bandwidths must be positive")
    n_layers, n_full = policy.num_layers, policy.full_count
    covered = min(budget * block_size, context_len)
    row = 2 * head_dim * bytes_per_elem
    full_bytes = n_layers * context_len * row
    hybrid_bytes = (n_full * context_len + (n_layers - n_full) * covered) * row
    return CostModelReport(
        kv_bytes_full=full_bytes, kv_bytes_hybrid=hybrid_bytes,
        bytes_ratio=hybrid_bytes / full_bytes,
        link_bytes_full=full_bytes, link_bytes_offload=hybrid_bytes,
        predicted_speedup=full_bytes / hybrid_bytes, tokens_covered=covered,
        hbm_seconds_full=full_bytes / hbm_bandwidth,
        hbm_seconds_hybrid=hybrid_bytes / hbm_bandwidth,
        link_seconds_full=full_bytes / link_bandwidth,
        link_seconds_offload=hybrid_bytes / link_bandwidth)


# ----------------------------------------------------------------------------- fidelity
@dataclass(frozen=True)
class FidelityReport:
    """Hybrid run vs an all-FULL trace (engine.py:371-385): output error tables plus the
    per (step, layer) selection agreement |shared| / max(sizes) and its per-layer mean."""

    rnmse: FidelityTable
    selection_overlap: np.ndarray
    per_layer_overlap: np.ndarray


def _members(sel) -> set:
    return set(sel.indices if isinstance(sel, TopKSet) else sel.block_indices)


def fidelity_report(baseline: DecodeTrace, hybrid: DecodeRunResult) -> FidelityReport:
    """engine.py:391-424: token-mode runs compare against the trace's token sets, block-mode
    runs against its block sets (block widths must match)."""
    if baseline.outputs.shape != hybrid.outputs.shape:
        raise InvalidInputError(
            f"shape mismatch: baseline {baseline.outputs.shape} vs hybrid {hybrid.outputs.shape}")
    if hybrid.block_size > 1 and baseline.block_size != hybrid.block_size:
        raise InvalidInputError(
            f"block size mismatch: baseline {baseline.block_size} vs hybrid {hybrid.block_size}")
    steps, layers = hybrid.outputs.shape[0], hybrid.outputs.shape[1]
    base_sets = baseline.topk if hybrid.block_size == 1 else baseline.blocks
    overlap = np.empty((steps, layers))
    for t in range(steps):
        for l in range(layers):
            a, b = _members(base_sets[t][l]), _members(hybrid.selections[t][l])
            overlap[t, l] = len(a & b) / max(len(a), len(b))
    overlap.setflags(write=False)
    per_layer = overlap.mean(axis=0)
    per_layer.setflags(write=False)
    return FidelityReport(rnmse=fidelity_tables(baseline.outputs, hybrid.outputs),
                          selection_overlap=overlap, per_layer_overlap=per_layer)

