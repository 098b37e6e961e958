"""B200-native (sm_100a) HyLRA decode-time hybrid attention.

Drop-in for the layer-policy interface of the reference package `layerreuse`
(arxiv 2602.00777): FULL layers run a fused split-K flash-decode kernel that also emits
the per-KV-head selection scores, a top-k SELECT kernel turns those into index sets,
REUSE layers run a sparse-gather kernel over only the selected rows, and an OVERLAP
kernel feeds the host-side DP planner. All device work goes through libhylra.so (C ABI,
include/hylra.h); there is no CPU fallback.
"""
from .errors import (ConfigurationError, CudaError, InvalidInputError, InvalidSelectionError,
                     LayerReuseError, NumericInputError, SelectionPrecisionWarning)
from .policy import (BRUTE_FORCE_MAX_LAYERS, Action, LayerPolicy, brute_force_policy,
                     dp_optimize, policy_from_actions, static_jump_policy, validate_policy)
from .profiling import (LayerSensitivity, SensitivityReport, SimilarityMatrix, kl_extended,
                        merge_similarity_matrices, overlap_counts, relative_l2_error,
                        sensitivity_profile, similarity_from_counts)
from .results import (CostModelReport, DecodeRunResult, DecodeTrace, FidelityReport,
                      FidelityTable, cost_model, fidelity_report)
from .sets import BlockSet, TopKSet

__version__ = "0.1.0"

__all__ = [
    "Action", "LayerPolicy", "dp_optimize", "brute_force_policy", "BRUTE_FORCE_MAX_LAYERS",
    "SelectionPrecisionWarning", "policy_from_actions", "static_jump_policy",
    "validate_policy", "SimilarityMatrix", "merge_similarity_matrices", "overlap_counts",
    "relative_l2_error", "similarity_from_counts", "LayerReuseError", "ConfigurationError",
    "NumericInputError", "InvalidSelectionError", "InvalidInputError", "CudaError",
    "TopKSet", "BlockSet", "full_attention", "topk_select", "block_select", "sparse_attention",
    "HybridDecoder", "PipelinedDecoder", "LayerwiseDecoder", "DecodeLoop", "decode_step", "hybrid_decode",
    "hybrid_decode_blocks", "run_full_trace", "build_similarity_matrix", "kl_extended",
    "LayerSensitivity", "SensitivityReport", "sensitivity_profile", "CostModelReport",
    "cost_model", "FidelityReport", "fidelity_report", "FidelityTable", "DecodeRunResult",
    "DecodeTrace",
]


def __getattr__(name):
    # torch-dependent entry points load lazily so the host-only parts import without it
    if name in ("full_attention", "topk_select", "block_select", "sparse_attention",
                "geometry"):
        from . import attention
        return getattr(attention, name)
    if name in ("HybridDecoder", "decode_step", "hybrid_decode", "hybrid_decode_blocks",
                "run_full_trace", "PipelinedDecoder", "LayerwiseDecoder", "DecodeLoop",
                "build_similarity_matrix", "StepResult"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
