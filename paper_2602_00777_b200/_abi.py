"""ctypes binding of libhylra.so — the C ABI declared in include/hylra.h.

The shared library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a). There
is no fallback: if the library is missing every op raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import STATUS_TO_ERROR, CudaError, LayerReuseError

# HYLRA_LIB: another build of the same ABI (A/B experiments between library versions)
LIB_PATH = Path(os.environ.get("HYLRA_LIB") or Path(__file__).resolve().parent / "libhylra.so")

# include/hylra.h HYLRA_ABI_VERSION this binding is written against (checked at load)
ABI_VERSION = 7
SELECT_COMPACT = 1  # hylra_topk_select_ex options (include/hylra.h)

HYLRA_BF16 = 0
HYLRA_F32 = 1

# status codes (include/hylra.h)
HYLRA_OK = 0
HYLRA_ERR_CONFIGURATION = 1
HYLRA_ERR_INVALID_INPUT = 2
HYLRA_ERR_INVALID_SELECTION = 3
HYLRA_ERR_NUMERIC_INPUT = 4
HYLRA_ERR_CUDA = 5

FLAG_INDEX_OUT_OF_RANGE = 1
FLAG_NON_FINITE_SCORE = 2
FLAG_REFINE_SKIPPED = 4
FLAG_INTERNAL = 8
FLAG_NON_FINITE_CACHE = 16


def raise_for_flags(words, strict: bool = False) -> None:
    """Map the workspace flag words (include/hylra.h: flag word, refine-skipped row count) to
    the reference's exceptions. HYLRA_FLAG_REFINE_SKIPPED means some selection row's k-th
    boundary could not be re-resolved in float64 (more than 1024 scores inside the
    refinement window): that row follows fp32 order with ties to the lower index, which can
    differ from the reference's float64 order (attention.py:264-275). It warns
    (SelectionPrecisionWarning), or raises InvalidSelectionError when `strict`."""
    flags, skipped = int(words[0]), int(words[1]) if len(words) > 1 else 0
    if flags & FLAG_INDEX_OUT_OF_RANGE:
        from .errors import InvalidSelectionError
        raise InvalidSelectionError("a selection index is out of range for the cache")
    if flags & FLAG_NON_FINITE_SCORE:
        from .errors import NumericInputError
        raise NumericInputError("selection scores contain non-finite entries")
    if flags & FLAG_NON_FINITE_CACHE:
        from .errors import NumericInputError
        raise NumericInputError("the KV cache contains non-finite entries")
    if flags & FLAG_INTERNAL:
        raise CudaError("a selection kernel invariant failed (internal error)")
    if flags & FLAG_REFINE_SKIPPED:
        msg = (f"{max(skipped, 1)} selection row(s) had more than 1024 scores within the "
               "float64 refinement window of the k-th value; their boundary follows fp32 "
               "order (ties to the lower index), not the reference's float64 order")
        if strict:
            from .errors import InvalidSelectionError
            raise InvalidSelectionError(msg)
        import warnings

        from .errors import SelectionPrecisionWarning
        warnings.warn(msg, SelectionPrecisionWarning, stacklevel=3)

# Every symbol include/hylra.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "hylra_abi_version",
    "hylra_status_string",
    "hylra_last_error",
    "hylra_launch_count",
    "hylra_set_tuning",
    "hylra_attention_workspace_bytes",
    "hylra_select_workspace_bytes",
    "hylra_full_decode",
    "hylra_topk_select",
    "hylra_topk_select_ex",
    "hylra_reuse_decode",
    "hylra_decode_layer",
    "hylra_decode_step_workspace_bytes",
    "hylra_decode_step",
    "hylra_decode_step_offload",
    "hylra_decode_step_ex",
    "hylra_append_kv",
    "hylra_append_kv_checked",
    "hylra_check_cache",
    "hylra_overlap_counts",
    "hylra_augment_selection",
    "hylra_block_select",
    "hylra_decode_step_blocks_workspace_bytes",
    "hylra_decode_step_blocks",
    "hylra_decode_step_blocks_ex",
    "hylra_read_flags",
    "hylra_clear_flags",
)


class Geometry(ctypes.Structure):
    """Mirror of `hylra_geometry` (include/hylra.h)."""

    _fields_ = [
        ("batch", ctypes.c_int32),
        ("q_heads", ctypes.c_int32),
        ("kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("capacity", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("num_layers", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("q_stride_layer", ctypes.c_int64),
        ("q_stride_batch", ctypes.c_int64),
        ("kv_stride_layer", ctypes.c_int64),
        ("kv_stride_batch", ctypes.c_int64),
        ("kv_stride_head", ctypes.c_int64),
        ("out_stride_layer", ctypes.c_int64),
        ("out_stride_batch", ctypes.c_int64),
    ]


class StepOptions(ctypes.Structure):
    """Mirror of `hylra_step_options` (include/hylra.h)."""

    _fields_ = [
        ("fuse_select", ctypes.c_int32),
        ("side_stream", ctypes.c_void_p),
        ("fork_event", ctypes.c_void_p),
        ("select_event", ctypes.c_void_p),
        ("full_event", ctypes.c_void_p),
        ("join_event", ctypes.c_void_p),
        ("reuse_wait_event", ctypes.c_void_p),
        ("layer_events", ctypes.c_void_p),
        ("append_k_rows", ctypes.c_void_p),
        ("append_v_rows", ctypes.c_void_p),
        ("append_pos", ctypes.c_int32),
        ("idx_mirror", ctypes.c_void_p),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libhylra.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise CudaError(
                f"{LIB_PATH} is missing: the sm_100a extension has not been built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
            )
        l = ctypes.CDLL(os.fspath(LIB_PATH))
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        gp = ctypes.POINTER(Geometry)
        l.hylra_abi_version.restype = i32
        if l.hylra_abi_version() != ABI_VERSION:
            raise CudaError(f"{LIB_PATH} implements ABI {l.hylra_abi_version()}, this binding "
                            f"needs {ABI_VERSION}: rebuild it (__graft_entry__.build())")
        l.hylra_status_string.restype = ctypes.c_char_p
        l.hylra_status_string.argtypes = [i32]
        l.hylra_last_error.restype = ctypes.c_char_p
        l.hylra_launch_count.restype = ctypes.c_uint64
        l.hylra_set_tuning.restype = i32
        l.hylra_set_tuning.argtypes = [ctypes.c_char_p, i32]
        l.hylra_attention_workspace_bytes.restype = sz
        l.hylra_attention_workspace_bytes.argtypes = [gp, i32, i32]
        l.hylra_select_workspace_bytes.restype = sz
        l.hylra_select_workspace_bytes.argtypes = [gp, i32, i32]
        l.hylra_full_decode.restype = i32
        l.hylra_full_decode.argtypes = [gp, vp, vp, vp, i32, i32, vp, vp, vp, vp, sz, vp]
        l.hylra_topk_select.restype = i32
        l.hylra_topk_select.argtypes = [gp, vp, i32, i32, i32, i32, vp, vp, vp, vp, i32, vp, vp,
                                        sz, vp]
        l.hylra_topk_select_ex.restype = i32
        l.hylra_topk_select_ex.argtypes = [gp, vp, i32, i32, i32, i32, vp, vp, vp, vp, i32, vp,
                                           vp, sz, vp, i32]
        l.hylra_reuse_decode.restype = i32
        l.hylra_reuse_decode.argtypes = [gp, vp, vp, vp, i32, i32, vp, vp, vp, vp, i32, i32,
                                         i32, vp, vp, sz, vp]
        l.hylra_decode_layer.restype = i32
        l.hylra_decode_layer.argtypes = [gp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                         vp, vp, vp, i32, vp, sz, vp]
        l.hylra_block_select.restype = i32
        l.hylra_block_select.argtypes = [gp, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, i32,
                                         vp, i32, vp, vp, vp, sz, vp]
        l.hylra_decode_step_blocks_workspace_bytes.restype = sz
        l.hylra_decode_step_blocks_workspace_bytes.argtypes = [gp, vp, i32, i32, i32, i32]
        l.hylra_decode_step_blocks.restype = i32
        l.hylra_decode_step_blocks.argtypes = [gp, vp, vp, vp, i32, vp, i32, i32, i32, i32, vp,
                                               vp, i32, vp, sz, vp]
        l.hylra_decode_step_blocks_ex.restype = i32
        l.hylra_decode_step_blocks_ex.argtypes = [gp, vp, vp, vp, i32, vp, i32, i32, i32, i32,
                                                  vp, vp, i32, vp, sz, vp,
                                                  ctypes.POINTER(StepOptions)]
        l.hylra_decode_step_workspace_bytes.restype = sz
        l.hylra_decode_step_workspace_bytes.argtypes = [gp, vp, i32, i32, i32, i32, i32]
        l.hylra_decode_step.restype = i32
        l.hylra_decode_step.argtypes = [gp, vp, vp, vp, i32, vp, i32, i32, i32, i32, i32, vp,
                                        vp, i32, vp, sz, vp]
        l.hylra_decode_step_offload.restype = i32
        l.hylra_decode_step_offload.argtypes = [gp, vp, vp, vp, vp, vp, i32, vp, i32, i32, i32,
                                                i32, i32, vp, vp, i32, vp, sz, vp]
        l.hylra_decode_step_ex.restype = i32
        l.hylra_decode_step_ex.argtypes = [gp, vp, vp, vp, i32, vp, i32, i32, i32, i32, i32,
                                           vp, vp, i32, vp, sz, vp, ctypes.POINTER(StepOptions)]
        l.hylra_append_kv.restype = i32
        l.hylra_append_kv.argtypes = [gp, vp, vp, vp, vp, i32, i32, vp, vp]
        l.hylra_append_kv_checked.restype = i32
        l.hylra_append_kv_checked.argtypes = [gp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
        l.hylra_check_cache.restype = i32
        l.hylra_check_cache.argtypes = [gp, vp, vp, i32, i32, vp, vp, vp]
        l.hylra_augment_selection.restype = i32
        l.hylra_augment_selection.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, i32, vp, vp]
        l.hylra_overlap_counts.restype = i32
        l.hylra_overlap_counts.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, vp]
        l.hylra_read_flags.restype = i32
        l.hylra_read_flags.argtypes = [vp, vp, vp]
        l.hylra_clear_flags.restype = i32
        l.hylra_clear_flags.argtypes = [vp, vp]
        _ = i64
        _lib = l
    return _lib


def check(status: int) -> None:
    """Raise the reference exception class matching a non-zero ABI status."""
    if status == 0:
        return
    detail = lib().hylra_last_error().decode(errors="replace")
    cls = STATUS_TO_ERROR.get(status, LayerReuseError)
    raise cls(detail or lib().hylra_status_string(status).decode())


def launch_count() -> int:
    return int(lib().hylra_launch_count())


class tuning:
    """Context manager over hylra_set_tuning: `with _abi.tuning(rowsel=0): ...` runs the
    block with the process-wide knobs set and restores the default rules afterwards."""

    def __init__(self, **knobs):
        self.knobs = knobs

    def __enter__(self):
        for name, value in self.knobs.items():
            check(lib().hylra_set_tuning(name.encode(), int(value)))
        return self

    def __exit__(self, *exc):
        for name in self.knobs:
            lib().hylra_set_tuning(name.encode(), -1)
        return False


def int32_array(values) -> ctypes.Array:
    values = list(values)
    return (ctypes.c_int32 * max(len(values), 1))(*values)


def pointer_array(values) -> ctypes.Array:
    """void* [n] (None -> NULL), e.g. per-layer cudaEvent_t handles."""
    values = list(values)
    return (ctypes.c_void_p * max(len(values), 1))(*values)


def uint8_array(values) -> ctypes.Array:
    values = list(values)
    return (ctypes.c_uint8 * max(len(values), 1))(*values)
