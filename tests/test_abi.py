"""The C-ABI library loads without a GPU, exports every symbol include/hylra.h declares,
and maps argument errors to the reference's exception classes (host-side validation runs
before any CUDA call)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2602_00777_b200 import _abi
from paper_2602_00777_b200.errors import ConfigurationError, InvalidInputError

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "hylra.h").read_text()
    # function declarations: "<return type> hylra_name(" at the start of a line
    pat = r"^(?:const\s+)?\w+\s*\**\s*(hylra_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(pat, text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    declared = header_symbols()
    assert len(declared) >= 14
    assert sorted(_abi.EXPORTED_SYMBOLS) == declared
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.hylra_abi_version() == _abi.ABI_VERSION
    assert lib.hylra_status_string(3) == b"InvalidSelectionError"


def _geom(**kw):
    g = _abi.Geometry()
    g.batch, g.q_heads, g.kv_heads, g.head_dim = 1, 8, 2, 64
    g.capacity, g.dtype, g.num_layers = 2048, _abi.HYLRA_F32, 4
    g.q_stride_layer, g.q_stride_batch = 8 * 64, 8 * 64
    g.kv_stride_head = 2048 * 64
    g.kv_stride_batch = 2 * 2048 * 64
    g.kv_stride_layer = 2 * 2048 * 64
    g.out_stride_layer, g.out_stride_batch = 8 * 64, 8 * 64
    for k, v in kw.items():
        setattr(g, k, v)
    return g


def test_workspace_queries_are_host_only():
    lib = _abi.lib()
    g = _geom()
    assert lib.hylra_attention_workspace_bytes(g, 2, 2048) > 256
    acts = _abi.uint8_array([1, 0, 1, 0])
    assert lib.hylra_decode_step_workspace_bytes(g, acts, 2048, 128, 1, 0, 0) > 0
    assert lib.hylra_decode_step_workspace_bytes(_geom(q_heads=7), acts, 2048, 128, 1, 0, 0) == 0


def test_status_codes_map_to_reference_exceptions():
    lib = _abi.lib()
    acts = _abi.uint8_array([0, 1, 1, 0])  # first layer REUSE
    with pytest.raises(InvalidInputError, match="first layer"):
        _abi.check(lib.hylra_decode_step(_geom(), None, None, None, 2048, acts, 128, 1, 1, 0, 0,
                                         None, None, 128, None, 0, None))
    with pytest.raises(InvalidInputError, match="budget"):
        _abi.check(lib.hylra_decode_step(_geom(), None, None, None, 2048,
                                         _abi.uint8_array([1, 0, 1, 0]), 0, 1, 1, 0, 0, None,
                                         None, 128, None, 0, None))
    with pytest.raises(ConfigurationError, match="multiple"):
        _abi.check(lib.hylra_decode_step(_geom(q_heads=7), None, None, None, 2048,
                                         _abi.uint8_array([1, 0, 1, 0]), 128, 1, 1, 0, 0, None,
                                         None, 128, None, 0, None))
    with pytest.raises(InvalidInputError, match="sinks"):
        _abi.check(lib.hylra_decode_step(_geom(), None, None, None, 2048,
                                         _abi.uint8_array([1, 0, 1, 0]), 128, 1, 1, -1, 0, None,
                                         None, 128, None, 0, None))
    with pytest.raises(ConfigurationError, match="head_dim"):
        _abi.check(lib.hylra_full_decode(_geom(head_dim=80), None, None, None, 10, 1,
                                         _abi.int32_array([0]), None, None, None, 0, None))
    with pytest.raises(ConfigurationError, match="workspace"):
        _abi.check(lib.hylra_decode_step(_geom(), 1, 1, 1, 2048,
                                         _abi.uint8_array([1, 0, 1, 0]), 128, 1, 1, 0, 0, 1, 1,
                                         128, None, 0, None))


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2602_00777_b200.errors import CudaError
    monkeypatch.setattr(_abi, "LIB_PATH", tmp_path / "libhylra.so")
    monkeypatch.setattr(_abi, "_lib", None)
    with pytest.raises(CudaError, match="not been built"):
        _abi.lib()


def test_step_ex_and_append_validate_on_the_host():
    lib = _abi.lib()
    g = _geom()
    acts = _abi.uint8_array([1, 0, 1, 0])
    need = lib.hylra_decode_step_workspace_bytes(g, acts, 2048, 128, 1, 0, 0)
    opt = _abi.StepOptions()
    opt.side_stream = 1  # a side stream without its four events
    with pytest.raises(ConfigurationError, match="four events"):
        _abi.check(lib.hylra_decode_step_ex(g, 1, 1, 1, 2048, acts, 128, 1, 1, 0, 0, 1, 1, 128,
                                            1, need, None, ctypes.byref(opt)))
    with pytest.raises(InvalidInputError, match="first layer"):
        _abi.check(lib.hylra_decode_step_ex(g, 1, 1, 1, 2048, _abi.uint8_array([0, 1, 1, 0]),
                                            128, 1, 1, 0, 0, 1, 1, 128, 1, need, None, None))
    with pytest.raises(InvalidInputError, match="pos"):
        _abi.check(lib.hylra_append_kv(g, 1, 1, 1, 1, 2048, 0, None, None))
    with pytest.raises(ConfigurationError, match="NULL"):
        _abi.check(lib.hylra_append_kv(g, None, 1, 1, 1, 5, 0, None, None))


def test_step_append_options_validate_on_the_host():
    """hylra_step_options append_* (ABI 5): both row buffers or neither, and a position
    inside the attended rows; rejected before anything is launched."""
    lib = _abi.lib()
    g = _geom()
    acts = _abi.uint8_array([1, 0, 1, 0])
    need = lib.hylra_decode_step_workspace_bytes(g, acts, 2048, 128, 1, 0, 0)
    opt = _abi.StepOptions()
    opt.fuse_select = 2
    opt.append_k_rows = 1
    with pytest.raises(ConfigurationError, match="both"):
        _abi.check(lib.hylra_decode_step_ex(g, 1, 1, 1, 2048, acts, 128, 1, 1, 0, 0, 1, 1, 128,
                                            1, need, None, ctypes.byref(opt)))
    opt.append_v_rows = 1
    opt.append_pos = 2048
    with pytest.raises(InvalidInputError, match="append_pos"):
        _abi.check(lib.hylra_decode_step_ex(g, 1, 1, 1, 2048, acts, 128, 1, 1, 0, 0, 1, 1, 128,
                                            1, need, None, ctypes.byref(opt)))


def test_layer_runs():
    from paper_2602_00777_b200.engine import _runs
    assert _runs([]) == []
    assert _runs([0, 1, 2, 8, 15, 16, 24, 31]) == [(0, 3), (8, 9), (15, 17), (24, 25), (31, 32)]
    assert _runs(range(3, 8)) == [(3, 8)]


def test_block_step_append_options_validate_on_the_host():
    """hylra_decode_step_blocks_ex takes the same append_* options (written by the
    single-launch block kernel or appended ahead): validated before any launch."""
    lib = _abi.lib()
    g = _geom()
    acts = _abi.uint8_array([1, 0, 1, 0])
    need = lib.hylra_decode_step_blocks_workspace_bytes(g, acts, 2048, 16, 64, 1)
    assert need > 0
    opt = _abi.StepOptions()
    opt.fuse_select = 2
    opt.append_v_rows = 1
    with pytest.raises(ConfigurationError, match="both"):
        _abi.check(lib.hylra_decode_step_blocks_ex(g, 1, 1, 1, 2048, acts, 16, 64, 1, 1, 1, 1,
                                                   16, 1, need, None, ctypes.byref(opt)))
    opt.append_k_rows = 1
    opt.append_pos = -1
    with pytest.raises(InvalidInputError, match="append_pos"):
        _abi.check(lib.hylra_decode_step_blocks_ex(g, 1, 1, 1, 2048, acts, 16, 64, 1, 1, 1, 1,
                                                   16, 1, need, None, ctypes.byref(opt)))


def test_tuning_knobs_validate_and_restore():
    """hylra_set_tuning: known knobs accept values and -1 restores the default rule; an unknown
    knob is a ConfigurationError (no GPU needed)."""
    lib = _abi.lib()
    with _abi.tuning(gather_tma=1, bulk_merge=0, cluster_merge=0, reuse_prefetch=2,
                     fused_fine_splits=1):
        pass
    with _abi.tuning(rowsel=0, select_threads=512, rowsel_cluster=4):
        pass
    assert lib.hylra_set_tuning(b"rowsel", -1) == 0
    with pytest.raises(ConfigurationError, match="unknown tuning knob"):
        _abi.check(lib.hylra_set_tuning(b"no_such_knob", 1))
    with pytest.raises(ConfigurationError):
        _abi.check(lib.hylra_set_tuning(None, 1))


def test_decode_layer_validates_before_launching():
    """hylra_decode_layer rejects bad arguments host-side, with the reference's exception
    classes: budget < 1 -> InvalidInputError, a slot out of range / a REUSE layer without
    selections / a FULL selection without score rows -> ConfigurationError."""
    lib = _abi.lib()
    g = _geom()
    ws = (ctypes.c_uint8 * 4096)()
    args = dict(n_valid=2048, layer=0, full=1, slot=0, budget=128, sel_group=1, refine=1,
                prefetch=0)

    def call(**kw):
        a = {**args, **kw}
        return lib.hylra_decode_layer(ctypes.byref(g), 1, 1, 1, a["n_valid"], a["layer"],
                                      a["full"], a["slot"], a["budget"], a["sel_group"],
                                      a["refine"], a["prefetch"], 1, kw.get("scores"),
                                      kw.get("idx"), 128, ws, 4096, None)
    with pytest.raises(InvalidInputError):
        _abi.check(call(budget=0))
    with pytest.raises(ConfigurationError):
        _abi.check(call(slot=-1))
    with pytest.raises(ConfigurationError):
        _abi.check(call(full=0))          # REUSE without selections
    with pytest.raises(ConfigurationError):
        _abi.check(call(idx=1))           # a FULL selection needs score rows
    with pytest.raises(ConfigurationError):
        _abi.check(call(sel_group=3))     # does not divide kv_heads
