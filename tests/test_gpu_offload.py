"""Index-guided offload (engine.py:314-368 offload mirror): REUSE layers' K/V
in pinned host memory, read in place over the link. Same kernels as the resident path, so
outputs and selections must be bit-identical to HybridDecoder on the same cache."""
import ctypes

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from oracle import hylra_oracle as orc  # noqa: E402
from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.engine import HybridDecoder, OffloadDecoder  # noqa: E402
from paper_2602_00777_b200.errors import ConfigurationError  # noqa: E402
from test_gpu_kernels import make_stack, max_head_err  # noqa: E402

ACTS = ("full", "reuse", "reuse", "full", "reuse", "reuse")


@pytest.mark.parametrize("dtype,sinks,recent,on_device", [
    ("bf16", 0, 0, False), ("bf16", 4, 16, False), ("f32", 0, 0, False), ("bf16", 0, 0, True)])
def test_offload_equals_resident(dtype, sinks, recent, on_device):
    L, B, Hq, Hkv, d, cap, n, k = 6, 2, 16, 4, 128, 4096, 4000, 256
    q, kc, vc, qn, kn, vn = make_stack(L, B, Hq, Hkv, d, cap, dtype, seed=3, planted=32)
    res_dec = HybridDecoder(ACTS, kc, vc, k, q_heads=Hq, include_sinks=sinks,
                            include_recent=recent)
    ref = res_dec.step(q, n)
    torch.cuda.synchronize()
    kf, vf, kr, vr = OffloadDecoder.split_cache(ACTS, kc, vc)
    if on_device:
        kr, vr = kr.cuda(), vr.cuda()
    else:
        assert kr.is_pinned() and not kr.is_cuda
    dec = OffloadDecoder(ACTS, kf, vf, kr, vr, k, q_heads=Hq, include_sinks=sinks,
                         include_recent=recent)
    got = dec.step(q, n)
    torch.cuda.synchronize()
    dec.check_flags()
    assert torch.equal(got.outputs, ref.outputs)
    assert torch.equal(got.selections, ref.selections)
    if sinks == 0 and recent == 0:
        ref_out, ref_sets, _ = orc.hybrid_step(qn, kn, vn, n, ACTS, k)
        for l in range(L):
            assert np.array_equal(got.selection(l).cpu().numpy(), ref_sets[l])
        tol = 2e-2 if dtype == "bf16" else 1e-3
        assert max_head_err(got.outputs.double().cpu().numpy(), ref_out) < tol


def test_offload_rejects_pageable_memory():
    L, B, Hq, Hkv, d, cap = 6, 1, 8, 2, 128, 1024
    q, kc, vc, *_ = make_stack(L, B, Hq, Hkv, d, cap, "bf16", seed=1)
    kf, vf, kr, vr = OffloadDecoder.split_cache(ACTS, kc, vc)
    with pytest.raises(ConfigurationError):
        OffloadDecoder(ACTS, kf, vf, kr.clone(), vr.clone(), 64, q_heads=Hq)  # unpinned copies
    # and at the C ABI: a pageable host pointer is refused, not dereferenced
    dec = OffloadDecoder(ACTS, kf, vf, kr, vr, 64, q_heads=Hq)
    g = dec._geometry(q)
    page = np.zeros(kr.numel(), dtype=np.uint16)
    ws = torch.zeros(int(_abi.lib().hylra_decode_step_workspace_bytes(
        g, dec._acts, cap, 64, 1, 0, 0)), dtype=torch.uint8, device="cuda")
    st = _abi.lib().hylra_decode_step_offload(
        g, q.data_ptr(), kf.data_ptr(), vf.data_ptr(), page.ctypes.data_as(ctypes.c_void_p),
        vr.data_ptr(), cap, dec._acts, 64, 1, 1, 0, 0, dec.out.data_ptr(), dec.idx.data_ptr(),
        dec.k_stride, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert st == _abi.HYLRA_ERR_CONFIGURATION
    assert b"page-locked" in _abi.lib().hylra_last_error()
