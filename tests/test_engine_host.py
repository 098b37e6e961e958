"""Host-side logic of HybridDecoder / DecodeLoop that needs no GPU: schedule eligibility,
the static auto rule, argument validation (CPU tensors; nothing is launched)."""
import pytest

torch = pytest.importorskip("torch")

from paper_2602_00777_b200 import ConfigurationError, InvalidInputError  # noqa: E402
from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402


def _cache(L=4, B=1, Hkv=2, cap=64, d=64, dtype=torch.float32):
    k = torch.zeros((L, B, Hkv, cap, d), dtype=dtype)
    return k, k.clone()


def test_fp32_caches_run_the_three_launch_step_only():
    k, v = _cache()
    dec = HybridDecoder(("full", "reuse", "full", "reuse"), k, v, 8, q_heads=4)
    assert dec.schedule == "fused3" and not dec.single and dec.kernels_per_step == 3
    for name in ("single", "fusedsel"):
        with pytest.raises(ConfigurationError, match="tensor-core"):
            dec.set_schedule(name)
    with pytest.raises(ConfigurationError, match="unknown schedule"):
        dec.set_schedule("warp-speed")


def test_policy_and_budget_validation():
    k, v = _cache()
    with pytest.raises(InvalidInputError, match="first layer"):
        HybridDecoder(("reuse", "full", "full", "reuse"), k, v, 8, q_heads=4)
    with pytest.raises(InvalidInputError, match="budget"):
        HybridDecoder(("full", "reuse", "full", "reuse"), k, v, 0, q_heads=4)
    with pytest.raises(ConfigurationError, match="layers"):
        HybridDecoder(("full", "reuse"), k, v, 8, q_heads=4)
    with pytest.raises(ConfigurationError, match="sel_group"):
        HybridDecoder(("full", "reuse", "full", "reuse"), k, v, 8, q_heads=4, sel_group=3)


def test_block_mode_schedules():
    k, v = _cache()
    dec = HybridDecoder(("full", "reuse", "full", "reuse"), k, v, 4, q_heads=4, block_size=8)
    assert dec.schedule == "fused3" and dec.kernels_per_step == 5
    with pytest.raises(ConfigurationError, match="token mode"):
        dec.set_schedule("fusedsel")
