"""Oracle parity at the exact bench configurations, through the exact headline schedules
("do this" 1): every FULL (layer, b, kv-head) index set equal to the
float64 oracle's, and one query head of every (layer, b, kv-head) pair (every head for a
few pairs) within the bf16 tolerance 2e-2 relative L2 (north_star).

* config 2 at B = 8 (the headline), all 32 layers, single-launch step;
* config 3 at B = 4 (128K context, KV 64 GB), single-launch step;
* config 4 at B = 16 (Qwen shape, G = 7), single-launch step;
* the DecodeLoop end-to-end step (host I/O, the new K/V row appended inside the step) at
  config 2 B = 8, checked on what reached the pinned host buffers.
"""
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from fullsize_oracle import check_step  # noqa: E402
from paper_2602_00777_b200.engine import DecodeLoop, HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,batch", [("cfg2", 8), ("cfg3", 4), ("cfg4", 16)])
def test_bench_config_single_launch_matches_oracle(name, batch):
    cfg = CONFIGS[name].with_(batch=batch)
    q, k, v = generate_torch(cfg, "cuda")
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    dec.set_schedule("single")
    assert dec.kernels_per_step == 1
    res = dec.step(q, cfg.context)
    torch.cuda.synchronize()
    dec.check_flags(strict=True)
    summary = check_step(q, k, v, cfg.context, cfg.actions, cfg.budget, res.outputs,
                         res.selections, res.slot_of_layer)
    print(name, batch, summary)
    assert summary["pairs"] == cfg.layers * batch * cfg.kv_heads
    del dec, res, q, k, v
    _free()


@pytest.mark.parametrize("batch", [1, 8])
def test_layer_sequential_decode_matches_oracle(batch):
    """The layer-sequential schedule (LayerwiseDecoder: one FULL / SELECT / REUSE launch per
    layer with early loads) at the headline config, against the float64 oracle."""
    from paper_2602_00777_b200.engine import LayerwiseDecoder
    cfg = CONFIGS["cfg2"].with_(batch=batch)
    q, k, v = generate_torch(cfg, "cuda")
    dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    res = dec.step(q, cfg.context)
    torch.cuda.synchronize()
    dec.check_flags(strict=True)
    summary = check_step(q, k, v, cfg.context, cfg.actions, cfg.budget, res.outputs,
                         res.selections, res.slot_of_layer)
    print("sequential", batch, summary)
    assert summary["pairs"] == cfg.layers * batch * cfg.kv_heads
    del dec, res, q, k, v
    _free()


def test_decode_loop_e2e_step_matches_oracle():
    cfg = CONFIGS["cfg2"]
    q, k, v = generate_torch(cfg, "cuda")
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    pos = cfg.context - 1
    loop = DecodeLoop(dec, pos)
    g = torch.Generator().manual_seed(77)
    loop.q_host.copy_(q.cpu())
    loop.k_host.copy_(torch.randn(loop.k_host.shape, generator=g).to(torch.bfloat16))
    loop.v_host.copy_(torch.randn(loop.v_host.shape, generator=g).to(torch.bfloat16))
    out = loop.run()
    dec.check_flags(strict=True)
    assert torch.equal(dec.k[:, :, :, pos].cpu(), loop.k_host)
    assert torch.equal(dec.v[:, :, :, pos].cpu(), loop.v_host)
    summary = check_step(q, dec.k, dec.v, pos + 1, cfg.actions, cfg.budget, out,
                         loop.sel_host, dec.slot_of_layer)
    print("DecodeLoop", dec.schedule, summary)
    del loop, dec, q, k, v
    _free()
