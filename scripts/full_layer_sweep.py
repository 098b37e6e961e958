"""Time a ONE-layer FULL launch (the layer-sequential schedule's FULL step) at a config:
    python scripts/full_layer_sweep.py [cfg2] [batch]
(HYLRA_FULL_WAVES / HYLRA_FULL_MIN_TILES override the split rule for A/B runs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.attention import geometry, scores_row_stride  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
if len(sys.argv) > 2:
    cfg = cfg.with_(batch=int(sys.argv[2]))
q, k, v = generate_torch(cfg, "cuda")
out = torch.empty(q.shape, dtype=torch.float32, device="cuda")
g = geometry(q, k, v, out)
sc = torch.empty((1, cfg.batch, cfg.kv_heads, scores_row_stride(cfg.context)), dtype=torch.float32,
                 device="cuda")
ws = torch.zeros(_abi.lib().hylra_attention_workspace_bytes(g, 1, cfg.context), dtype=torch.uint8,
                 device="cuda")
st = torch.cuda.current_stream().cuda_stream
layers = [l for l, a in enumerate(cfg.actions) if a == "full"]


def op(i):
    _abi.check(_abi.lib().hylra_full_decode(g, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                            cfg.context, 1, _abi.int32_array([layers[i % 8]]),
                                            out.data_ptr(), sc.data_ptr(), ws.data_ptr(),
                                            ws.numel(), st))


for i in range(3):
    op(i)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(40):
    op(i)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 40
by = cfg.batch * cfg.kv_heads * 2 * cfg.context * cfg.head_dim * 2
print(f"{cfg.name} B={cfg.batch} one FULL layer {ms * 1e3:.1f} us  {by / ms / 1e6:.0f} GB/s",
      flush=True)
