"""Time the REUSE launch of a BASELINE config (all REUSE layers in one launch):
    python scripts/reuse_sweep.py [cfg2] [batch]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.attention import geometry  # noqa: E402
from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
if len(sys.argv) > 2:
    cfg = cfg.with_(batch=int(sys.argv[2]))
q, k, v = generate_torch(cfg, "cuda")
dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
dec.step(q, cfg.context)
torch.cuda.synchronize()
g = geometry(q, k, v, dec.out)
rl = [l for l in range(cfg.layers) if cfg.actions[l] == "reuse"]
src = [dec.slot_of_layer[l] for l in rl]
ke = min(cfg.budget, cfg.context)
ws = torch.zeros(_abi.lib().hylra_attention_workspace_bytes(g, len(rl), ke), dtype=torch.uint8,
                 device="cuda")
st = torch.cuda.current_stream().cuda_stream


def op():
    _abi.check(_abi.lib().hylra_reuse_decode(g, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             cfg.context, len(rl), _abi.int32_array(rl),
                                             _abi.int32_array(src), dec.idx.data_ptr(), None,
                                             dec.k_stride, ke, 1, dec.out.data_ptr(),
                                             ws.data_ptr(), ws.numel(), st))


for _ in range(3):
    op()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    op()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
by = len(rl) * cfg.batch * cfg.kv_heads * 2 * ke * cfg.head_dim * 2
print(f"{cfg.name} B={cfg.batch} reuse {ms * 1e3:.1f} us  {by / ms / 1e6:.0f} GB/s", flush=True)
