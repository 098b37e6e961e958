"""One LayerwiseDecoder step at cfg2 (B from argv) after warm-up: the launch list of the
layer-sequential schedule for ncu (scripts/seq_ab.py times it)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import LayerwiseDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = CONFIGS["cfg2"].with_(batch=B)
q, k, v = generate_torch(cfg, "cuda")
dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
for _ in range(3):
    dec.step(q, cfg.context)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
dec.step(q, cfg.context)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
