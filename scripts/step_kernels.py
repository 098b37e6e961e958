"""Eager steps of one schedule for a launch list (ncu --metrics gpu__time_duration.sum):
    python scripts/step_kernels.py [schedule] [batch] [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

sched = sys.argv[1] if len(sys.argv) > 1 else "fused3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = CONFIGS["cfg2"].with_(batch=B)
q, k, v = generate_torch(cfg, "cuda")
dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
dec.set_schedule(sched)
for _ in range(steps):
    dec.step(q, cfg.context)
torch.cuda.synchronize()
dec.check_flags()
print("ok", sched, B)
