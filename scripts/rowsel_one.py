import sys; sys.path.insert(0, '.')
import torch
from paper_2602_00777_b200 import _abi
from paper_2602_00777_b200.attention import full_attention, topk_select
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch
cfg = CONFIGS['cfg2'].with_(batch=1)
q, k, v = generate_torch(cfg, 'cuda')
_, sc = full_attention(q, k, v, cfg.context, layers=[2])
for _ in range(3):
    idx = topk_select(sc, cfg.budget, cfg.context, q=q, k=k, layers=[2])
torch.cuda.synchronize()
print('ok')
