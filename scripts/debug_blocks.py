import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import torch
from oracle import hylra_oracle as orc
from paper_2602_00777_b200.attention import full_attention, block_select, topk_select
from refmodel import load_npz
z = load_npz("tests/golden/block_reference.npz")
for n in (512, 513):
    K = torch.tensor(z["keys"][:, :, :n], dtype=torch.float32).cuda()[:, None]   # [L,1,H,n,d]
    V = torch.tensor(z["values"][:, :, :n], dtype=torch.float32).cuda()[:, None]
    t = n - 512
    Q = torch.tensor(z["queries"][t], dtype=torch.float32).cuda()[:, None]       # [L,1,H,d]
    out, sc = full_attention(Q, K.contiguous(), V.contiguous(), n)
    for refine in (False, True):
        bl, tok, cnt, inf = block_select(sc, 2, 128, n, sel_group=2, q=Q if refine else None, k=K.contiguous() if refine else None, info=True)
        print(n, refine, bl[:, 0, 0].cpu().numpy().tolist(), cnt[:, 0, 0].cpu().numpy().tolist(), inf[:, 0, 0, :4].cpu().numpy().tolist())
    s = sc[:, 0, :, :n].sum(1).double().cpu().numpy()
    print("fp32 block maxima", [orc.block_max_of_logits(s[l], 128).round(6).tolist() for l in range(2)])
    print("oracle", [orc.topk_of_logits(orc.block_max_of_logits(s[l], 128), 2).tolist() for l in range(5)])
    # tiny token rows
    idx, inf = topk_select(torch.tensor(np.array([[[[3.0, 1.0, 2.0, 0.5, 0, 0, 0, 0]]]], dtype=np.float32)).cuda(), 2, 4, info=True)
    print("tiny", idx.cpu().numpy().ravel().tolist(), inf.cpu().numpy().ravel().tolist())
