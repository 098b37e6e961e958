"""Timeline of one single-launch step from a diagnostics build (-DHYLRA_TRACE):
    nvcc ... -DHYLRA_TRACE -o build/libhylra_trace.so .../hylra_abi.cu
    HYLRA_LIB=$PWD/build/libhylra_trace.so python scripts/trace_single.py [--batch 1]
Per CTA (ticket order): globaltimer at ticket, fused select start/end, REUSE ready, done."""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
cfg = CONFIGS[a.config].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads, single_launch=True)
for _ in range(3):
    dec.step(q, cfg.context)
torch.cuda.synchronize()
buf = torch.zeros(200000 * 8, dtype=torch.int64, device="cuda")
lib = _abi.lib()
lib.hylra_trace_set.argtypes = [ctypes.c_void_p]
lib.hylra_trace_set(buf.data_ptr())
info = torch.zeros(100000 * 8, dtype=torch.int32, device="cuda")
lib.hylra_trace_set_select_info.argtypes = [ctypes.c_void_p]
lib.hylra_trace_set_select_info(info.data_ptr())
dec.step(q, cfg.context)
torch.cuda.synchronize()
lib.hylra_trace_set(None)
lib.hylra_trace_set_select_info(None)
inf = info.view(-1, 8).cpu().numpy()
inf = inf[inf[:, 0] != 0]
if len(inf):
    names = (["hist", "row pass", "T+window", "rescore+rank"] if (inf[:, 2] == 6).all()
             else ["A sample", "B pass(+H)", "C+D", "E window+compact"])
    print("  fused select phases (median cycles):",
          {nm: int(np.median(inf[:, 4 + j])) for j, nm in enumerate(names)},
          "modes", dict(zip(*[x.tolist() for x in np.unique(inf[:, 2], return_counts=True)])),
          "band median", int(np.median(inf[:, 3])), "compaction (diag build)",
          int(np.median(inf[:, 1])))
tr = buf.view(-1, 8).cpu().numpy()
n = int((tr[:, 0] != 0).sum())
tr = tr[:n]
t0 = tr[:, 0].min()
rel = lambda x: (x - t0) / 1e3  # noqa: E731
done = rel(tr[:, 4])
sel = tr[:, 1] != 0
ready = tr[:, 2] != 0
full = ~ready & (np.arange(n) < n)  # FULL tickets come first
n_reuse = int(ready.sum())
n_full = n - n_reuse
print(f"{cfg.name} B={a.batch}: {n} CTAs ({n_full} FULL, {n_reuse} REUSE), step span "
      f"{done.max():.1f} us")
f = slice(0, n_full)
print(f"  FULL items: start {rel(tr[f, 0]).min():.1f}..{rel(tr[f, 0]).max():.1f}, "
      f"done {done[f].min():.1f}..{done[f].max():.1f} us")
if sel.any():
    print(f"  fused selects ({int(sel.sum())}): start {rel(tr[sel, 1]).min():.1f}..{rel(tr[sel, 1]).max():.1f},"
          f" end {rel(tr[sel, 3]).min():.1f}..{rel(tr[sel, 3]).max():.1f}, median length "
          f"{np.median(rel(tr[sel, 3]) - rel(tr[sel, 1])):.1f} us")
r = slice(n_full, n)
if n_reuse:
    wait = rel(tr[r, 2]) - rel(tr[r, 0])
    print(f"  REUSE items: claimed {rel(tr[r, 0]).min():.1f}..{rel(tr[r, 0]).max():.1f}, ready "
          f"{rel(tr[r, 2]).min():.1f}..{rel(tr[r, 2]).max():.1f}, done {done[r].min():.1f}.."
          f"{done[r].max():.1f} us; wait median {np.median(wait):.1f} max {wait.max():.1f}; "
          f"gather median {np.median(done[r] - rel(tr[r, 2])):.1f} us")
    hist = np.histogram(rel(tr[r, 0]), bins=8)
    print("  REUSE claim histogram", hist[0].tolist(), np.round(hist[1], 0).tolist())
