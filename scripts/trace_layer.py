"""Per-CTA timeline of one layer-sequential FULL launch and one REUSE launch from a
diagnostics build (-DHYLRA_TRACE):
    python scripts/trace_layer.py --build            # here: paper_2602_00777_b200/build_trace/
    HYLRA_LIB=$PWD/paper_2602_00777_b200/build_trace/libhylra_trace.so \\
        python scripts/trace_layer.py [--batch 1]     # on the GPU
Marks per CTA (globaltimer, ns): start, first stage consumed, main loop end, done."""
import argparse
import ctypes
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", default="full,reuse")
a = ap.parse_args()

if a.build:
    import __graft_entry__ as ge
    out = ge.PKG / "build_trace"
    flags = [f for f in ge.NVCC_FLAGS if f != "-shared"] + ["-DHYLRA_TRACE"]
    objs = ge._compile_units(ge.UNITS, flags, False, obj_dir=out)
    subprocess.run([ge._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                    str(out / "libhylra_trace.so"), *map(str, objs)], check=True)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_00777_b200 import _abi  # noqa: E402
from paper_2602_00777_b200.engine import LayerwiseDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402

cfg = CONFIGS["cfg2"].with_(batch=a.batch)
q, k, v = generate_torch(cfg, "cuda")
n = cfg.context
dec = LayerwiseDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
for _ in range(2):
    dec.step(q, n)
torch.cuda.synchronize()
lib = _abi.lib()
for f in ("hylra_trace_set_full", "hylra_trace_set_reuse"):
    getattr(lib, f).argtypes = [ctypes.c_void_p]
buf = torch.zeros(100000 * 8, dtype=torch.int64, device="cuda")
full = [l for l, x in enumerate(cfg.actions) if x == "full"]
reuse = [l for l, x in enumerate(cfg.actions) if x == "reuse"]
bytes_row = cfg.head_dim * 2 * 2  # K + V bf16
for kind in a.layers.split(","):
    l = full[0] if kind == "full" else reuse[0]
    setter = lib.hylra_trace_set_full if kind == "full" else lib.hylra_trace_set_reuse
    buf.zero_()
    # flush L2 so the launch reads HBM
    junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    junk.fill_(1)
    torch.cuda.synchronize()
    setter(buf.data_ptr())
    dec._prev = "reuse"
    dec.layer(l, q, n)
    dec.finish()
    torch.cuda.synchronize()
    setter(None)
    t = buf.view(-1, 8).cpu().numpy()
    t = t[t[:, 0] != 0]
    t0 = t[:, 0].min()
    rel = (t[:, [0, 6, 7, 4]] - t0) / 1e3
    rows = (cfg.context if kind == "full" else cfg.budget) * cfg.batch * cfg.kv_heads
    total = rows * bytes_row
    end = rel[:, 3].max()
    print(f"{kind} layer {l}: {len(t)} CTAs, {total / 1e6:.1f} MB, first start -> last done "
          f"{end:.2f} us ({total / end / 1e3:.0f} GB/s)")
    for name, j in (("start", 0), ("first stage", 1), ("loop end", 2), ("done", 3)):
        c = rel[:, j]
        print(f"  {name:12s} min {c.min():7.2f}  p10 {np.percentile(c, 10):7.2f}  "
              f"p50 {np.median(c):7.2f}  p90 {np.percentile(c, 90):7.2f}  max {c.max():7.2f} us")
    d = rel[:, 2] - rel[:, 1]
    print(f"  loop (first stage -> loop end) p50 {np.median(d):.2f} us; "
          f"merge (loop end -> done) p50 {np.median(rel[:, 3] - rel[:, 2]):.2f} "
          f"max {np.max(rel[:, 3] - rel[:, 2]):.2f} us")
    sm = t[:, 5]
    print(f"  SMs used {len(np.unique(sm))}, CTAs per SM max {np.bincount(sm).max()}")
