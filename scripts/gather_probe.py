"""HBM ceiling of the REUSE access pattern (libhylra_probe.so): the same K/V rows a REUSE
launch reads, read by a load-only kernel; compared with the REUSE kernel itself.
    python scripts/gather_probe.py [--config cfg2] [--batch 8]"""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2602_00777_b200.engine import HybridDecoder  # noqa: E402
from paper_2602_00777_b200.synthetic import CONFIGS, generate_torch  # noqa: E402


def probe_lib():
    lib = ctypes.CDLL(str(ROOT / "paper_2602_00777_b200" / "libhylra_probe.so"))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    lib.hylra_probe_gather.restype = i32
    lib.hylra_probe_gather.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32, i32, i32, i32, i32,
                                       vp, vp, vp, i32, vp]
    return lib


def gather_peak(dec, q, k, v, k_eff, blocks_per_sm=(1, 2, 4, 8), reps=20):
    """Best GB/s of the load-only gather over the REUSE layers' rows, and its settings."""
    lib = probe_lib()
    L = k.shape[0]
    rl = [l for l in range(L) if dec.actions[l].value == "reuse"]
    src = [dec.slot_of_layer[l] for l in rl]
    es = k.element_size()
    B, Hkv, d = k.shape[1], k.shape[2], k.shape[4]
    sink = torch.zeros(4, dtype=torch.int32, device=k.device)
    layers = (ctypes.c_int32 * len(rl))(*rl)
    slots = (ctypes.c_int32 * len(rl))(*src)
    nbytes = len(rl) * B * Hkv * 2 * k_eff * d * es
    best = (0.0, None)
    for bps in blocks_per_sm:
        def run():
            rc = lib.hylra_probe_gather(k.data_ptr(), v.data_ptr(), dec.idx.data_ptr(),
                                        k.stride(0) * es, k.stride(1) * es, k.stride(2) * es,
                                        d * es, B, Hkv, k_eff, dec.k_stride, len(rl), layers,
                                        slots, sink.data_ptr(), bps,
                                        torch.cuda.current_stream().cuda_stream)
            assert rc == 0
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        gbs = nbytes / (e0.elapsed_time(e1) / reps * 1e-3) / 1e9
        if gbs > best[0]:
            best = (gbs, bps)
    return best


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--context", type=int, default=None)
    ap.add_argument("--budget", type=int, default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    if a.batch:
        cfg = cfg.with_(batch=a.batch)
    if a.context:
        cfg = cfg.with_(context=a.context)
    if a.budget:
        cfg = cfg.with_(budget=a.budget)
    q, k, v = generate_torch(cfg, "cuda")
    dec = HybridDecoder(cfg.actions, k, v, cfg.budget, q_heads=cfg.q_heads)
    dec.step(q, cfg.context)
    torch.cuda.synchronize()
    k_eff = min(cfg.budget, cfg.context)
    for bps in (1, 2, 4, 8, 16):
        g, _ = gather_peak(dec, q, k, v, k_eff, blocks_per_sm=(bps,))
        print(f"{cfg.name} B={cfg.batch} splits/pair={bps}: gather probe {g:.0f} GB/s")
