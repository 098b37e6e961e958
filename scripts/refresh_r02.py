"""Copy a scripts/gpu_profile.sh bundle from gpurun_out/ into profiles/ (round tag r02) and
refresh the derived files: profiles/r02_launch_shares.txt (from the launch list) and
profiles/ncu_summary.json (DRAM traffic per launch from the ncu --set full summaries).
    python scripts/refresh_r02.py"""
import collections
import csv
import json
import shutil
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
G, P = ROOT / "gpurun_out", ROOT / "profiles"
for f in G.glob("r02_ncu_*"):
    shutil.copy(f, P / f.name)
shutil.copy(G / "launches.csv", P / "r02_launches_cfg2_b8.csv")
for src, dst in (("bench.json", "r02_bench_cfg2_b8.json"),
                 ("bench_ref.json", "r02_bench_reference_arm.json")):
    lines = [l for l in open(G / src) if l.strip().startswith("{")]
    (P / dst).write_text(lines[-1])


def tb(r):
    return (r["dram_read_bytes"] or 0) + (r["dram_write_bytes"] or 0)


s = json.load(open(P / "r02_ncu_single_cfg2_b8.json"))
f = json.load(open(P / "r02_ncu_fusedsel_cfg2_b8.json"))
b1 = json.load(open(P / "r02_ncu_fused3_cfg2_b1.json"))
out = json.load(open(P / "ncu_summary.json"))
out["cfg2_b8"].update({"step_traffic_bytes_per_launch": tb(s[0]),
                       "full_traffic_bytes_per_launch": tb(f[0]),
                       "select_traffic_bytes_per_launch": tb(f[1]),
                       "reuse_traffic_bytes_per_launch": tb(f[2])})
out["cfg2_b1"].update({"full_traffic_bytes_per_launch": tb(b1[0]),
                       "select_traffic_bytes_per_launch": tb(b1[1]),
                       "reuse_traffic_bytes_per_launch": tb(b1[2])})
json.dump(out, open(P / "ncu_summary.json", "w"), indent=1)

# launch list: ncu CSV rows (ID, ..., Kernel Name, ..., Metric Value)
rows = list(csv.DictReader(l for l in open(P / "r02_launches_cfg2_b8.csv")
                           if l.startswith('"')))
name_key = "Kernel Name"
unit_scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
launches = [(r[name_key], float(r["Metric Value"].replace(",", "")) *
             unit_scale.get(r.get("Metric Unit", "ns"), 1e-3)) for r in rows]


def short(n):
    n = n.replace("hylra::", "").replace("void ", "")
    return n.split("(")[0]


tail = []
for n, t in reversed(launches):
    if "step_mma_kernel" not in n:
        if tail:
            break
        continue
    tail.append(t)
tot = collections.OrderedDict()
for n, t in launches:
    k = short(n)
    c, s_ = tot.get(k, (0, 0.0))
    tot[k] = (c + 1, s_ + t)
all_t = sum(t for _, t in launches)
txt = ["ncu --metrics gpu__time_duration.sum --clock-control none launch list of",
       "`python bench.py --steps 2 --warmup 3 --no-extra --no-cpu` (cfg2 B=8; autotune runs every "
       "schedule first)", "",
       f"headline run (last consecutive step_mma_kernel launches): {len(tail)} launches, mean "
       f"{sum(tail) / max(1, len(tail)):.1f} us each (ncu: serialised, cold cache)",
       "the headline step = 1 kernel (step_mma_kernel) = 100% of the step's launch time", "",
       "all launches of the command, by kernel:"]
for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    txt.append(f"  {k[:110]:48s} {c:5d} launches {t / 1e3:10.3f} ms {100 * t / all_t:6.1f}%")
(P / "r02_launch_shares.txt").write_text("\n".join(txt) + "\n")
print("\n".join(txt[:12]))
print(json.dumps(out, indent=1))
