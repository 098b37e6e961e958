"""Summarise an ncu report: per kernel launch, key SOL / memory / occupancy metrics and
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum). Usage:
    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Issue Slots Busy", "L2 Hit Rate", "Waves Per SM", "Dynamic Shared Memory Per Block",
        "Warp Cycles Per Issued Instruction"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, ni, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                           h.index("Metric Unit"), h.index("ID"))
    res = {}
    for r in rows[1:]:
        key = (r[idi], r[ki])
        if r[ni] in WANT:
            res.setdefault(key, {})[r[ni]] = f"{r[vi]} {r[ui]}"
    return res


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        def get(m):
            v = d.get(m)
            if v is None:
                return None
            v = float(v.replace(",", ""))
            # bytes to B, times to ns (ncu picks the unit per value: a 1.46 ms launch is
            # reported as "1.46 msecond", not in ns)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
                     "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}.get(u.get(m, "byte"), 1)
            return v * scale
        res.append({"id": d.get("ID"), "kernel": d.get("Kernel Name"),
                    "dram_read_bytes": get("dram__bytes_read.sum"),
                    "dram_write_bytes": get("dram__bytes_write.sum"),
                    "duration_ns": get("gpu__time_duration.sum")})
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    det = details(rep)
    rw = raw(rep)
    summary = []
    for r in rw:
        key = next((k for k in det if k[0] == r["id"]), None)
        r["metrics"] = det.get(key, {})
        tb = (r["dram_read_bytes"] or 0) + (r["dram_write_bytes"] or 0)
        r["traffic_bytes"] = tb
        summary.append(r)
        print(f"[{r['id']}] {r['kernel'][:90]}")
        print(f"    dram read {r['dram_read_bytes']:.4g} B  write {r['dram_write_bytes']:.4g} B  "
              f"duration {r['duration_ns']} ns")
        for m, v in r["metrics"].items():
            print(f"    {m}: {v}")
    if "--json" in sys.argv:
        json.dump(summary, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
