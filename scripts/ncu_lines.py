"""Per-CUDA-source-line attribution of an ncu report (needs -lineinfo + --import-source):
    python scripts/ncu_lines.py report.ncu-rep [kernel-regex] [top]
Prints warp-stall samples and executed warp instructions per source line."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname, func, hdr, cur = {}, None, None, None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        wi, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if func is None or not re.search(kre, func):
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1][:70])
        continue
    if cur is None:
        continue
    try:
        w, i = int(r[wi] or 0), int(r[ii] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += w
    a[1] += i
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tw}  warp-instructions {ti}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*v[0]/tw:5.1f}% stall  {100*v[1]/ti:5.1f}% instr  {k[0]}:{k[1]}  {k[2]}")
