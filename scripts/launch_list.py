"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file F`):
    python scripts/launch_list.py F [kernel-regex] [--first N]
Prints, per kernel name of ours (hylra::), launches and mean duration, and each kernel's
share of the summed duration of our kernels. --first N keeps only our first N launches
(bench.py runs the headline schedule's warm-up steps first: 3 launches per fused step)."""
import collections
import csv
import re
import sys

argv = [x for x in sys.argv[1:]]
first = None
if "--first" in argv:
    i = argv.index("--first")
    first = int(argv[i + 1])
    del argv[i:i + 2]
sys.argv[1:] = argv
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
kre = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"hylra|attn_|topk_|block_|augment|overlap")
agg = collections.OrderedDict()
n_ours = 0
for r in rows:
    name = r[ki]
    if not kre.search(name):
        continue
    n_ours += 1
    if first is not None and n_ours > first:
        break
    short = re.sub(r"^void ", "", name).split("(")[0]
    agg.setdefault(short, []).append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
for name, v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v):9.1f} us  share {sum(v) / tot:6.1%}  {name}")
