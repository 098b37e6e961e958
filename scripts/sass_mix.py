"""Instruction mix of every kernel in libhylra.so (cuobjdump -sass; no GPU needed): per
kernel, counts of the SASS mnemonics that show which hardware paths it uses — TMA
(UTMALDG, UBLKCP), cp.async gathers (LDGSTS), tensor cores (HMMA / UTCMMA), mbarriers
(SYNCS), shared / global atomics (ATOMS, ATOMG, RED), FP64 (DFMA), warp collectives, CTA
and cluster barriers.
    python scripts/sass_mix.py [lib] > profiles/r02_sass_mix.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2602_00777_b200/libhylra.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["UTMALDG", "UBLKCP", "UTCMMA", "LDGSTS", "HMMA", "SYNCS", "LDG", "STG", "LDS", "STS",
       "ATOMS", "ATOMG", "RED", "REDG", "DFMA", "SHFL", "VOTE", "MATCH", "BAR", "UCGABAR_ARV",
       "UCGABAR_WAIT", "MUFU"]
mix, fn = collections.OrderedDict(), None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        mix[fn] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if fn and m:
        mix[fn][m.group(1)] += 1
names = subprocess.run(["c++filt"], input="\n".join(mix), capture_output=True,
                       text=True).stdout.splitlines()
for (raw, c), name in zip(mix.items(), names):
    name = re.sub(r"\(.*", "", name).replace("hylra::", "")
    total = sum(c.values())
    print(f"{name}  [{total} instr]: " + " ".join(f"{op}={c[op]}" for op in OPS if c[op]))
