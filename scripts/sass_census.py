#!/usr/bin/env python
"""SASS census of the product kernels in lib/libblade_asa.so: per kernel, the
instructions that prove the sm_100a paths (UTC*MMA = tcgen05.mma, UTMALDG =
TMA tensor loads, LDTM / STTM = tcgen05.ld / st, MUFU.EX2, FFMA2 / FADD2
packed fp32x2, DMMA = fp64 tensor-core MMA, HMMA = legacy mma.sync).

    python scripts/sass_census.py > profiles/r02_sass_census.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_10774_b200", "lib", "libblade_asa.so")
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "MUFU.EX2", "FFMA2", "FADD2",
        "FMUL2", "FMNMX3", "DMMA", "DFMA", "HMMA", "LDGSTS", "SYNCS"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
counts = collections.OrderedDict()
name = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        counts[name] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and name:
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                counts[name][k] += 1


def short(n):
    n = re.sub(r"_ZN5blade\d+_GLOBAL__N__\w+?_\d+(\w+?)I", r"\1<", n)
    return n[:70]


print(f"# SASS census of {os.path.relpath(LIB, ROOT)} (static instruction counts)")
print("kernel".ljust(72) + "".join(k[:8].rjust(9) for k in KEYS))
for n, c in counts.items():
    if not any(c.values()):
        continue
    print(short(n).ljust(72) + "".join(str(c.get(k, 0)).rjust(9) for k in KEYS))
