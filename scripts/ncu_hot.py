"""Top SASS instructions of an ncu report by warp-stall samples.

    python scripts/ncu_hot.py rep.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ex = h.index("Instructions Executed")
body = [r for r in rows[hi + 1:] if len(r) > si and r[si] not in ("", None)]
tot = sum(float(r[si]) for r in body)
print(f"total stall samples {tot:.0f}")
ops = Counter()
for r in body:
    ops[r[src].split()[0] if not r[src].strip().startswith("@") else r[src].split()[1]] += float(r[si])
print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(15)))
for i, r in sorted(enumerate(body), key=lambda x: -float(x[1][si]))[:n]:
    print(f"{float(r[si]) / tot:6.1%} idx{i:5d} exec {r[ex]:>8s}  {r[src].strip()[:90]}")
