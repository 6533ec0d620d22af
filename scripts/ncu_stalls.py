"""Warp-stall breakdown of an ncu report restricted to instructions whose
execution count matches a given per-role count (e.g. the softmax loop body).

    python scripts/ncu_stalls.py rep.ncu-rep [exec_count ...]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
want = {int(x) for x in sys.argv[2:]}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
ex = h.index("Instructions Executed")
src = h.index("Source")
tot = Counter()
n = 0
execs = Counter()
for r in rows[hi + 1:]:
    if len(r) <= max(cols):
        continue
    e = int(float(r[ex] or 0))
    execs[e] += 1
    if want and e not in want:
        continue
    n += 1
    for c in cols:
        tot[h[c]] += float(r[c] or 0)
s = sum(tot.values())
print(f"{n} instructions, {s:.0f} samples")
for k, v in tot.most_common():
    if v:
        print(f"  {k:22s} {v:8.0f} {v / s:6.1%}")
if not want:
    print("most common execution counts:", execs.most_common(12))
