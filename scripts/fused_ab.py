#!/usr/bin/env python
"""Interleaved A/B of the fused call (blade_asa_fwd / blade_asa_gt_fwd) against
the separate calls on the same inputs: alternating blocks of 50 steps, three
rounds, so clock / power drift hits both arms alike."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs  # noqa: E402

wl, mode = sys.argv[1], sys.argv[2]  # mode: keep | tau | gt
keep = {"wan": 51, "cog": 25}[wl]
q, k, v = (x.cuda() for x in inputs.make(wl, "smooth"))
kw = dict(tau=0.9) if mode == "tau" else dict(tau=0.9, keep_min=keep, keep_max=keep)
st = torch.cuda.current_stream()


def two():
    if mode == "gt":
        A.asa_gt_forward(q, k, v, window=128, **kw)
    else:
        A.asa_forward(q, k, v, **kw)


fo = [None]


def fused():
    if mode == "gt":
        fo[0] = A.blade_asa_gt_fwd(q, k, v, window=128, out=fo[0], **kw)
    else:
        fo[0] = A.blade_asa_fwd(q, k, v, out=fo[0], **kw)


def block(f, n=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        f()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for f in (two, fused):
    for _ in range(5):
        f()
torch.cuda.synchronize()
res = {"two": [], "fused": []}
for r in range(3):
    order = (("two", two), ("fused", fused)) if r % 2 == 0 else (("fused", fused), ("two", two))
    for name, f in order:
        res[name].append(block(f))
print(json.dumps({"workload": wl, "mode": mode, **{k: [round(x, 4) for x in v] for k, v in res.items()},
                  "median_two": round(statistics.median(res["two"]), 4),
                  "median_fused": round(statistics.median(res["fused"]), 4)}))
