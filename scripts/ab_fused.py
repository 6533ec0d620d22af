#!/usr/bin/env python
"""Interleaved A/B of whole libraries on the fused call blade_asa_fwd:
alternating blocks of 50 calls per library (BLADE_LIB names under lib/),
three rounds, same inputs.

    python scripts/ab_fused.py wan|cog keep|tau[-attn] libA.so libB.so ...
    (-attn: time blade_bsa_fwd alone on lists from the first library)
"""
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import importlib.util  # noqa: E402

from paper_2508_10774_b200 import inputs  # noqa: E402

wl, mode, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
ATTN_ONLY = mode.endswith("-attn")
mode = mode.replace("-attn", "")
keep = {"wan": 51, "cog": 25}[wl]
q, k, v = (x.cuda() for x in inputs.make(wl, "smooth"))
kw = dict(tau=0.9) if mode == "tau" else dict(tau=0.9, keep_min=keep, keep_max=keep)
mods = []
for n, lib in enumerate(libs):  # one module object per library (reload would reuse one)
    os.environ["BLADE_LIB"] = lib
    spec = importlib.util.spec_from_file_location(
        f"asa_ab{n}", os.path.join(ROOT, "paper_2508_10774_b200", "asa.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mods.append(mod)
st = torch.cuda.current_stream()
outs = {}


lists = mods[0].blade_asa_mask(q, k, **kw)


def run(i, n):
    A = mods[i]
    o = outs.get(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        if ATTN_ONLY:  # blade_bsa_fwd on the same lists
            o = A.blade_bsa_fwd(q, k, v, lists.kv_idx, lists.kv_cnt)
        else:
            o = A.blade_asa_fwd(q, k, v, out=o, **kw)
    e1.record(st)
    torch.cuda.synchronize()
    outs[i] = o
    return e0.elapsed_time(e1) / n


for i in range(len(libs)):
    run(i, 5)
res = {lib: [] for lib in libs}
for r in range(3):
    for i in (range(len(libs)) if r % 2 == 0 else reversed(range(len(libs)))):
        res[libs[i]].append(run(i, 50))
# bit-level agreement of the outputs with the first library
same = [bool(torch.equal(outs[0][0].view(torch.int16), outs[i][0].view(torch.int16)))
        for i in range(len(libs))]
print(json.dumps({"workload": wl, "mode": mode,
                  **{lib: [round(x, 4) for x in v] for lib, v in res.items()},
                  "median": {lib: round(statistics.median(v), 4) for lib, v in res.items()},
                  "o_equal_to_first": same}))
