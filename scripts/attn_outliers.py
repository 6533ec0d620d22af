#!/usr/bin/env python
"""Per-call attention times of the two-call path (blade_asa_mask then
blade_bsa_fwd) over many steps, for one or more libraries: min / median /
max, to catch stalls that a mean hides.

    python scripts/attn_outliers.py wan 200 libA.so [libB.so ...]
"""
import importlib.util
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_10774_b200 import inputs  # noqa: E402

wl, steps, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
keep = {"wan": 51, "cog": 25}[wl]
q, k, v = (x.cuda() for x in inputs.make(wl, "smooth"))
st = torch.cuda.current_stream()
for n, lib in enumerate(libs):
    os.environ["BLADE_LIB"] = lib
    spec = importlib.util.spec_from_file_location(
        f"asa_o{n}", os.path.join(ROOT, "paper_2508_10774_b200", "asa.py"))
    A = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(A)
    for fused_first in (True, False):
        if fused_first:
            for _ in range(20):
                A.blade_asa_fwd(q, k, v, tau=0.9, keep_min=keep, keep_max=keep)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b, c in ev:
            a.record(st)
            m = A.blade_asa_mask(q, k, tau=0.9, keep_min=keep, keep_max=keep)
            b.record(st)
            A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt)
            c.record(st)
        torch.cuda.synchronize()
        t = [b.elapsed_time(c) for a, b, c in ev]
        print(json.dumps({"lib": lib, "after_fused": fused_first, "min": min(t),
                          "median": statistics.median(t), "max": max(t),
                          "argmax": t.index(max(t)), "n_over_2x": sum(x > 2 * min(t) for x in t)}),
              flush=True)
