#!/usr/bin/env python
"""Experiment: split the units of one layer into G groups and run each
group's fused forward (blade_asa_fwd) on its own stream, so one group's mask
kernels overlap another group's attention.  Prints ms per layer for the
single call and for G = 2, 3, 4 (results are identical: the sampler is keyed
by unit_offset)."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "wan"
keep = {"wan": 51, "cog": 25}[wl]
q, k, v = (x.cuda() for x in inputs.make(wl, "smooth"))
BH = q.shape[0]
orig = A._workspace
cur = {"g": 0}
A._workspace = lambda n, dev, tag: orig(n, dev, f"{tag}_{cur['g']}")
main = torch.cuda.current_stream()


def run(G, streams, outs, stagger):
    bounds = [BH * g // G for g in range(G + 1)]
    ev0 = torch.cuda.Event()
    ev0.record(main)
    evs = []
    prev = ev0
    for g in range(G):
        s = streams[g]
        s.wait_event(prev if stagger else ev0)
        cur["g"] = g
        a, b = bounds[g], bounds[g + 1]
        A.blade_asa_fwd(q[a:b], k[a:b], v[a:b], keep_min=keep, keep_max=keep, unit_offset=a,
                        out=outs[g], stream=s)
        e = torch.cuda.Event()
        e.record(s)
        evs.append(e)
        if stagger:  # next group starts after this group's mask (~ its first kernels)
            prev = e
    for e in evs:
        main.wait_event(e)


def timeit(f, steps=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        f()
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


res = {}
full_out = None


def single():
    global full_out
    cur["g"] = 99
    full_out = A.blade_asa_fwd(q, k, v, keep_min=keep, keep_max=keep, out=full_out)


res["single"] = timeit(single)
ref_o = full_out[0].clone()
for G in (2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(G)]
    bounds = [BH * g // G for g in range(G + 1)]
    outs = [None] * G
    for g in range(G):
        a, b = bounds[g], bounds[g + 1]
        outs[g] = (torch.empty_like(q[a:b]), torch.empty((b - a, q.shape[1]), device="cuda"),
                   torch.empty((b - a, full_out[2].shape[1], full_out[2].shape[2]),
                               dtype=torch.int32, device="cuda"),
                   torch.empty((b - a, full_out[3].shape[1]), dtype=torch.int32, device="cuda"))
    res[f"G{G}_concurrent"] = timeit(lambda: run(G, streams, outs, False))
    same = all(torch.equal(outs[g][0], ref_o[bounds[g]:bounds[g + 1]]) for g in range(G))
    res[f"G{G}_same"] = same
print(json.dumps({"workload": wl, **res}))
