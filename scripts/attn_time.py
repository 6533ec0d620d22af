#!/usr/bin/env python
"""Attention-only timing of one library build (BLADE_LIB) on the bench
workloads: the keep-ratio lists are computed once, then blade_bsa_fwd runs
back to back behind a GPU sleep (so host enqueue stalls cannot open gaps);
prints the per-call ms of several blocks and the median.

    BLADE_LIB=libblade_asa_X.so python scripts/attn_time.py [--workload wan|cog] [--calls 50]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan")
ap.add_argument("--calls", type=int, default=50)
ap.add_argument("--blocks", type=int, default=5)
ap.add_argument("--tau", type=float, default=None)
ap.add_argument("--fused", action="store_true", help="time blade_asa_fwd instead")
args = ap.parse_args()

keep = {"wan": 51, "cog": 25}[args.workload]
q, k, v = (x.cuda() for x in inputs.make(args.workload, "smooth"))
kw = dict(tau=args.tau) if args.tau else dict(tau=0.9, keep_min=keep, keep_max=keep)
m = A.blade_asa_mask(q, k, want_mask=False, **kw)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
fo = [None]


def call():
    if args.fused:
        fo[0] = A.blade_asa_fwd(q, k, v, out=fo[0], **kw)
    else:
        A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt)


for _ in range(5):
    call()
torch.cuda.synchronize()
res = []
for _ in range(args.blocks):
    torch.cuda._sleep(20_000_000)  # ~10 ms of GPU spin while the host enqueues
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.calls):
        call()
    e1.record(st)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / args.calls)
cnt = m.kv_cnt.cpu().numpy()
print(json.dumps({"lib": os.environ.get("BLADE_LIB", "libblade_asa.so"), "workload": args.workload,
                  "fused": args.fused, "ms": [round(x, 4) for x in res],
                  "median": round(statistics.median(res), 4), "kept": int(cnt.sum())}))
