#!/usr/bin/env python
"""Time blade_asa_mask alone (CUDA events, L2 flushed before each call) on a
BASELINE workload in keep-ratio or tau mode; prints one JSON line per config.

    python scripts/mask_time.py [--workload wan|cog] [--steps 20]
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
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--configs", default="keep51,tau0.9,tau0.95,tau0.99")
args = ap.parse_args()
w = inputs.WORKLOADS[args.workload]
q, k, v = (t.cuda() for t in inputs.make(args.workload, "smooth"))
Nb = A.num_blocks(w.N)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for cfg in args.configs.split(","):
    if cfg.startswith("keep"):
        kk = int(cfg[4:])
        kw = dict(tau=0.9, keep_min=kk, keep_max=kk)
    else:
        kw = dict(tau=float(cfg[3:]), keep_min=max(1, -(-5 * Nb // 100)))
    for _ in range(3):
        m = A.blade_asa_mask(q, k, want_mask=False, **kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda._sleep(2_000_000)  # GPU busy while the host enqueues the timed call
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        m = A.blade_asa_mask(q, k, want_mask=False, **kw)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"workload": args.workload, "cfg": cfg, "ms_median": statistics.median(ts),
                      "ms_min": min(ts), "refined": int(m.n_refined.item()),
                      "sparsity": 1 - m.kv_cnt.sum().item() / (m.kv_cnt.numel() * Nb)}),
          flush=True)
