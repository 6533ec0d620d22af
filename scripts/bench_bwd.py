#!/usr/bin/env python
"""Time the block-sparse attention backward (F3) on the Wan / Cog layer with
the bench's mask; algorithmic FLOP = 2.5 x the forward's active FLOP (the five
GEMM-shaped products S, dP, dV, dK, dQ per kept (query, key) pair).

    python scripts/bench_bwd.py [--workload wan|cog] [--variant asa|asa_gt] [--steps 20]

asa_gt adds the global tokens (window 128): their FLOP, 10 d per (query,
global token) pair, are counted in the algorithmic FLOP.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="wan", choices=["wan", "cog"])
    ap.add_argument("--variant", default="asa", choices=["asa", "asa_gt"])
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    keep = {"wan": 51, "cog": 25}[args.workload]
    q, k, v = (x.cuda() for x in inputs.make(args.workload, "smooth"))
    do = torch.randn_like(q)
    BH, N, d = q.shape
    gt = args.variant == "asa_gt"
    if gt:
        o, lse, m = A.asa_gt_forward(q, k, v, window=128, tau=0.9, keep_min=keep, keep_max=keep)
        kg, vg = A.blade_gt_pool(k, v, window=128)

        def run():
            A.blade_bsa_gt_bwd(q, k, v, kg, vg, o, lse, do, m.kv_idx, m.kv_cnt, window=128)
    else:
        o, lse, m = A.asa_forward(q, k, v, tau=0.9, keep_min=keep, keep_max=keep)

        def run():
            A.blade_bsa_bwd(q, k, v, o, lse, do, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    Nb = (N + 127) // 128
    valid = np.array([min(128, N - i * 128) for i in range(Nb)], dtype=np.float64)
    idx, cnt = m.kv_idx.cpu().numpy(), m.kv_cnt.cpu().numpy()
    pairs = sum(valid[i] * valid[idx[u, i, :cnt[u, i]]].sum() for u in range(BH) for i in range(Nb))
    if gt:
        pairs += BH * N * A.num_global_tokens(N, 128)
    flop = 10.0 * d * pairs
    for _ in range(3):
        run()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    print(json.dumps({"workload": args.workload, "variant": args.variant, "keep": keep, "ms_bwd": ms,
                      "tflops": flop / (ms * 1e-3) / 1e12,
                      "frac_bf16_peak": flop / (ms * 1e-3) / 1e12 / peak,
                      "kernels": "tcgen05: bwd_dkdv_tc_kernel (transposed lists) + bwd_dq_tc_kernel; D_r and list transpose on CUDA cores"}))


if __name__ == "__main__":
    main()
