#!/usr/bin/env python
"""Sparsity sweep on the Wan2.1-1.3B layer shape (BASELINE.json configs[3],
SURVEY §8(d)): keep-ratio points from dense to 95% block sparsity and a tau
sweep, each timed on the GPU with CUDA events on the launching stream.

    python scripts/sweep.py [--steps 20] [--recipe smooth|iid] > sweep.jsonl

Per point (one JSON line): sparsity, t_mask / t_attn (ms, median of steps,
L2 flushed before every timed call by writing a 256 MB scratch buffer),
attention TFLOP/s on active blocks and as a fraction of the measured bf16
peak, and the mask kernels' algorithmic HBM bytes / t_mask (sampled Q and K
rows read + kv lists written) next to the measured HBM peak,
plus sampled-probe exponentials per second (N_k^2 per unit).
"""

from __future__ import annotations

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


def active_flop(kv_idx, kv_cnt, N, d, b=128):
    Nb = kv_cnt.shape[1]
    valid = np.array([min(b, N - i * b) for i in range(Nb)], dtype=np.float64)
    tot = 0.0
    for u in range(kv_cnt.shape[0]):
        for i in range(Nb):
            tot += valid[i] * valid[kv_idx[u, i, :kv_cnt[u, i]]].sum()
    return 4.0 * d * tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--recipe", default="smooth", choices=["smooth", "iid"])
    ap.add_argument("--workload", default="wan", choices=["wan", "cog"])
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    w = inputs.WORKLOADS[args.workload]
    q, k, v = (t.cuda() for t in inputs.make(args.workload, args.recipe))
    BH, N, d = q.shape
    Nb = (N + 127) // 128
    kk = 16
    nk = sum(min(kk, min(128, N - i * 128)) for i in range(Nb))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    keeps = [Nb, (3 * Nb) // 4, Nb // 2, Nb // 4, round(0.199 * Nb), round(0.148 * Nb),
             round(0.102 * Nb), round(0.051 * Nb)]
    points = [dict(tau=0.9, keep_min=m, keep_max=m, label=f"keep{m}") for m in keeps]
    points += [dict(tau=t, keep_min=max(1, -(-5 * Nb // 100)), keep_max=Nb, label=f"tau{t}")
               for t in (1.0, 0.99, 0.95, 0.9, 0.8, 0.7, 0.5)]
    for pt in points:
        mp = {x: pt[x] for x in ("tau", "keep_min", "keep_max")}
        m = A.blade_asa_mask(q, k, want_mask=False, **mp)
        A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt)
        torch.cuda.synchronize()
        cnt = m.kv_cnt.cpu().numpy()
        flop = active_flop(m.kv_idx.cpu().numpy(), cnt, N, d)
        tm, ta = [], []
        for _ in range(args.steps):
            flush.fill_(1)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            m = A.blade_asa_mask(q, k, want_mask=False, out=m, **mp)
            e[1].record(stream)
            flush.fill_(2)  # attention also starts from a cold L2
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record(stream)
            A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt)
            e[2].record(stream)
            torch.cuda.synchronize()
            tm.append(e[0].elapsed_time(e[1]))
            ta.append(e2.elapsed_time(e[2]))
        t_mask, t_attn = statistics.median(tm), statistics.median(ta)
        mask_bytes = BH * (2 * nk * d * 2 + Nb * Nb * 4 + Nb * 4)
        tf = flop / (t_attn * 1e-3) / 1e12
        print(json.dumps({
            "workload": w.name, "recipe": args.recipe, "point": pt["label"], "tau": pt["tau"],
            "keep": [pt["keep_min"], pt["keep_max"]],
            "sparsity": round(1.0 - cnt.sum() / (BH * Nb * Nb), 4),
            "ms_mask": t_mask, "ms_attn": t_attn, "attn_tflops": tf,
            "attn_frac_bf16_peak": tf / peaks["bf16_tflops"],
            "mask_gbs_algorithmic": mask_bytes / (t_mask * 1e-3) / 1e9,
            "mask_frac_hbm_peak": mask_bytes / (t_mask * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "probe_exps_per_s": BH * nk * nk / (t_mask * 1e-3),
            "rows_refined_fp64": int(m.n_refined.item()), "l2": "flushed before each call",
        }), flush=True)


if __name__ == "__main__":
    main()
