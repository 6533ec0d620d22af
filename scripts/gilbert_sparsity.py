#!/usr/bin/env python
"""Natural (tau-mode) block sparsity of the ASA mask with raster vs Gilbert
token order on the smooth-field Wan / CogVideoX inputs (F2; the paper's
Table 4 ablation measures the same effect as a quality score).

    python scripts/gilbert_sparsity.py [--tau 0.9] > gilbert_sparsity.jsonl
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tau", type=float, default=0.9)
    args = ap.parse_args()
    for name in ("wan", "cog"):
        w = inputs.WORKLOADS[name]
        q, k, v = (x.cuda() for x in inputs.make(name, "smooth"))
        BH, N, d = q.shape
        Nb = (N + 127) // 128
        perm = A.gilbert_order(*w.grid, n_text=w.n_text).cuda()
        res = {"workload": w.name, "tau": args.tau}
        for order in ("raster", "gilbert"):
            qq, kk = (q, k) if order == "raster" else (A.blade_permute_tokens(q, perm),
                                                        A.blade_permute_tokens(k, perm))
            m = A.blade_asa_mask(qq, kk, tau=args.tau, keep_min=1, want_mask=False)
            torch.cuda.synchronize()
            res[f"sparsity_{order}"] = round(1.0 - m.kv_cnt.sum().item() / (BH * Nb * Nb), 4)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
