"""Quick bounded check of one attention library build (BLADE_LIB) on d=64/128:
AUTO (persistent kernel) vs the pair kernel on the same lists."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2508_10774_b200 import asa as A, inputs
for d in (64, 128):
    q, k, v = inputs.smooth(1, 3, 2000, d, (1, 1, 2000), ell=3.0, beta=9.0, seed=d)
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    m = A.blade_asa_mask(qd, kd, tau=0.9, keep_min=2, keep_max=12)
    o1, l1 = A.blade_bsa_fwd(qd, kd, vd, m.kv_idx, m.kv_cnt, impl=A.ATTN_TCGEN05_PAIR)
    o2, l2 = A.blade_bsa_fwd(qd, kd, vd, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    print(d, "max|dO|", (o1.float() - o2.float()).abs().max().item(), "max|dLSE|", (l1 - l2).abs().max().item(), flush=True)
