"""Measure the fp32 probe error vs the fp64 oracle and the refine-queue size
per guard value (sets the default refine_guard; R-14)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2508_10774_b200 import asa as A, inputs
from oracle import asa_oracle as O

for wl, kw in (("wan", dict(tau=0.9, keep_min=51, keep_max=51)), ("wan", dict(tau=0.9, keep_min=13)),
               ("cog", dict(tau=0.95, keep_min=7))):
    q, k, v = inputs.make(wl, "smooth")
    BH = q.shape[0]
    units = list(range(min(BH, 6)))
    ref = O.asa_mask(q, k, O.AsaParams(**kw), units=units)
    qd, kd = q.cuda(), k.cuda()
    # guard tiny -> no refinement: raw fp32 decisions and raw fp32 P_imp
    m = A.blade_asa_mask(qd, kd, want_pimp=True, refine_guard=1e-30, **kw)
    torch.cuda.synchronize()
    g = m.p_imp.cpu().numpy().astype(np.float64)[units]
    r = ref.p_imp[units]
    rel = np.abs(g - r) / r
    print(wl, kw, "P_imp rel err: max %.3e  p99.9 %.3e  mean %.3e" % (rel.max(), np.quantile(rel, 0.999), rel.mean()))
    # margins of the oracle rows
    lo, hi = O.clamp_bounds(ref.p_imp.shape[1], O.AsaParams(**kw))
    for guard in (2e-5, 1e-5, 5e-6, 3e-6, 2e-6):
        mg = A.blade_asa_mask(qd, kd, refine_guard=guard, **kw)
        torch.cuda.synchronize()
        print("   guard %.0e -> rows refined %d of %d" % (guard, int(mg.n_refined.item()), BH * ref.p_imp.shape[1]))
    # mismatches of the unrefined fp32 decisions (outside tie band)
    bad = 0
    kv = m.kv_idx.cpu().numpy(); kc = m.kv_cnt.cpu().numpy()
    for u in units:
        for i in range(ref.p_imp.shape[1]):
            if O.check_row_against(ref.rows[u][i], float(np.float32(kw['tau'])), lo, hi, kv[u, i, :kc[u, i]].tolist()) is not None:
                bad += 1
    print("   unrefined fp32 rows outside tie band:", bad)
