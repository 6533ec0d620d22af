import os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ["BLADE_LIB"] = "libblade_asa_BLADE_ATTN2_TRACE.so"
from paper_2508_10774_b200 import asa as A, inputs
for wl, keep in (("wan", 51), ("cog", 25)):
    q, k, v = (x.cuda() for x in inputs.make(wl, "smooth"))
    m = A.blade_asa_mask(q, k, tau=0.9, keep_min=keep, keep_max=keep)
    for _ in range(10):
        A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    print("done", wl, file=sys.stderr, flush=True)
