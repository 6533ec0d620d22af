"""Small product-path calls for compute-sanitizer (memcheck / racecheck /
synccheck): mask, attention, fused call, ASA_GT, backward, Gilbert gather on
tiny and odd N, with refined rows forced.  No oracle: the sanitizer checks
memory and synchronisation, parity is the -m gpu suite's job."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs  # noqa: E402

dev = torch.device("cuda:0")
for (B, H, N, d) in [(1, 1, 1, 64), (1, 1, 512, 64), (1, 2, 129, 128), (1, 3, 700, 128),
                     (2, 2, 1000, 64)]:
    q, k, v = (t.to(dev) for t in inputs.iid(B, H, N, d, seed=N))
    Nb = A.num_blocks(N)
    for guard in (0.0, 1e9):  # default tie guard, then every row through the fp64 refine
        m = A.blade_asa_mask(q, k, tau=0.9, keep_min=1, keep_max=Nb, refine_guard=guard)
        o, lse = A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt)
        of = A.blade_asa_fwd(q, k, v, tau=0.9, keep_min=1, keep_max=Nb, refine_guard=guard)
    og = A.asa_gt_forward(q, k, v, window=128, tau=0.9, keep_min=1, keep_max=Nb)
    do = torch.randn_like(q)
    A.blade_bsa_bwd(q, k, v, o, lse, do, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    print(f"ok B{B} H{H} N{N} d{d}", flush=True)
perm = A.gilbert_order(1, 16, 32).to(dev)
x = torch.randn(1, 512, 64, device=dev).to(torch.bfloat16)
A.blade_permute_tokens(x, perm)
torch.cuda.synchronize()
print("sanitize cases done")
