"""Multi-rank check of the (batch, head) sharding on the GPU.

Run under torchrun with BLADE_BENCH_SHARE_GPU=1 semantics (every rank on
cuda:0, gloo): each rank draws its GLOBAL units of a small stack with
``inputs.smooth_device`` (per-unit seeds), runs ``blade_asa_fwd`` per layer
with ``unit_offset`` = its first unit, and gathers O, LSE, kv_idx, kv_cnt to
rank 0, which recomputes the whole batch in one process and writes whether
everything matches bit for bit to the JSON path given as argv[1]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_10774_b200 import asa as A  # noqa: E402
from paper_2508_10774_b200 import inputs, shard  # noqa: E402

out_path = sys.argv[1]
units, N, d, layers = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), 2
torch.cuda.set_device(0)
dev = torch.device("cuda:0")
dist.init_process_group("gloo")
ws, rank = dist.get_world_size(), dist.get_rank()
lo, hi = shard.unit_range(ws, rank, units)
grid = (1, 1, N)
kw = dict(tau=0.9, keep_min=1)  # tau mode: LPT order and refined rows active
res = []
for layer in range(layers):
    q, k, v = inputs.smooth_device(range(lo, hi), N, d, grid, dev, seed=42 + layer, beta=9.0)
    o, lse, idx, cnt = A.blade_asa_fwd(q, k, v, unit_offset=lo, seed=42 + layer,
                                       refine_guard=1e-3, **kw)
    torch.cuda.synchronize()
    res.append([shard.gather_units(t, units) for t in (o.float(), lse, idx, cnt)])  # bf16 -> fp32 exact
ok = True
if rank == 0:
    for layer in range(layers):
        q, k, v = inputs.smooth_device(range(units), N, d, grid, dev, seed=42 + layer, beta=9.0)
        o, lse, idx, cnt = A.blade_asa_fwd(q, k, v, seed=42 + layer, refine_guard=1e-3, **kw)
        torch.cuda.synchronize()
        for a, b in zip(res[layer], (o.float(), lse, idx, cnt)):
            ok &= torch.equal(a.cpu(), b.cpu())
    json.dump({"ok": bool(ok), "world": ws, "units": units}, open(out_path, "w"))
dist.destroy_process_group()
