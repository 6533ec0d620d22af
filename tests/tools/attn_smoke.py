"""Run one small tcgen05 attention call with a host-side watchdog (debug aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2508_10774_b200 import asa as A, inputs
from oracle import asa_oracle as O

def run(B, H, N, d, density, impl, seed=0):
    q, k, v = inputs.iid(B, H, N, d, seed)
    BH, Nb = B * H, (N + 127) // 128
    rng = np.random.default_rng(seed)
    kv_idx = np.full((BH, Nb, Nb), -1, np.int32); kv_cnt = np.zeros((BH, Nb), np.int32)
    for u in range(BH):
        for i in range(Nb):
            keep = np.flatnonzero(rng.random(Nb) < density)
            if keep.size == 0: keep = np.array([rng.integers(Nb)])
            kv_idx[u, i, :keep.size] = keep; kv_cnt[u, i] = keep.size
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    ki, kc = torch.from_numpy(kv_idx).cuda(), torch.from_numpy(kv_cnt).cuda()
    ev = torch.cuda.Event()
    o, lse = A.blade_bsa_fwd(qd, kd, vd, ki, kc, impl=impl)
    ev.record()
    t0 = time.time()
    while not ev.query():
        if time.time() - t0 > 10:
            print(f"HANG B{B} H{H} N{N} d{d} impl{impl}", flush=True); os._exit(3)
        time.sleep(0.01)
    o_ref, lse_ref = O.sparse_attention(q, k, v, kv_idx, kv_cnt, 128)
    err = np.abs(o.float().cpu().numpy() - o_ref)
    lerr = np.abs(lse.cpu().numpy() - lse_ref)
    print(f"B{B} H{H} N{N} d{d} dens{density} impl{impl}: o_max {err.max():.3e} o_mean {err.mean():.3e} lse_max {lerr.max():.3e}", flush=True)

if __name__ == "__main__":
    impl = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    for case in [(1,1,256,128,1.0), (1,1,512,128,0.5), (1,1,512,64,0.5), (1,2,1000,128,0.4), (1,1,300,64,0.6), (2,2,4096,128,0.3)]:
        run(*case, impl=impl)
