"""Block-sparse attention backward (F3; reading R-23) on the GPU vs
the fp64 oracle.  The GPU rounds P and dS to bf16 for their MMAs and reads
the bf16 forward output O for D_r = dO.O; each gradient entry sums up to
N_kept products whose terms carry ~2^-9 relative rounding, so the test bounds
the error relative to the gradient's scale: max |err| <= 2e-2 max|ref| and
mean |err| <= 2e-3 max|ref| for each of dQ, dK, dV (the same 2e-2 / 2e-3
factors as BASELINE.json's forward O tolerance, applied to the scale of the
quantity); key rows no query keeps are exactly zero."""

import numpy as np
import pytest
import torch

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs

from . import _parity as PT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A(cuda_dev):
    from paper_2508_10774_b200 import asa
    return asa


def _lists(BH, Nb, rng, density):
    kv_idx = np.full((BH, Nb, Nb), -1, np.int32)
    kv_cnt = np.zeros((BH, Nb), np.int32)
    for u in range(BH):
        for i in range(Nb):
            keep = np.flatnonzero(rng.random(Nb) < density)
            if keep.size == 0:
                keep = np.array([rng.integers(Nb)])
            kv_idx[u, i, :keep.size] = keep
            kv_cnt[u, i] = keep.size
    return kv_idx, kv_cnt


def _check(got, ref, name):
    g = got.float().cpu().numpy().astype(np.float64)
    scale = np.abs(ref).max()
    err = np.abs(g - ref)
    assert np.isfinite(g).all(), name
    assert err.max() <= 2e-2 * scale, (name, err.max(), scale)
    assert err.mean() <= 2e-3 * scale, (name, err.mean(), scale)
    return err.max() / scale


CASES = [(1, 512, 64, 0.5), (2, 300, 128, 0.6), (1, 70, 64, 1.0), (2, 1000, 128, 0.3),
         (1, 129, 128, 0.7), (1, 2048, 64, 0.2)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_backward_parity_given_mask(A, case):
    BH, N, d, density = case
    q, k, v = inputs.iid(1, BH, N, d, seed=N + d)
    do = inputs.iid(1, BH, N, d, seed=N + d + 1)[0]
    Nb = O.num_blocks(N, 128)
    kv_idx, kv_cnt = _lists(BH, Nb, np.random.default_rng(N), density)
    qd, kd, vd, dod = PT.to_dev(q, k, v, do)
    ki, kc = PT.lists_to_dev(kv_idx, kv_cnt)
    o, lse = A.blade_bsa_fwd(qd, kd, vd, ki, kc)
    dq, dk, dv = A.blade_bsa_bwd(qd, kd, vd, o, lse, dod, ki, kc)
    torch.cuda.synchronize()
    rq, rk, rv = O.sparse_attention_backward(q, k, v, do, kv_idx, kv_cnt, 128)
    for got, ref, nm in ((dq, rq, "dq"), (dk, rk, "dk"), (dv, rv, "dv")):
        _check(got, ref, nm)
    # key blocks no query keeps: exactly zero gradient
    for u in range(BH):
        kept = set(kv_idx[u][kv_idx[u] >= 0].tolist())
        for j in range(Nb):
            if j not in kept:
                assert dk[u, j * 128:(j + 1) * 128].abs().max().item() == 0.0
                assert dv[u, j * 128:(j + 1) * 128].abs().max().item() == 0.0


def test_backward_on_asa_mask_smooth(A):
    q, k, v = inputs.smooth(1, 2, 1500, 128, (1, 1, 1500), ell=3.0, beta=9.0, seed=2)
    do = inputs.iid(1, 2, 1500, 128, seed=7)[0]
    qd, kd, vd, dod = PT.to_dev(q, k, v, do)
    o, lse, m = A.asa_forward(qd, kd, vd, tau=0.9)
    dq, dk, dv = A.blade_bsa_bwd(qd, kd, vd, o, lse, dod, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    rq, rk, rv = O.sparse_attention_backward(q, k, v, do, m.kv_idx.cpu().numpy(),
                                             m.kv_cnt.cpu().numpy(), 128)
    for got, ref, nm in ((dq, rq, "dq"), (dk, rk, "dk"), (dv, rv, "dv")):
        _check(got, ref, nm)


def test_backward_deterministic(A):
    q, k, v = inputs.iid(1, 2, 700, 64, seed=1)
    do = inputs.iid(1, 2, 700, 64, seed=2)[0]
    qd, kd, vd, dod = PT.to_dev(q, k, v, do)
    o, lse, m = A.asa_forward(qd, kd, vd, tau=0.8)
    g1 = A.blade_bsa_bwd(qd, kd, vd, o, lse, dod, m.kv_idx, m.kv_cnt)
    g2 = A.blade_bsa_bwd(qd, kd, vd, o, lse, dod, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    for a, b in zip(g1, g2):
        assert torch.equal(a, b)


GT_CASES = [(1, 512, 64, 0.5, 128), (2, 300, 128, 0.6, 100), (1, 1000, 128, 0.3, 7),
            (2, 129, 64, 1.0, 128), (1, 2048, 128, 0.2, 128), (1, 70, 64, 1.0, 1000)]


@pytest.mark.parametrize("case", GT_CASES, ids=lambda c: "x".join(map(str, c)))
def test_gt_backward_parity_given_mask(A, case):
    """ASA_GT backward (F1 + F3) vs the oracle, same bounds as above; window
    sizes span full, ragged, tiny (n = 7: N_g = 143 spans three 64-row tiles)
    and larger than N (one global token)."""
    BH, N, d, density, n = case
    q, k, v = inputs.iid(1, BH, N, d, seed=N + d + 3)
    do = inputs.iid(1, BH, N, d, seed=N + d + 4)[0]
    Nb = O.num_blocks(N, 128)
    kv_idx, kv_cnt = _lists(BH, Nb, np.random.default_rng(N + 1), density)
    qd, kd, vd, dod = PT.to_dev(q, k, v, do)
    ki, kc = PT.lists_to_dev(kv_idx, kv_cnt)
    kg, vg = A.blade_gt_pool(kd, vd, window=n)
    o, lse = A.blade_bsa_gt_fwd(qd, kd, vd, ki, kc, kg, vg, window=n)
    dq, dk, dv = A.blade_bsa_gt_bwd(qd, kd, vd, kg, vg, o, lse, dod, ki, kc, window=n)
    g2 = A.blade_bsa_gt_bwd(qd, kd, vd, kg, vg, o, lse, dod, ki, kc, window=n)
    torch.cuda.synchronize()
    for a, b in zip((dq, dk, dv), g2):
        assert torch.equal(a, b)  # deterministic
    rq, rk, rv = O.sparse_attention_gt_backward(q, k, v, do, kv_idx, kv_cnt, 128, n)
    for got, ref, nm in ((dq, rq, "dq"), (dk, rk, "dk"), (dv, rv, "dv")):
        _check(got, ref, nm)


def test_gt_backward_smooth_end_to_end(A):
    q, k, v = inputs.smooth(1, 2, 1500, 128, (1, 1, 1500), ell=3.0, beta=9.0, seed=3)
    do = inputs.iid(1, 2, 1500, 128, seed=8)[0]
    qd, kd, vd, dod = PT.to_dev(q, k, v, do)
    o, lse, m = A.asa_gt_forward(qd, kd, vd, window=128, tau=0.9)
    kg, vg = A.blade_gt_pool(kd, vd, window=128)
    dq, dk, dv = A.blade_bsa_gt_bwd(qd, kd, vd, kg, vg, o, lse, dod, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    rq, rk, rv = O.sparse_attention_gt_backward(q, k, v, do, m.kv_idx.cpu().numpy(),
                                                m.kv_cnt.cpu().numpy(), 128, 128)
    for got, ref, nm in ((dq, rq, "dq"), (dk, rk, "dk"), (dv, rv, "dv")):
        _check(got, ref, nm)


@pytest.mark.parametrize("variant", ["asa", "asa_gt"])
def test_backward_fullsize_wan_unit(A, variant):
    """BASELINE.json configs[1] (Wan2.1-1.3B layer, 12 x 32760 x 128), keep
    51/256 as bench.py times it, the bench's launch configuration (all 12
    units in one call); the oracle recomputes unit 0's dQ, dK, dV in full
    (every row of the unit, 256 query blocks x 6528 kept keys)."""
    q, k, v = inputs.make("wan", "smooth")
    do = inputs.iid(1, q.shape[0], q.shape[1], q.shape[2], seed=11)[0]
    qd, kd, vd, dod = PT.to_dev(q, k, v, do)
    if variant == "asa":
        o, lse, m = A.asa_forward(qd, kd, vd, tau=0.9, keep_min=51, keep_max=51)
        dq, dk, dv = A.blade_bsa_bwd(qd, kd, vd, o, lse, dod, m.kv_idx, m.kv_cnt)
    else:
        o, lse, m = A.asa_gt_forward(qd, kd, vd, window=128, tau=0.9, keep_min=51, keep_max=51)
        kg, vg = A.blade_gt_pool(kd, vd, window=128)
        dq, dk, dv = A.blade_bsa_gt_bwd(qd, kd, vd, kg, vg, o, lse, dod, m.kv_idx, m.kv_cnt)
    torch.cuda.synchronize()
    kv_idx, kv_cnt = m.kv_idx.cpu().numpy(), m.kv_cnt.cpu().numpy()
    scale = O.default_scale(q.shape[2])
    if variant == "asa":
        refs = O.sparse_attention_backward_unit(q[0], k[0], v[0], do[0], kv_idx[0], kv_cnt[0],
                                                128, scale)
    else:
        refs = O.sparse_attention_gt_backward_unit(q[0], k[0], v[0], do[0], kv_idx[0],
                                                   kv_cnt[0], 128, scale, 128)
    for got, ref, nm in zip((dq, dk, dv), refs, ("dq", "dk", "dv")):
        _check(got[0], ref, nm)
