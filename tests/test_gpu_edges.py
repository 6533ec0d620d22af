"""Edge cases of the whole path (mask + attention + backward) against the
oracle: the smallest inputs (N = 1, one token; N = 2), a last block of one
row, the maximum block count the GPU path supports (N_b = 512, N = 65536),
k = b (every row sampled), a single kept block per row (lo = hi = 1), the
dense limit (tau = 1), many units (BH = 200) and the unsupported sizes'
error codes."""

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


def _full_check(A, q, k, v, p: O.AsaParams, units=None, qblocks=None):
    qd, kd, vd = PT.to_dev(q, k, v)
    o, lse, m = A.asa_forward(qd, kd, vd, tau=p.tau, keep_min=p.keep_min, keep_max=p.keep_max,
                              samples=p.samples)
    torch.cuda.synchronize()
    ref = O.asa_mask(q, k, p, units=units)
    PT.check_mask(ref, m, p, units=units)
    kv_idx, kv_cnt = m.kv_idx.cpu().numpy(), m.kv_cnt.cpu().numpy()
    for u in (range(q.shape[0]) if units is None else units):
        o_ref, lse_ref = O.sparse_attention_unit(q[u], k[u], v[u], kv_idx[u], kv_cnt[u], 128,
                                                 O.default_scale(q.shape[2]), qblocks)
        PT.check_attention(o[u], lse[u], o_ref, lse_ref)
    return o, lse, m


@pytest.mark.parametrize("N", [1, 2, 127, 128, 129, 257])
@pytest.mark.parametrize("d", [64, 128])
def test_tiny_and_single_row_blocks(A, N, d):
    q, k, v = inputs.iid(1, 2, N, d, seed=N)
    _full_check(A, q, k, v, O.AsaParams(tau=0.9))


def test_max_blocks_65536_tokens(A):
    """N_b = 512 (the GPU limit), one unit, d = 64; masks of every row and the
    attention of sampled query blocks."""
    N = 512 * 128
    q, k, v = inputs.smooth(1, 1, N, 64, (1, 256, 256), ell=3.0, beta=9.0, seed=3)
    _full_check(A, q, k, v, O.AsaParams(tau=0.9), qblocks=[0, 1, 255, 510, 511])


def test_k_equals_b_and_single_kept_block(A):
    q, k, v = inputs.smooth(1, 2, 1000, 128, (1, 1, 1000), ell=3.0, beta=9.0, seed=5)
    _full_check(A, q, k, v, O.AsaParams(tau=0.9, samples=128))
    _full_check(A, q, k, v, O.AsaParams(tau=0.9, keep_min=1, keep_max=1))


def test_tau_one_is_dense(A):
    q, k, v = inputs.smooth(1, 2, 900, 64, (1, 1, 900), ell=3.0, beta=9.0, seed=6)
    o, lse, m = _full_check(A, q, k, v, O.AsaParams(tau=1.0))
    assert (m.kv_cnt.cpu().numpy() == 8).all()


def test_many_units(A):
    q, k, v = inputs.iid(1, 200, 300, 64, seed=9)
    _full_check(A, q, k, v, O.AsaParams(tau=0.85), units=[0, 77, 199], qblocks=[0, 2])


def test_backward_single_token_and_ragged(A):
    for N in (1, 129):
        q, k, v = inputs.iid(1, 1, N, 64, seed=N)
        do = inputs.iid(1, 1, N, 64, seed=N + 1)[0]
        qd, kd, vd, dod = PT.to_dev(q, k, v, do)
        o, lse, m = A.asa_forward(qd, kd, vd, tau=0.9)
        dq, dk, dv = A.blade_bsa_bwd(qd, kd, vd, o, lse, dod, m.kv_idx, m.kv_cnt)
        torch.cuda.synchronize()
        rq, rk, rv = O.sparse_attention_backward(q, k, v, do, m.kv_idx.cpu().numpy(),
                                                 m.kv_cnt.cpu().numpy(), 128)
        for got, ref in ((dq, rq), (dk, rk), (dv, rv)):
            g = got.float().cpu().numpy()
            scale = max(np.abs(ref).max(), 1e-6)
            assert np.abs(g - ref).max() <= 2e-2 * scale


def test_unsupported_sizes_raise(A):
    q = torch.zeros((1, 513 * 128, 64), dtype=torch.bfloat16, device="cuda")   # N_b = 513
    with pytest.raises(A.BladeError) as e:
        A.blade_asa_mask(q, q)
    assert e.value.status == A.BLADE_ERR_UNSUPPORTED
    q = torch.zeros((1, 256, 96), dtype=torch.bfloat16, device="cuda")           # d = 96
    with pytest.raises(A.BladeError) as e:
        A.blade_asa_mask(q, q)
    assert e.value.status == A.BLADE_ERR_UNSUPPORTED
