"""Gilbert rearrangement on the GPU (F2; Alg. 1 l.1): the token
gather is bit-exact against numpy fancy indexing with the oracle's
permutation, undo inverts it bit for bit, and ASA on rearranged tokens
matches the oracle run on the oracle-rearranged inputs (masks bit-exact
outside the tie band, O / LSE within tolerance after undoing the order)."""

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


@pytest.mark.parametrize("t,h,w,n_text,d", [(2, 6, 10, 0, 64), (3, 8, 12, 5, 128), (1, 5, 9, 0, 8),
                                            (4, 30, 52, 0, 128), (2, 30, 45, 226, 64)])
def test_permute_bit_exact(A, t, h, w, n_text, d):
    N = n_text + t * h * w
    x = inputs.iid(1, 3, N, d, seed=N)[0]
    perm = O.gilbert_permutation(t, h, w, n_text)
    pd = torch.from_numpy(perm.astype(np.int32)).cuda()
    y = A.blade_permute_tokens(x.cuda(), pd)
    z = A.blade_permute_tokens(y, pd, inverse=True)
    torch.cuda.synchronize()
    want = x.view(torch.int16).numpy()[:, perm]
    assert (y.cpu().view(torch.int16).numpy() == want).all()
    assert torch.equal(z.cpu().view(torch.int16), x.view(torch.int16))


def test_asa_on_gilbert_order_matches_oracle(A):
    t, h, w = 2, 24, 32                      # N = 1536, 12 blocks of 128
    N, d = t * h * w, 64
    q, k, v = inputs.smooth(1, 2, N, d, (t, h, w), ell=3.0, beta=9.0, seed=3)
    perm = A.gilbert_order(t, h, w)
    pd = perm.cuda()
    qd, kd, vd = (A.blade_permute_tokens(x.cuda(), pd) for x in (q, k, v))
    o, lse, m = A.asa_forward(qd, kd, vd, tau=0.9, want_pimp=True)
    o_raster = A.blade_permute_tokens(o, pd, inverse=True)
    torch.cuda.synchronize()
    pn = perm.numpy().astype(np.int64)
    qg, kg, vg = (O.apply_permutation(x.float().numpy(), pn) for x in (q, k, v))
    p = O.AsaParams(tau=0.9)
    ref = O.asa_mask(qg, kg, p)
    PT.check_mask(ref, m, p)
    o_ref, lse_ref = O.sparse_attention(qg, kg, vg, ref.kv_idx, ref.kv_cnt, 128)
    PT.check_attention(o_raster, torch.from_numpy(O.undo_permutation(lse[..., None].cpu().numpy(), pn)[..., 0]),
                       O.undo_permutation(o_ref, pn), O.undo_permutation(lse_ref[..., None], pn)[..., 0])
