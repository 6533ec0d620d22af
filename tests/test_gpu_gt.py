"""ASA_GT (global tokens) CUDA path vs the fp64 oracle through the C ABI.

Pooling: the bf16 window means equal the oracle's (exact mean rounded once to
bf16, reading R-19) except where fp32 summation lands on the other side of a
bf16 rounding tie: at most one bf16 ulp, on a tiny fraction of entries.
Attention (given a mask): O max abs <= 2e-2, mean abs <= 2e-3, LSE <= 1e-3
(BASELINE.json tolerances), small ragged cases and the full Wan layer on
sampled query blocks in the launch configuration of the bench."""

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


def _bf16_ulp(x):
    m, e = np.frexp(np.abs(x))
    return np.ldexp(1.0, e - 8)


@pytest.mark.parametrize("N,d,n", [(512, 64, 128), (1000, 128, 128), (300, 64, 100),
                                   (777, 128, 7), (70, 64, 128), (4096, 128, 1000), (33, 64, 1)])
def test_pool_parity(A, N, d, n):
    _, k, v = inputs.smooth(1, 3, N, d, (1, 1, N), ell=3.0, beta=9.0, seed=N)
    kg, vg = A.blade_gt_pool(k.cuda(), v.cuda(), window=n)
    torch.cuda.synchronize()
    for u in range(3):
        kr, vr, bias = O.global_tokens(k[u], v[u], n)
        for got, ref in ((kg[u], kr), (vg[u], vr)):
            g = got.double().cpu().numpy()
            diff = np.abs(g - ref)
            assert (diff <= _bf16_ulp(ref) + 1e-300).all()
            assert (diff == 0).mean() >= 0.99


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


GT_CASES = [  # (BH, N, d, window, density)
    (1, 512, 64, 128, 0.5), (2, 1000, 128, 128, 0.3), (2, 300, 64, 128, 0.6),
    (1, 70, 128, 128, 1.0), (1, 2000, 64, 64, 0.2), (2, 1500, 128, 100, 0.25),
    (1, 640, 64, 5, 0.4),     # N_g = 128: exactly one full global tile
    (1, 1300, 128, 7, 0.3),   # N_g = 186: two global tiles, ragged
    (1, 4000, 128, 4000, 0.1),  # one global token
]


@pytest.mark.parametrize("impl", [1, 3], ids=["tcgen05", "pair"])
@pytest.mark.parametrize("case", GT_CASES, ids=lambda c: "x".join(map(str, c)))
def test_gt_attention_parity_given_mask(A, case, impl):
    BH, N, d, n, density = case
    q, k, v = inputs.iid(1, BH, N, d, seed=N + d + n)
    Nb = O.num_blocks(N, 128)
    kv_idx, kv_cnt = _lists(BH, Nb, np.random.default_rng(N + n), density)
    o_ref, lse_ref = O.sparse_attention_gt(q, k, v, kv_idx, kv_cnt, 128, n)
    qd, kd, vd = PT.to_dev(q, k, v)
    ki, kc = PT.lists_to_dev(kv_idx, kv_cnt)
    kg, vg = A.blade_gt_pool(kd, vd, window=n)
    o, lse = A.blade_bsa_gt_fwd(qd, kd, vd, ki, kc, kg, vg, window=n, impl=impl)
    torch.cuda.synchronize()
    PT.check_attention(o, lse, o_ref, lse_ref)


def test_gt_smooth_end_to_end_and_ones(A):
    q, k, v = inputs.smooth(1, 2, 1500, 128, (1, 1, 1500), ell=3.0, beta=9.0, seed=4)
    qd, kd, vd = PT.to_dev(q, k, v)
    o, lse, m = A.asa_gt_forward(qd, kd, vd, window=128, tau=0.9)
    torch.cuda.synchronize()
    p = O.AsaParams(tau=0.9)
    PT.check_mask(O.asa_mask(q, k, p), m, p)   # global tokens do not change the mask (R-20)
    o_ref, lse_ref = O.sparse_attention_gt(q, k, v, m.kv_idx.cpu().numpy(),
                                           m.kv_cnt.cpu().numpy(), 128, 128)
    PT.check_attention(o, lse, o_ref, lse_ref)
    ones = torch.ones_like(vd)
    o1, _, _ = A.asa_gt_forward(qd, kd, ones, window=128, tau=0.9)
    torch.cuda.synchronize()
    assert (o1.float() - 1).abs().max().item() <= 4e-3    # probabilities sum to 1


def test_gt_mma_impl_is_unsupported(A):
    q, k, v = inputs.iid(1, 1, 256, 64, seed=1)
    qd, kd, vd = PT.to_dev(q, k, v)
    kg, vg = A.blade_gt_pool(kd, vd, window=128)
    kv_idx = torch.tensor([[[0, 1], [0, 1]]], dtype=torch.int32, device="cuda")
    kv_cnt = torch.tensor([[2, 2]], dtype=torch.int32, device="cuda")
    with pytest.raises(A.BladeError) as e:
        A.blade_bsa_gt_fwd(qd, kd, vd, kv_idx, kv_cnt, kg, vg, window=128, impl=A.ATTN_MMA_SYNC)
    assert e.value.status == A.BLADE_ERR_UNSUPPORTED


def test_gt_fullsize_wan_sampled(A):
    """Wan layer, keep 51/256, n = 128 (256 global tokens), sampled query blocks."""
    q, k, v = inputs.make("wan", "smooth")
    BH, N, d = q.shape
    qd, kd, vd = PT.to_dev(q, k, v)
    o, lse, m = A.asa_gt_forward(qd, kd, vd, window=128, tau=0.9, keep_min=51, keep_max=51)
    torch.cuda.synchronize()
    kv_idx, kv_cnt = m.kv_idx.cpu().numpy(), m.kv_cnt.cpu().numpy()
    Nb = O.num_blocks(N, 128)
    for u in (0, BH - 1):
        # the oracle's per-unit function with a subset of query blocks
        o_ref, lse_ref = O.sparse_attention_gt_unit(q[u], k[u], v[u], kv_idx[u], kv_cnt[u], 128,
                                                    O.default_scale(d), 128,
                                                    qblocks=[0, Nb // 2, Nb - 1])
        PT.check_attention(o[u], lse[u], o_ref, lse_ref)
