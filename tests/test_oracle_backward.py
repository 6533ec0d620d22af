"""Pins of the oracle's block-sparse attention backward (F3; P:158-161;
reading R-23): torch autograd (fp64) through scaled_dot_product_attention
with the block mask expanded to a token mask (library VJP), central finite
differences of <O, G> on tiny inputs, the dead-path case (a key block no
query keeps gets zero dK, dV) and the all-ones mask == dense attention."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs


def _lists(Nb, rng, density):
    kv_idx = np.full((Nb, Nb), -1, np.int32)
    kv_cnt = np.zeros(Nb, np.int32)
    for i in range(Nb):
        keep = np.flatnonzero(rng.random(Nb) < density)
        if keep.size == 0:
            keep = np.array([int(rng.integers(Nb))])
        kv_idx[i, :keep.size] = keep
        kv_cnt[i] = keep.size
    return kv_idx, kv_cnt


def _token_mask(kv_idx, kv_cnt, N, b):
    M = torch.zeros((N, N), dtype=torch.bool)
    for i in range(len(kv_cnt)):
        for j in kv_idx[i, :kv_cnt[i]]:
            M[i * b:(i + 1) * b, j * b:(j + 1) * b] = True
    return M


@pytest.mark.parametrize("N,d,b,density,seed", [(512, 32, 128, 0.5, 0), (300, 16, 128, 0.6, 1),
                                                (70, 16, 128, 1.0, 2), (1000, 32, 64, 0.3, 3)])
def test_backward_equals_autograd(N, d, b, density, seed):
    q, k, v, g = (inputs.iid(1, 2, N, d, seed)[i][0].double() for i in (0, 1, 2, 0))
    g = torch.from_numpy(np.random.default_rng(seed + 9).standard_normal((N, d)))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _lists(Nb, np.random.default_rng(seed), density)
    scale = O.default_scale(d)
    dq, dk, dv = O.sparse_attention_backward_unit(q.numpy(), k.numpy(), v.numpy(), g.numpy(),
                                                  kv_idx, kv_cnt, b, scale)
    qt, kt, vt = (x.clone().requires_grad_(True) for x in (q, k, v))
    M = _token_mask(kv_idx, kv_cnt, N, b)
    out = F.scaled_dot_product_attention(qt[None], kt[None], vt[None], attn_mask=M[None],
                                         scale=scale)[0]
    out.backward(g)
    for mine, ref in ((dq, qt.grad), (dk, kt.grad), (dv, vt.grad)):
        np.testing.assert_allclose(mine, ref.numpy(), rtol=0, atol=1e-11)


def test_backward_finite_differences():
    N, d, b = 20, 4, 8
    rng = np.random.default_rng(5)
    q, k, v, g = (rng.standard_normal((N, d)) for _ in range(4))
    Nb = O.num_blocks(N, b)
    kv_idx = np.array([[0, 2, -1], [1, -1, -1], [0, 1, 2]], np.int32)
    kv_cnt = np.array([2, 1, 3], np.int32)
    scale = 0.5

    def loss(q_, k_, v_):
        o, _ = O.sparse_attention_unit(q_, k_, v_, kv_idx, kv_cnt, b, scale)
        return float((o * g).sum())

    dq, dk, dv = O.sparse_attention_backward_unit(q, k, v, g, kv_idx, kv_cnt, b, scale)
    eps = 1e-6
    for which, grad in ((0, dq), (1, dk), (2, dv)):
        for (r, c) in [(0, 0), (7, 3), (8, 1), (13, 2), (19, 0)]:
            args = [q.copy(), k.copy(), v.copy()]
            args[which][r, c] += eps
            lp = loss(*args)
            args[which][r, c] -= 2 * eps
            lm = loss(*args)
            assert abs((lp - lm) / (2 * eps) - grad[r, c]) <= 1e-6 * max(1.0, abs(grad[r, c]))


def test_dead_key_block_gets_zero_gradient():
    N, d, b = 384, 16, 128
    q, k, v = (x[0].double().numpy() for x in inputs.iid(1, 1, N, d, 4))
    g = np.random.default_rng(4).standard_normal((N, d))
    kv_idx = np.array([[0, 2, -1], [0, -1, -1], [2, 0, -1]], np.int32)   # block 1 never kept
    kv_cnt = np.array([2, 1, 2], np.int32)
    dq, dk, dv = O.sparse_attention_backward_unit(q, k, v, g, kv_idx, kv_cnt, b, 0.25)
    assert np.abs(dk[128:256]).max() == 0.0 and np.abs(dv[128:256]).max() == 0.0
    assert np.abs(dk[:128]).max() > 0 and np.abs(dq).max() > 0


def test_all_ones_mask_is_dense_backward():
    N, d, b = 256, 16, 128
    q, k, v = (x[0].double() for x in inputs.iid(1, 1, N, d, 6))
    g = torch.from_numpy(np.random.default_rng(6).standard_normal((N, d)))
    kv_idx = np.tile(np.arange(2, dtype=np.int32), (2, 1))
    kv_cnt = np.full(2, 2, np.int32)
    dq, dk, dv = O.sparse_attention_backward_unit(q.numpy(), k.numpy(), v.numpy(), g.numpy(),
                                                  kv_idx, kv_cnt, b, 0.25)
    qt, kt, vt = (x.clone().requires_grad_(True) for x in (q, k, v))
    F.scaled_dot_product_attention(qt[None], kt[None], vt[None], scale=0.25)[0].backward(g)
    np.testing.assert_allclose(dq, qt.grad.numpy(), atol=1e-11, rtol=0)
    np.testing.assert_allclose(dk, kt.grad.numpy(), atol=1e-11, rtol=0)
    np.testing.assert_allclose(dv, vt.grad.numpy(), atol=1e-11, rtol=0)


@pytest.mark.parametrize("N,d,b,n,seed", [(384, 16, 128, 128, 0), (300, 16, 128, 100, 1),
                                          (200, 8, 64, 7, 2)])
def test_gt_backward_equals_autograd(N, d, b, n, seed):
    """ASA_GT gradients vs torch autograd (fp64) through avg_pool1d (ceil
    mode) and SDPA over [K; MeanPool_n(K)] with the ln(n_w) additive mask; the
    oracle's bf16 rounding of the pooled rows is matched by feeding autograd
    the same rounded values with a straight-through estimator."""
    q, k, v = (inputs.iid(1, 1, N, d, seed)[i][0].double() for i in range(3))
    g = torch.from_numpy(np.random.default_rng(seed + 5).standard_normal((N, d)))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _lists(Nb, np.random.default_rng(seed), 0.5)
    scale = O.default_scale(d)
    dq, dk, dv = O.sparse_attention_gt_backward_unit(q.numpy(), k.numpy(), v.numpy(), g.numpy(),
                                                     kv_idx, kv_cnt, b, scale, n)
    qt, kt, vt = (x.clone().requires_grad_(True) for x in (q, k, v))

    def pool_ste(x):  # mean over windows, rounded to bf16 in the forward only
        m = F.avg_pool1d(x.T[None], n, n, ceil_mode=True)[0].T
        r = m.float().to(torch.bfloat16).double()
        return m + (r - m).detach()

    kg, vg = pool_ste(kt), pool_ste(vt)
    Ng = kg.shape[0]
    nw = torch.tensor([min(n, N - w * n) for w in range(Ng)], dtype=torch.float64)
    M = _token_mask(kv_idx, kv_cnt, N, b)
    bias = torch.full((N, N + Ng), float("-inf"), dtype=torch.float64)
    bias[:, :N][M] = 0.0
    bias[:, N:] = torch.log(nw)[None, :]
    out = F.scaled_dot_product_attention(qt[None], torch.cat([kt, kg])[None],
                                         torch.cat([vt, vg])[None], attn_mask=bias[None],
                                         scale=scale)[0]
    out.backward(g)
    for mine, ref in ((dq, qt.grad), (dk, kt.grad), (dv, vt.grad)):
        np.testing.assert_allclose(mine, ref.numpy(), rtol=0, atol=1e-10)
