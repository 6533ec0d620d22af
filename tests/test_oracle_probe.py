"""Pins of the oracle's probe (A3-A6)."""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs


def torch_probe(q, k, s, Nb, b, kk, scale):
    """Library recomputation of A4-A6: the sampled logits laid out on an
    Nb*kk grid (missing samples of ragged tail blocks are masked), softmax
    over the valid sampled keys (torch.softmax), then kk x kk max-pooling
    (torch max_pool2d)."""
    qt = torch.from_numpy(np.asarray(q, np.float64))
    kt = torch.from_numpy(np.asarray(k, np.float64))
    Qs = torch.zeros((Nb * kk, q.shape[1]), dtype=torch.float64)
    Ks = torch.zeros((Nb * kk, q.shape[1]), dtype=torch.float64)
    qv = torch.zeros(Nb * kk, dtype=torch.bool)
    kv = torch.zeros(Nb * kk, dtype=torch.bool)
    for i in range(Nb):
        for r, o in enumerate(s.offsets_q[i]):
            Qs[i * kk + r] = qt[i * b + o]
            qv[i * kk + r] = True
        for r, o in enumerate(s.offsets_k[i]):
            Ks[i * kk + r] = kt[i * b + o]
            kv[i * kk + r] = True
    L = torch.matmul(Qs, Ks.T) * scale
    L[:, ~kv] = float("-inf")
    P = torch.softmax(L, dim=-1)
    P[~qv] = float("-inf")
    P[:, ~kv] = float("-inf")
    return F.max_pool2d(P[None, None], kernel_size=kk, stride=kk)[0, 0].numpy()


@pytest.mark.parametrize("N,d,b,k,seed", [(512, 64, 128, 16, 1), (300, 32, 128, 16, 2),
                                          (70, 16, 128, 16, 3), (1000, 64, 64, 8, 4),
                                          (256, 16, 32, 32, 5), (130, 8, 128, 16, 6)])
def test_probe_equals_library_softmax_maxpool(N, d, b, k, seed):
    q, kk_, _ = (t[0].float().numpy() for t in inputs.iid(1, 1, N, d, seed))
    p = O.AsaParams(block=b, samples=k, seed=seed)
    Nb = O.num_blocks(N, b)
    s = O.draw_samples(N, p, 0)
    scale = O.default_scale(d)
    got = O.probe_pimp(q, kk_, s, Nb, scale)
    ref = torch_probe(q, kk_, s, Nb, b, k, scale)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)


@pytest.mark.parametrize("N,d,b,seed", [(512, 32, 128, 1), (200, 16, 64, 2), (96, 8, 32, 3)])
def test_exhaustive_probe_equals_dense_importance(N, d, b, seed):
    """k = b: the probe samples every token, so P_imp is the conceptual full
    importance of P:117 (dense softmax, then b x b max-pool) — checked
    against torch.softmax + max_pool2d(ceil_mode) on the full logits."""
    q, k, _ = (t[0].float().numpy() for t in inputs.iid(1, 1, N, d, seed))
    scale = O.default_scale(d)
    p = O.AsaParams(block=b, samples=b, seed=seed)
    Nb = O.num_blocks(N, b)
    s = O.draw_samples(N, p, 0)
    probe = O.probe_pimp(q, k, s, Nb, scale)
    Pfull = torch.softmax(torch.from_numpy(q.astype(np.float64) @ k.astype(np.float64).T) * scale, -1)
    ref = F.max_pool2d(Pfull[None, None], kernel_size=b, stride=b, ceil_mode=True)[0, 0].numpy()
    np.testing.assert_allclose(probe, ref, rtol=1e-12, atol=0)
    np.testing.assert_allclose(O.dense_importance_map(q, k, b, scale), ref, rtol=1e-12, atol=0)
    # and the masks agree exactly (SPEC S:643 acceptance criterion)
    for i in range(Nb):
        assert O.select_row(probe[i], 0.9, 1, Nb).kept == O.select_row(ref[i], 0.9, 1, Nb).kept


def test_uniform_logits_theorem1_factor():
    """Theorem 1 exact case: constant logits => every sampled entry is
    1/N_k, every full entry is 1/N, ratio b/k = 8 at b=128, k=16."""
    N, d, b, k = 1024, 16, 128, 16
    q = np.zeros((N, d))
    kk = np.random.default_rng(0).standard_normal((N, d))
    scale = O.default_scale(d)
    p = O.AsaParams(block=b, samples=k)
    s = O.draw_samples(N, p, 0)
    Nb = N // b
    sparse = O.probe_pimp(q, kk, s, Nb, scale)
    full = O.dense_importance_map(q, kk, b, scale)
    assert np.all(sparse == 1.0 / (Nb * k))
    np.testing.assert_allclose(full, 1.0 / N, rtol=1e-15)
    np.testing.assert_allclose(sparse / full, b / k, rtol=1e-12)
    # normalised maps, hence masks, are identical (Appendix B §5)
    for i in range(Nb):
        assert O.select_row(sparse[i], 0.5, 1, Nb).kept == O.select_row(full[i], 0.5, 1, Nb).kept


@pytest.mark.parametrize("N,d,b,k,seed", [(512, 64, 128, 16, 1), (300, 32, 128, 16, 2),
                                          (777, 16, 64, 8, 3)])
def test_streaming_alg3_equals_two_pass(N, d, b, k, seed):
    """Alg. 3 (running M, l, stashed R) == softmax-then-maxpool."""
    q, kk, _ = (t[0].float().numpy() for t in inputs.smooth(1, 1, N, d, (1, 1, N), seed=seed))
    p = O.AsaParams(block=b, samples=k, seed=seed)
    Nb = O.num_blocks(N, b)
    s = O.draw_samples(N, p, 0)
    scale = O.default_scale(d)
    np.testing.assert_allclose(O.probe_pimp_streaming(q, kk, s, Nb, scale),
                               O.probe_pimp(q, kk, s, Nb, scale), rtol=1e-12, atol=1e-300)


def test_single_block_is_max_of_softmax_row():
    """N_b = 1: the only entry is the max of a row-stochastic matrix."""
    q, k, _ = (t[0].float().numpy() for t in inputs.iid(1, 1, 100, 16, 9))
    p = O.AsaParams(block=128, samples=16, seed=9)
    s = O.draw_samples(100, p, 0)
    scale = O.default_scale(16)
    L = torch.from_numpy(q[s.rows_q].astype(np.float64) @ k[s.rows_k].astype(np.float64).T) * scale
    assert abs(O.probe_pimp(q, k, s, 1, scale)[0, 0] - torch.softmax(L, -1).max().item()) < 1e-15
