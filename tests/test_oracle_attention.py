"""Pins of the oracle's block-sparse attention (A9).

The independent reference is torch.nn.functional.scaled_dot_product_attention
in fp64 with the block mask expanded to a boolean token mask, and
torch.logsumexp for the LSE (reading R-10)."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs


def _random_lists(Nb, rng, density=0.4):
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


@pytest.mark.parametrize("N,d,b,seed", [(512, 64, 128, 0), (300, 32, 128, 1), (70, 16, 128, 2),
                                        (1000, 64, 64, 3), (129, 8, 128, 4)])
def test_sparse_attention_equals_sdpa_masked(N, d, b, seed):
    q, k, v = (t[0].double() for t in inputs.iid(1, 1, N, d, seed))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _random_lists(Nb, np.random.default_rng(seed))
    scale = O.default_scale(d)
    Oo, L = O.sparse_attention_unit(q.numpy(), k.numpy(), v.numpy(), kv_idx, kv_cnt, b, scale)
    M = _token_mask(kv_idx, kv_cnt, N, b)
    ref = F.scaled_dot_product_attention(q[None], k[None], v[None], attn_mask=M[None], scale=scale)[0]
    np.testing.assert_allclose(Oo, ref.numpy(), rtol=0, atol=1e-12)
    logits = (q @ k.T) * scale
    logits[~M] = float("-inf")
    np.testing.assert_allclose(L, torch.logsumexp(logits, -1).numpy(), rtol=0, atol=1e-12)


def test_all_ones_mask_is_dense_attention():
    N, d, b = 384, 32, 128
    q, k, v = (t[0].double() for t in inputs.iid(1, 1, N, d, 5))
    Nb = O.num_blocks(N, b)
    kv_idx = np.tile(np.arange(Nb, dtype=np.int32), (Nb, 1))
    kv_cnt = np.full(Nb, Nb, np.int32)
    scale = O.default_scale(d)
    Oo, _ = O.sparse_attention_unit(q.numpy(), k.numpy(), v.numpy(), kv_idx, kv_cnt, b, scale)
    ref = F.scaled_dot_product_attention(q[None], k[None], v[None], scale=scale)[0]
    np.testing.assert_allclose(Oo, ref.numpy(), rtol=0, atol=1e-12)


def test_value_identities():
    N, d, b = 300, 16, 128
    q, k, _ = (t[0].double().numpy() for t in inputs.iid(1, 1, N, d, 6))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _random_lists(Nb, np.random.default_rng(6))
    scale = O.default_scale(d)
    ones = np.ones((N, d))
    Oo, _ = O.sparse_attention_unit(q, k, ones, kv_idx, kv_cnt, b, scale)
    np.testing.assert_allclose(Oo, 1.0, atol=1e-14)                 # V = 1 => O = 1
    Oz, _ = O.sparse_attention_unit(q, k, np.zeros((N, d)), kv_idx, kv_cnt, b, scale)
    assert np.all(Oz == 0)                                           # V = 0 => O = 0


def test_identity_values_read_back_probabilities():
    """N <= d and V = I: O = P, the masked attention probabilities, whose
    rows sum to 1."""
    N, d, b = 96, 96, 32
    q, k, _ = (t[0].double().numpy() for t in inputs.iid(1, 1, N, d, 7))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _random_lists(Nb, np.random.default_rng(7))
    scale = O.default_scale(d)
    Oo, _ = O.sparse_attention_unit(q, k, np.eye(N), kv_idx, kv_cnt, b, scale)
    M = _token_mask(kv_idx, kv_cnt, N, b)
    logits = torch.from_numpy(q @ k.T) * scale
    logits[~M] = float("-inf")
    np.testing.assert_allclose(Oo, torch.softmax(logits, -1).numpy(), atol=1e-14)
    np.testing.assert_allclose(Oo.sum(1), 1.0, atol=1e-13)
    assert np.all(Oo[~M.numpy()] == 0)


def test_single_kept_block_is_restricted_softmax():
    N, d, b = 256, 16, 64
    q, k, v = (t[0].double().numpy() for t in inputs.iid(1, 1, N, d, 8))
    Nb = 4
    kv_idx = np.full((Nb, Nb), -1, np.int32)
    kv_idx[:, 0] = [2, 0, 3, 1]
    kv_cnt = np.ones(Nb, np.int32)
    scale = O.default_scale(d)
    Oo, _ = O.sparse_attention_unit(q, k, v, kv_idx, kv_cnt, b, scale)
    for i in range(Nb):
        j = kv_idx[i, 0]
        S = torch.from_numpy(q[i * b:(i + 1) * b] @ k[j * b:(j + 1) * b].T) * scale
        ref = torch.softmax(S, -1).numpy() @ v[j * b:(j + 1) * b]
        np.testing.assert_allclose(Oo[i * b:(i + 1) * b], ref, atol=1e-13)
