"""Pins of the oracle's ASA_GT attention (global tokens; readings
R-18..R-20).  Independent references: torch avg_pool1d (the pooling), torch
fp32->bf16 conversion (the rounding, on fp32-representable values), torch
scaled_dot_product_attention (fp64) over the concatenated K_aug / V_aug with
an additive float mask, and a closed form: with K and V constant inside
every pooling window and an all-ones block mask, each global token stands for
its n_w identical fine tokens exactly (the ln n_w bias), so
O_GT = O_dense and LSE_GT = LSE_dense + ln 2."""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs


def test_round_to_bf16_matches_torch_on_fp32_values():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000), rng.standard_normal(2000) * 1e-30,
                        rng.standard_normal(2000) * 1e30]).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(O.round_to_bf16(x.astype(np.float64)), want)


def test_round_to_bf16_single_rounding():
    # 1 + 2^-8 + 2^-30 is just above the half-way point between the bf16
    # values 1 and 1 + 2^-7: one rounding gives 1 + 2^-7; a detour through
    # fp32 (which drops 2^-30) would make it a tie and round to even, 1.0
    x = 1.0 + 2.0 ** -8 + 2.0 ** -30
    assert O.round_to_bf16(np.array([x]))[0] == 1.0 + 2.0 ** -7
    assert O.round_to_bf16(np.array([1.0 + 2.0 ** -8]))[0] == 1.0          # tie -> even
    assert O.round_to_bf16(np.array([1.0 + 3 * 2.0 ** -8]))[0] == 1.0 + 2.0 ** -6
    assert O.round_to_bf16(np.array([0.0, -0.0]))[0] == 0.0


@pytest.mark.parametrize("N,n", [(512, 128), (300, 128), (1000, 32), (77, 7), (5, 8), (64, 1)])
def test_mean_pool_equals_avg_pool1d(N, n):
    x = inputs.iid(1, 1, N, 16, seed=N + n)[0][0].double()
    pooled, counts = O.mean_pool_windows(x.numpy(), n)
    ref = F.avg_pool1d(x.T[None], kernel_size=n, stride=n, ceil_mode=True)[0].T
    np.testing.assert_allclose(pooled, ref.numpy(), rtol=0, atol=1e-15)
    assert counts.sum() == N and (counts[:-1] == n).all() and 1 <= counts[-1] <= n


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


@pytest.mark.parametrize("N,d,b,n,seed", [(512, 32, 128, 128, 0), (300, 16, 128, 128, 1),
                                          (700, 32, 128, 48, 2), (129, 8, 64, 16, 3)])
def test_gt_equals_sdpa_on_augmented_kv(N, d, b, n, seed):
    q, k, v = (t[0].double() for t in inputs.iid(1, 1, N, d, seed))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _random_lists(Nb, np.random.default_rng(seed))
    scale = O.default_scale(d)
    Oo, L = O.sparse_attention_gt_unit(q.numpy(), k.numpy(), v.numpy(), kv_idx, kv_cnt, b,
                                       scale, n)
    # library side: pooled windows by avg_pool1d, bf16 rounding by torch on
    # the (exactly representable) fp32 value of the mean
    kg = F.avg_pool1d(k.T[None], n, n, ceil_mode=True)[0].T
    vg = F.avg_pool1d(v.T[None], n, n, ceil_mode=True)[0].T
    kg = kg.float().to(torch.bfloat16).double()
    vg = vg.float().to(torch.bfloat16).double()
    Ng = kg.shape[0]
    nw = torch.tensor([min(n, N - w * n) for w in range(Ng)], dtype=torch.float64)
    bias = torch.full((N, N + Ng), float("-inf"), dtype=torch.float64)
    for i in range(Nb):
        for j in kv_idx[i, :kv_cnt[i]]:
            bias[i * b:(i + 1) * b, j * b:(j + 1) * b] = 0.0
    bias[:, N:] = torch.log(nw)[None, :]
    K_aug, V_aug = torch.cat([k, kg]), torch.cat([v, vg])
    ref = F.scaled_dot_product_attention(q[None], K_aug[None], V_aug[None], attn_mask=bias[None],
                                         scale=scale)[0]
    # fp32 means vs exact means may round to different bf16 neighbours only
    # at exact ties; iid data never hits one, so the match is to fp64 rounding
    np.testing.assert_allclose(Oo, ref.numpy(), rtol=0, atol=1e-12)
    lse = torch.logsumexp((q @ K_aug.T) * scale + bias, -1)
    np.testing.assert_allclose(L, lse.numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("N,d,b,n", [(512, 16, 128, 128), (300, 16, 128, 128), (500, 8, 128, 32),
                                     (250, 8, 64, 7)])
def test_window_constant_kv_closed_form(N, d, b, n):
    rng = np.random.default_rng(N)
    Ng = (N + n - 1) // n
    # bf16-representable per-window rows, repeated over each window
    kb = O.round_to_bf16(rng.standard_normal((Ng, d)))
    vb = O.round_to_bf16(rng.standard_normal((Ng, d)))
    win = np.arange(N) // n
    k, v = kb[win], vb[win]
    q = O.round_to_bf16(rng.standard_normal((N, d)))
    Nb = O.num_blocks(N, b)
    kv_idx = np.tile(np.arange(Nb, dtype=np.int32), (Nb, 1))
    kv_cnt = np.full(Nb, Nb, np.int32)
    scale = O.default_scale(d)
    Og, Lg = O.sparse_attention_gt_unit(q, k, v, kv_idx, kv_cnt, b, scale, n)
    Od, Ld = O.sparse_attention_unit(q, k, v, kv_idx, kv_cnt, b, scale)
    np.testing.assert_allclose(Og, Od, rtol=0, atol=1e-12)
    np.testing.assert_allclose(Lg, Ld + math.log(2.0), rtol=0, atol=1e-12)


def test_gt_rows_are_convex_combinations():
    N, d, b, n = 384, 16, 128, 64
    q, k, _ = (t[0].double().numpy() for t in inputs.iid(1, 1, N, d, 9))
    Nb = O.num_blocks(N, b)
    kv_idx, kv_cnt = _random_lists(Nb, np.random.default_rng(9), 0.3)
    ones = np.ones((N, d))
    Oo, _ = O.sparse_attention_gt_unit(q, k, ones, kv_idx, kv_cnt, b, O.default_scale(d), n)
    np.testing.assert_allclose(Oo, 1.0, rtol=0, atol=1e-13)          # probabilities sum to 1
    Oz, _ = O.sparse_attention_gt_unit(q, k, np.zeros((N, d)), kv_idx, kv_cnt, b,
                                       O.default_scale(d), n)
    assert np.abs(Oz).max() == 0.0
