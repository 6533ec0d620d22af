"""Pins of the oracle's sampler (A2; reading R-1)."""

import json
import math
import os

import numpy as np
import pytest

from oracle import asa_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sampler_kat.json")))


def test_splitmix64_public_sequence():
    # splitmix64 seeded with 0: state advances by G, output = fmix64(state)
    assert [format(O.sm(0, n), "016x") for n in range(2)] == GOLD["splitmix64_seed0"]
    assert format(O.fmix64(1), "016x") == GOLD["fmix64_1"]


def test_survey_known_answers():
    assert format(O.sample_key(42, 0, 0, 0), "016x") == GOLD["key_42_0_0_0"]
    for c in GOLD["samples"]:
        got = O.sample_offsets(c["seed"], c["u"], c["blk"], c["which"], c["valid"], c["k"])
        assert got == c["offsets"], c


@pytest.mark.parametrize("valid,k", [(128, 16), (120, 16), (5, 16), (128, 128), (1, 1), (17, 16)])
def test_subset_properties(valid, k):
    for u in range(5):
        off = O.sample_offsets(7, u, 3, 1, valid, k)
        assert len(off) == min(k, valid)
        assert off == sorted(set(off))
        assert all(0 <= o < valid for o in off)
    if k >= valid:   # exhaustive sample = the block itself in index order
        assert O.sample_offsets(7, 0, 0, 0, valid, k) == list(range(valid))


def test_chi_square_uniformity():
    """Offset counts over 200 units x 64 blocks (seed 7): chi^2 on 127 dof.
    SURVEY App. A quotes 126.5; accept anything below the 1e-6 upper tail."""
    counts = np.zeros(128)
    for u in range(200):
        for i in range(64):
            for o in O.sample_offsets(7, u, i, 0, 128, 16):
                counts[o] += 1
    expected = counts.sum() / 128
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    assert abs(chi2 - GOLD["chi2_seed7_200units_64blocks"]) < 0.05
    assert chi2 < 127 + 5 * math.sqrt(2 * 127)


def _rank_law(n, k):
    mean = (n + 1) / (k + 1)
    var = k * (n - k) * (n + 1) / ((k + 1) ** 2 * (k + 2))
    return mean, var


def test_paper_rank_law_numbers():
    """Appendix B: E[Rank] = (n+1)/(k+1) = 16385/257 (printed
    63.74; exact 63.755 — reading R-13), Var ~ 3970, sigma ~ 63."""
    mean, var = _rank_law(16384, 256)
    assert abs(mean - 16385 / 257) < 1e-12
    assert abs(mean - 63.74) < 0.02
    assert abs(var - 3970) < 5
    assert abs(math.sqrt(var) - 63) < 0.5


@pytest.mark.parametrize("n,k,trials", [(128, 16, 12800), (1024, 16, 1500)])
def test_sampler_obeys_rank_law(n, k, trials):
    """The minimum sampled position (rank 1 = first offset) of a uniform
    k-subset of n follows the order-statistics law of P:450-454."""
    mean, var = _rank_law(n, k)
    ranks = []
    t = 0
    u = 0
    while t < trials:
        for i in range(64):
            ranks.append(O.sample_offsets(11, u, i, t % 2, n, k)[0] + 1)
            t += 1
            if t == trials:
                break
        u += 1
    ranks = np.array(ranks, dtype=np.float64)
    se = math.sqrt(var / trials)
    assert abs(ranks.mean() - mean) < 4 * se
    assert abs(ranks.var() - var) < 0.15 * var


def test_strided_mode():
    assert O.sample_offsets(0, 0, 0, 0, 128, 16, mode=1) == [4 + 8 * j for j in range(16)]
    assert O.sample_offsets(0, 0, 0, 0, 5, 16, mode=1) == [0, 1, 2, 3, 4]


def test_draw_samples_layout_and_share():
    p = O.AsaParams(block=128, samples=16, seed=3)
    s = O.draw_samples(300, p, 5)
    assert [len(x) for x in s.offsets_q] == [16, 16, 16]
    assert (np.diff(s.rows_q) > 0).all() and (np.diff(s.rows_k) > 0).all()
    assert s.rows_q.max() < 300
    p.share_qk = True
    s2 = O.draw_samples(300, p, 5)
    assert (s2.rows_q == s2.rows_k).all()
    s3 = O.draw_samples(70, p, 5)
    assert s3.offsets_q == [O.sample_offsets(3, 5, 0, 0, 70, 16)]
