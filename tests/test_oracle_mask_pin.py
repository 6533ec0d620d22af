"""Pins of the oracle's composed mask ``asa_mask`` (Alg. 1).

The composition sample -> probe -> select has no worked example in the paper,
so it is pinned against an independent recomputation that shares nothing
with ``oracle/asa_oracle.py`` beyond the KAT-pinned sampler (tests/golden):

* k = b (P:117 vs P:146-147): sampling every token of every block makes the
  probe the conceptual full importance map, so ``asa_mask`` must equal torch
  dense softmax over all N keys + ``max_pool2d(ceil_mode)`` followed by a
  brute-force selection (math.fsum normalisation and prefix sums, numpy
  lexsort order, the clamp of P:151).
* k = 16: the library probe (torch.softmax + max_pool2d on the sampled
  logits, ``tests/test_oracle_probe.torch_probe``) on the KAT-pinned sample
  offsets of the GLOBAL unit index, then the same brute-force selection.

A plausible wiring mistake in ``asa_mask`` — Q and K swapped in the probe, a
wrong scale, the local instead of the global unit index, Q and K sharing one
sample draw, the clamp applied before the cut, an off-by-one in m — changes
``kv_idx`` / ``kv_cnt`` on these inputs and fails here.

Rows whose brute-force decision sits within 1e-9 of a tie (cut or membership)
are checked for validity instead of bit-exactness: fsum and the oracle's
sequential fp64 sums may legitimately decide them differently; the count of
such rows is asserted to be tiny.
"""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs
from tests.test_oracle_probe import torch_probe

TIE = 1e-9


def brute_select(p_row, tau: float, lo: int, hi: int):
    """Alg. 1 l.7-10 by brute force: (kept ascending, m, near_tie)."""
    Nb = len(p_row)
    Z = math.fsum(float(x) for x in p_row)
    phat = np.array([float(x) / Z for x in p_row])
    order = np.lexsort((np.arange(Nb), -phat))          # p-hat desc, then block id asc
    prefix = [math.fsum(phat[order[:m]]) for m in range(1, Nb + 1)]
    m0 = Nb
    if tau < 1.0:
        m0 = next((m for m in range(1, Nb + 1) if prefix[m - 1] >= tau), Nb)
    m = min(max(m0, lo), hi)
    # tau = 1 is dense by definition (reading R-4), never a cut tie
    near = tau < 1.0 and any(abs(prefix[mm - 1] - tau) <= TIE * tau
                             for mm in (m0 - 1, m0) if mm >= 1)
    if m < Nb:
        a, b = phat[order[m - 1]], phat[order[m]]
        near |= (a - b) <= TIE * a
    return sorted(order[:m].tolist()), m, near, phat


def check_against(mr, u, P_ref, tau, lo, hi):
    """Compare one unit of asa_mask with the brute-force selection of P_ref."""
    Nb = P_ref.shape[0]
    n_near = 0
    for i in range(Nb):
        kept, m, near, phat = brute_select(P_ref[i], tau, lo, hi)
        got_m = int(mr.kv_cnt[u, i])
        got = mr.kv_idx[u, i, :got_m].tolist()
        assert (mr.kv_idx[u, i, got_m:] == -1).all()
        assert lo <= got_m <= hi
        if near:
            n_near += 1
            # validity: every kept block at least as important as every dropped one
            dropped = sorted(set(range(Nb)) - set(got))
            if dropped:
                assert phat[got].min() >= phat[dropped].max() * (1 - 1e-9)
            continue
        assert got_m == m, (u, i, got_m, m)
        assert got == kept, (u, i)
    return n_near


def clamp_lohi(Nb, lo, hi):
    return min(lo, Nb), min(hi, Nb)


@pytest.mark.parametrize("N,d,b,seed,recipe", [
    (512, 32, 128, 1, "iid"), (700, 32, 128, 2, "smooth"), (333, 16, 64, 3, "smooth"),
    (200, 16, 32, 4, "iid"), (96, 8, 32, 5, "smooth")])
@pytest.mark.parametrize("tau,lo,hi", [(0.5, 1, 1 << 30), (0.9, 1, 1 << 30), (0.95, 2, 5),
                                      (0.9, 3, 3), (1.0, 1, 1 << 30)])
def test_exhaustive_mask_equals_dense_importance_selection(N, d, b, seed, recipe, tau, lo, hi):
    """k = b: asa_mask == torch dense softmax + max_pool2d(ceil_mode) + brute
    selection (P:117 full importance; Alg. 1 l.7-10)."""
    if recipe == "iid":
        q, k, _ = inputs.iid(1, 2, N, d, seed)
    else:
        side = int(math.ceil(math.sqrt(N)))
        grid = None
        for t in range(1, N + 1):   # any (t, y, x) with t*y*x == N
            if N % t == 0 and (N // t) % side == 0:
                grid = (t, side, N // t // side)
                break
        grid = grid or (1, 1, N)
        q, k, _ = inputs.smooth(1, 2, N, d, grid, ell=2.0, beta=6.0, seed=seed)
    p = O.AsaParams(block=b, samples=b, tau=tau, keep_min=lo, keep_max=hi, seed=seed,
                    unit_offset=7)
    mr = O.asa_mask(q, k, p)
    Nb = (N + b - 1) // b
    lo_c, hi_c = clamp_lohi(Nb, lo, hi)
    scale = float(np.float32(1.0 / math.sqrt(d)))
    n_near = 0
    for u in range(q.shape[0]):
        qt = q[u].double()
        kt = k[u].double()
        P = torch.softmax((qt @ kt.T) * scale, dim=-1)
        P_imp = F.max_pool2d(P[None, None], kernel_size=b, stride=b, ceil_mode=True)[0, 0]
        P_imp = P_imp.numpy()
        np.testing.assert_allclose(mr.p_imp[u], P_imp, rtol=1e-12, atol=0)
        n_near += check_against(mr, u, P_imp, tau, lo_c, hi_c)
    assert n_near <= 1


@pytest.mark.parametrize("N,d,seed,recipe,unit_offset", [
    (1000, 32, 11, "iid", 0), (2000, 64, 12, "smooth", 5), (777, 16, 13, "smooth", 3),
    (130, 32, 14, "iid", 9)])
@pytest.mark.parametrize("tau,lo,hi", [(0.9, 1, 1 << 30), (0.95, 2, 1 << 30), (0.8, 2, 4),
                                      (0.9, 3, 3)])
def test_sampled_mask_equals_library_probe_selection(N, d, seed, recipe, unit_offset, tau, lo,
                                                     hi):
    """k = 16: asa_mask == library probe (torch softmax + max_pool2d on the
    sampled logits) on the KAT-pinned offsets of the global unit index, then
    brute selection (Alg. 1 l.3-10)."""
    b, kk = 128, 16
    if recipe == "iid":
        q, k, _ = inputs.iid(1, 3, N, d, seed)
    else:
        grid = {2000: (2, 25, 40), 777: (1, 21, 37)}[N]
        q, k, _ = inputs.smooth(1, 3, N, d, grid, ell=3.0, beta=8.0, seed=seed)
    p = O.AsaParams(block=b, samples=kk, tau=tau, keep_min=lo, keep_max=hi, seed=seed + 100,
                    unit_offset=unit_offset)
    mr = O.asa_mask(q, k, p)
    Nb = (N + b - 1) // b
    lo_c, hi_c = clamp_lohi(Nb, lo, hi)
    scale = float(np.float32(1.0 / math.sqrt(d)))
    n_near = 0
    for u in range(q.shape[0]):
        ug = unit_offset + u
        oq = [O.sample_offsets(seed + 100, ug, i, 0, min(b, N - i * b), kk) for i in range(Nb)]
        ok = [O.sample_offsets(seed + 100, ug, i, 1, min(b, N - i * b), kk) for i in range(Nb)]
        for i in range(Nb):
            assert mr.sample_idx[u, 0, i, :len(oq[i])].tolist() == oq[i]
            assert mr.sample_idx[u, 1, i, :len(ok[i])].tolist() == ok[i]

        class S:  # the fields torch_probe reads
            offsets_q, offsets_k = oq, ok
        P_imp = torch_probe(q[u].float().numpy(), k[u].float().numpy(), S, Nb, b, kk, scale)
        np.testing.assert_allclose(mr.p_imp[u], P_imp, rtol=1e-12, atol=0)
        n_near += check_against(mr, u, P_imp, tau, lo_c, hi_c)
    assert n_near <= 1


def test_brute_selection_detects_swapped_probe():
    """Sanity of the pin itself: a deliberately mis-wired mask (Q and K
    swapped in the probe) is caught by the comparison above."""
    N, d = 1000, 32
    q, k, _ = inputs.iid(1, 1, N, d, 21)
    p = O.AsaParams(tau=0.9, seed=5)
    good = O.asa_mask(q, k, p)
    bad = O.asa_mask(k, q, p)
    assert not np.array_equal(good.kv_idx, bad.kv_idx)


@pytest.mark.parametrize("lo,hi", [(0, 4), (3, 2), (-1, 5)])
def test_invalid_clamps_rejected_like_the_abi(lo, hi):
    """keep_min < 1 or keep_max < keep_min is an argument error, as
    blade_asa_mask returns BLADE_ERR_INVALID_ARG (include/blade_asa.h)."""
    q, k, _ = inputs.iid(1, 1, 256, 16, 1)
    with pytest.raises(ValueError):
        O.asa_mask(q, k, O.AsaParams(keep_min=lo, keep_max=hi))


def test_clamps_above_nb_are_clipped():
    """keep_min / keep_max above N_b clip to N_b (the ABI does the same)."""
    q, k, _ = inputs.iid(1, 1, 300, 16, 2)
    r = O.asa_mask(q, k, O.AsaParams(tau=0.1, keep_min=10, keep_max=20))
    assert (r.kv_cnt == 3).all()
