"""Pins of the oracle's selection (A7-A8)."""

import math

import numpy as np
import pytest

from oracle import asa_oracle as O


def test_spec_worked_examples():
    # normalised [0.5, 0.3, 0.15, 0.05], tau 0.9 -> m = 3, [1,1,1,0]
    s = O.select_row(np.array([0.5, 0.3, 0.15, 0.05]), 0.9, 1, 4)
    assert s.m == 3 and s.kept == [0, 1, 2]
    # uniform row, N_b = 4, tau 0.5 -> m = 2
    assert O.select_row(np.full(4, 0.25), 0.5, 1, 4).m == 2
    # tau = 1 -> every block kept (dense)
    assert O.select_row(np.array([0.7, 0.1, 0.1, 0.1]), 1.0, 1, 4).kept == [0, 1, 2, 3]
    # ties -> ascending block index
    assert O.select_row(np.array([0.5, 0.5]), 0.5, 1, 2).order == [0, 1]
    assert O.select_row(np.array([0.1, 0.9]), 0.5, 1, 2).order == [1, 0]
    assert O.select_row(np.full(8, 1.0), 0.3, 1, 8).order == list(range(8))


def test_unnormalised_input_is_normalised():
    # P:149 Alg. 1 l.7: the row is L1-normalised before the cut
    a = O.select_row(np.array([5.0, 3.0, 1.5, 0.5]), 0.9, 1, 4)
    assert a.m == 3 and abs(sum(a.phat) - 1) < 1e-15


def _brute_force_m0(row, tau):
    """Library-independent brute force: exact (fsum) mass of the top m blocks
    in np.lexsort order (p desc, id asc)."""
    phat = row / row.sum()
    order = np.lexsort((np.arange(len(row)), -phat))
    for m in range(1, len(row) + 1):
        if math.fsum(phat[order[:m]]) >= tau:
            return m, order
    return len(row), order


def test_cut_matches_brute_force_outside_tie_band():
    rng = np.random.default_rng(0)
    checked = 0
    for trial in range(400):
        Nb = int(rng.integers(1, 300))
        row = rng.dirichlet(np.full(Nb, float(rng.uniform(0.05, 2.0)))) * rng.uniform(0.1, 10)
        tau = float(np.float32(rng.uniform(0.3, 1.0)))
        sel = O.select_row(row, tau, 1, Nb)
        if O.tie_exemption(sel, tau, 1, Nb)["exempt"]:
            continue
        m0, order = _brute_force_m0(row, tau)
        assert sel.m0 == m0
        assert sel.kept == sorted(order[:m0].tolist())
        checked += 1
    assert checked > 350


def test_topm_mode_equals_library_sort():
    """lo = hi = m turns the rule into exact top-m (P:151 clamp)."""
    rng = np.random.default_rng(1)
    for _ in range(100):
        Nb = int(rng.integers(2, 260))
        row = rng.exponential(size=Nb)
        row[rng.integers(0, Nb, size=Nb // 4)] = row[0]       # inject ties
        m = int(rng.integers(1, Nb + 1))
        sel = O.select_row(row, 0.9, m, m)
        order = np.lexsort((np.arange(Nb), -(row / row.sum())))
        assert sel.kept == sorted(order[:m].tolist())


def test_power_of_two_scale_invariance_bit_exact():
    """P_imp * 2^e gives a bit-identical mask (Appendix B §5):
    normalisation divides the exact same mantissas."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        Nb = int(rng.integers(1, 200))
        row = rng.exponential(size=Nb)
        tau = float(rng.uniform(0.2, 1.0))
        base = O.select_row(row, tau, 1, Nb)
        for e in (-7, -1, 1, 5):
            assert O.select_row(row * 2.0 ** e, tau, 1, Nb).kept == base.kept


def test_arbitrary_scale_invariance_modulo_ties():
    rng = np.random.default_rng(3)
    for _ in range(300):
        Nb = int(rng.integers(1, 200))
        row = rng.exponential(size=Nb)
        tau = float(rng.uniform(0.2, 1.0))
        base = O.select_row(row, tau, 1, Nb)
        got = O.select_row(row * float(rng.uniform(0.01, 100)), tau, 1, Nb)
        assert O.check_row_against(base, tau, 1, Nb, got.kept) is None


def test_tau_monotonicity_before_clamp():
    rng = np.random.default_rng(4)
    for _ in range(300):
        Nb = int(rng.integers(1, 200))
        row = rng.exponential(size=Nb)
        t1, t2 = sorted(rng.uniform(0.05, 1.0, size=2))
        a = O.select_row(row, t1, 1, Nb)
        b = O.select_row(row, t2, 1, Nb)
        assert set(a.kept) <= set(b.kept)


@pytest.mark.parametrize("lo,hi", [(1, 1), (3, 3), (2, 10), (5, 256)])
def test_clamp_safety(lo, hi):
    rng = np.random.default_rng(5)
    for case in range(50):
        Nb = int(rng.integers(1, 300))
        l, h = min(lo, Nb), min(hi, Nb)
        if case % 3 == 0:
            row = np.zeros(Nb)
            row[rng.integers(Nb)] = 1.0                           # single spike
        elif case % 3 == 1:
            row = np.full(Nb, 0.3)                                # all ties
        else:
            row = rng.exponential(size=Nb)
        sel = O.select_row(row, float(rng.uniform(0.1, 1.0)), l, max(l, h))
        assert l <= sel.m <= max(l, h) and len(sel.kept) == sel.m
        assert sel.kept == sorted(set(sel.kept))


def test_tie_band_example():
    """SURVEY §8(c) example: [0.3, 0.3, 0.3, 0.1], tau = 0.9.  The top-3 mass
    equals tau up to fp64 rounding (C_3 = 0.9000000000000001 here, after the
    l.7 normalisation), so the row is exempt (T1) and both m = 3 and m = 4
    are accepted; any other count or membership is not."""
    row = np.array([0.3, 0.3, 0.3, 0.1])
    sel = O.select_row(row, 0.9, 1, 4)
    assert sel.m0 in (3, 4)
    te = O.tie_exemption(sel, 0.9, 1, 4)
    assert te["exempt"] and te["t1"] and te["counts"] == {3, 4}
    assert O.check_row_against(sel, 0.9, 1, 4, [0, 1, 2]) is None
    assert O.check_row_against(sel, 0.9, 1, 4, [0, 1, 2, 3]) is None
    assert O.check_row_against(sel, 0.9, 1, 4, [0, 1, 3]) is not None
    assert O.check_row_against(sel, 0.9, 1, 4, [0, 1]) is not None


def test_non_exempt_mismatch_is_rejected():
    sel = O.select_row(np.array([0.5, 0.3, 0.15, 0.05]), 0.9, 1, 4)
    assert O.check_row_against(sel, 0.9, 1, 4, [0, 1]) is not None
    assert O.check_row_against(sel, 0.9, 1, 4, [0, 1, 2]) is None


def test_tau_one_is_dense_even_when_fp64_sum_saturates():
    """S:259 'tau = 1 -> dense': with every score positive the exact
    cumulative mass reaches 1 only at N_b, although the fp64 running sum of
    [1, 1e-20, 1e-20] already equals 1.0 after the first term."""
    row = np.array([1.0, 1e-20, 1e-20, 1e-30])
    sel = O.select_row(row, 1.0, 1, 4)
    assert sel.csum[0] == 1.0           # the fp64 sum saturates at m = 1 ...
    assert sel.m0 == 4 and sel.m == 4   # ... but tau = 1 keeps every block
    assert sel.kept == [0, 1, 2, 3]
    assert O.select_row(row, 1.0, 1, 2).m == 2          # the clamp still applies
    te = O.tie_exemption(sel, 1.0, 1, 4)
    assert not te["t1"]
