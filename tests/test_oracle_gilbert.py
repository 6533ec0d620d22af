"""Pins of the oracle's Gilbert rearrangement (F2; Alg. 1 l.1;
readings R-21, R-22): a bijection; inside a frame every two consecutive
curve cells are 4-neighbours (exhaustive over all 2-D grids up to 32 x 32,
the property that makes it a space-filling curve); for 2^k x 2^k grids the
curve is a Hilbert curve (starts at a corner, ends at the adjacent corner,
and every aligned 2^j x 2^j quadrant is visited contiguously); blocks of
consecutive tokens are more compact than raster blocks; apply/undo round trip."""

import numpy as np
import pytest

from oracle import asa_oracle as O


def _check_curve(w, h):
    cells = O.gilbert2d_cells(w, h)
    assert len(cells) == w * h
    assert len(set(cells)) == w * h
    assert all(0 <= x < w and 0 <= y < h for x, y in cells)
    assert cells[0] == (0, 0)
    for (x0, y0), (x1, y1) in zip(cells, cells[1:]):
        assert abs(x0 - x1) + abs(y0 - y1) == 1, (w, h, (x0, y0), (x1, y1))


def test_adjacency_exhaustive_small():
    """Unit steps everywhere unless the longer side is odd and the shorter
    even: the curve runs from (0, 0) to the far corner of the longer side,
    two cells of the same checkerboard colour, which a unit-step path over an
    even number of cells cannot join (parity), so one diagonal step is needed
    and the curve takes exactly one."""
    for w in range(1, 33):
        for h in range(1, 33):
            if max(w, h) % 2 == 1 and min(w, h) % 2 == 0 and w != h:
                continue
            _check_curve(w, h)


def test_odd_long_side_has_one_diagonal():
    for w in range(1, 33):
        for h in range(1, 33):
            if not (max(w, h) % 2 == 1 and min(w, h) % 2 == 0 and w != h):
                continue
            cells = O.gilbert2d_cells(w, h)
            assert len(set(cells)) == w * h and cells[0] == (0, 0)
            steps = [(abs(x0 - x1), abs(y0 - y1)) for (x0, y0), (x1, y1) in zip(cells, cells[1:])]
            assert all(s in ((1, 0), (0, 1), (1, 1)) for s in steps)
            assert sum(s == (1, 1) for s in steps) <= 1


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_power_of_two_is_hilbert(k):
    n = 1 << k
    cells = O.gilbert2d_cells(n, n)
    pos = {c: i for i, c in enumerate(cells)}
    # ends on a corner adjacent to the start corner
    assert cells[-1] in ((n - 1, 0), (0, n - 1))
    # every aligned 2^j x 2^j quadrant occupies a contiguous range of the curve
    for j in range(1, k):
        s = 1 << j
        for qx in range(0, n, s):
            for qy in range(0, n, s):
                idx = sorted(pos[(x, y)] for x in range(qx, qx + s) for y in range(qy, qy + s))
                assert idx[-1] - idx[0] == s * s - 1


@pytest.mark.parametrize("t,h,w,n_text", [(1, 16, 32, 0), (21, 30, 52, 0), (13, 30, 45, 226),
                                          (2, 1, 7, 3), (3, 5, 1, 0)])
def test_permutation_bijection_and_frame_major(t, h, w, n_text):
    perm = O.gilbert_permutation(t, h, w, n_text)
    N = n_text + t * h * w
    assert sorted(perm.tolist()) == list(range(N))
    assert (perm[:n_text] == np.arange(n_text)).all()          # R-22
    frames = (perm[n_text:] - n_text) // (h * w)
    assert (frames == np.repeat(np.arange(t), h * w)).all()     # R-21: frame-major


def test_blocks_are_more_compact_than_raster():
    """Mean pairwise Manhattan distance inside 128-token blocks (Wan frame 30 x 52)."""
    h, w, b = 30, 52, 128
    perm = O.gilbert_permutation(1, h, w)
    ys, xs = np.divmod(np.arange(h * w), w)

    def spread(order):
        tot = []
        for s in range(0, len(order) - b + 1, b):
            idx = order[s:s + b]
            dy = np.abs(ys[idx][:, None] - ys[idx][None, :])
            dx = np.abs(xs[idx][:, None] - xs[idx][None, :])
            tot.append((dy + dx).mean())
        return float(np.mean(tot))

    assert spread(perm) < 0.7 * spread(np.arange(h * w))


def test_apply_undo_round_trip():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 1 + 4 * 6, 5))
    perm = O.gilbert_permutation(1, 4, 6, n_text=1)
    y = O.apply_permutation(x, perm)
    assert (y[:, 0] == x[:, perm[0]]).all() and (y[:, 5] == x[:, perm[5]]).all()
    assert (O.undo_permutation(y, perm) == x).all()
    rev = np.arange(3)[::-1]
    assert (O.apply_permutation(np.arange(3)[:, None], rev)[:, 0] == rev).all()
