"""Structural checks of the oracle's whole mask (Alg. 1 composed).

The end-to-end composition sample -> probe -> select has no worked example
in the paper, so this file checks invariants only."""

import numpy as np
import pytest

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs


@pytest.mark.parametrize("recipe", ["iid", "smooth"])
def test_tiny_mask_invariants(recipe):
    q, k, v = inputs.make("tiny", recipe)
    p = O.AsaParams(tau=0.9, keep_min=1, keep_max=4)
    r = O.asa_mask(q, k, p)
    BH, Nb, _ = r.mask.shape
    assert (Nb, BH) == (4, 1)
    for u in range(BH):
        for i in range(Nb):
            c = r.kv_cnt[u, i]
            assert 1 <= c <= 4
            idx = r.kv_idx[u, i, :c]
            assert (np.diff(idx) > 0).all() and (r.kv_idx[u, i, c:] == -1).all()
            assert set(np.flatnonzero(r.mask[u, i])) == set(idx.tolist())
            np.testing.assert_allclose(r.p_imp[u, i].max() <= 1.0, True)


def test_tau_one_is_dense_and_clamps_hold():
    q, k, _ = inputs.make("tiny", "smooth")
    r = O.asa_mask(q, k, O.AsaParams(tau=1.0))
    # tau = 1 keeps every block unless fp rounding leaves C_{N_b} < 1, in
    # which case m0 = N_b anyway (reading R-4)
    assert (r.kv_cnt == 4).all()
    r = O.asa_mask(q, k, O.AsaParams(tau=0.01, keep_min=2, keep_max=3))
    assert ((r.kv_cnt >= 2) & (r.kv_cnt <= 3)).all()


def test_sharding_invariance_of_unit_offset():
    """A shard [2, 4) run with unit_offset = 2 reproduces units 2, 3 of the
    full run bit-for-bit (the sampler is keyed by the global unit)."""
    q, k, _ = inputs.iid(1, 4, 384, 32, seed=3)
    full = O.asa_mask(q, k, O.AsaParams(tau=0.8))
    part = O.asa_mask(q[2:4], k[2:4], O.AsaParams(tau=0.8, unit_offset=2))
    assert (part.kv_idx == full.kv_idx[2:4]).all()
    assert (part.sample_idx == full.sample_idx[2:4]).all()
    assert (part.p_imp == full.p_imp[2:4]).all()


def test_supplied_samples_mode_replays():
    q, k, _ = inputs.iid(1, 2, 300, 16, seed=4)
    a = O.asa_mask(q, k, O.AsaParams(tau=0.85, seed=9))
    b = O.asa_mask(q, k, O.AsaParams(tau=0.85, sample_mode=2), supplied_samples=a.sample_idx)
    assert (a.kv_idx == b.kv_idx).all() and (a.p_imp == b.p_imp).all()
