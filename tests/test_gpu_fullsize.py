"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (all units of one layer in one call).

Masks: every unit vs the oracle (bit-exact outside the 1e-6 tie band).
Attention: sampled query blocks, computed one by one by the oracle, using
the GPU's own kv lists (mask parity is checked separately above)."""

import numpy as np
import pytest
import torch

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs

from . import _parity as PT

pytestmark = pytest.mark.gpu

CASES = {
    # BASELINE.json configs[1]: Wan2.1-1.3B layer, keep-ratio 51/256 (bench default)
    "wan-keep51": ("wan", dict(tau=0.9, keep_min=51, keep_max=51)),
    # Wan, pure tau mode (lo = ceil(0.05 N_b) = 13)
    "wan-tau0.9": ("wan", dict(tau=0.9, keep_min=13)),
    # BASELINE.json configs[2]: CogVideoX-5B layer, keep-ratio 25/139
    "cog-keep25": ("cog", dict(tau=0.9, keep_min=25, keep_max=25)),
    "cog-tau0.95": ("cog", dict(tau=0.95, keep_min=7)),
}


@pytest.fixture(scope="module")
def A(cuda_dev):
    from paper_2508_10774_b200 import asa
    return asa


_cache = {}


def _inputs(name):
    if name not in _cache:
        _cache[name] = inputs.make(name, "smooth")
    return _cache[name]


@pytest.mark.parametrize("case", list(CASES), ids=list(CASES))
def test_fullsize_mask_and_sampled_attention(A, case):
    wl, kw = CASES[case]
    q, k, v = _inputs(wl)
    BH, N, d = q.shape
    p = O.AsaParams(**kw)
    qd, kd, vd = PT.to_dev(q, k, v)
    o, lse, m = A.asa_forward(qd, kd, vd, want_pimp=True, **kw)
    torch.cuda.synchronize()
    # --- mask: all units ---
    units = list(range(BH)) if BH <= 12 else list(range(0, BH, 4))
    ref = O.asa_mask(q, k, p, units=units)
    stats = PT.check_mask(ref, m, p, units=units)
    assert stats["exempt"] <= stats["rows"] // 50, stats
    # --- attention: sampled query blocks, oracle one by one ---
    Nb = O.num_blocks(N, 128)
    kv_idx, kv_cnt = m.kv_idx.cpu().numpy(), m.kv_cnt.cpu().numpy()
    qblocks = [0, 1, Nb // 2, Nb - 2, Nb - 1]
    for u in (0, BH // 2, BH - 1):
        o_ref, lse_ref = O.sparse_attention_unit(q[u], k[u], v[u], kv_idx[u], kv_cnt[u], 128,
                                                 O.default_scale(d), qblocks)
        PT.check_attention(o[u], lse[u], o_ref, lse_ref)


def test_fullsize_one_block_kernel_agrees(A):
    """The one-block tcgen05 kernel and the pair kernel (AUTO) on the Wan layer."""
    q, k, v = _inputs("wan")
    qd, kd, vd = PT.to_dev(q, k, v)
    m = A.blade_asa_mask(qd, kd, tau=0.9, keep_min=51, keep_max=51)
    o1, l1 = A.blade_bsa_fwd(qd, kd, vd, m.kv_idx, m.kv_cnt, impl=A.ATTN_TCGEN05)
    o2, l2 = A.blade_bsa_fwd(qd, kd, vd, m.kv_idx, m.kv_cnt, impl=A.ATTN_AUTO)
    torch.cuda.synchronize()
    assert (o1.float() - o2.float()).abs().max().item() <= 2e-2
    assert (l1 - l2).abs().max().item() <= 1e-3
