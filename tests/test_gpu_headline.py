"""The headline path at BASELINE.json's full sizes, exactly as bench.py times
it: the single fused call ``blade_asa_fwd`` (PDL attention behind the fp64
refinement, provisional negative counts, LPT order in tau mode) and the
host-buffer entry point ``blade_asa_fwd_host`` (the bench's e2e leg).

Masks: every unit vs the fp64 oracle (bit-exact outside the 1e-6 tie band).
Attention: the oracle one query block at a time on the GPU's own lists, for
fixed query blocks plus the rows with the smallest decision margin (the rows
the fp64 refinement recomputes) — i.e. the CTAs that waited in
griddepcontrol.wait."""

import numpy as np
import pytest
import torch

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs

from . import _parity as PT

pytestmark = pytest.mark.gpu

CASES = {
    # bench default (BASELINE.json configs[1]): keep-ratio 51/256
    "wan-keep51": ("wan", dict(tau=0.9, keep_min=51, keep_max=51)),
    # Wan, tau mode: LPT order active, refined rows in the fused call
    "wan-tau0.9": ("wan", dict(tau=0.9, keep_min=13)),
    # BASELINE.json configs[2]: every one of the 48 CogVideoX units
    "cog-keep25": ("cog", dict(tau=0.9, keep_min=25, keep_max=25)),
    "cog-tau0.9": ("cog", dict(tau=0.9, keep_min=7)),
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


def _margin(sel: O.RowSelection, tau: float) -> float:
    """Relative distance of the row's decision from a flip (cut or membership)."""
    Nb = len(sel.phat)
    cands = [abs(sel.csum[m - 1] - tau) / tau for m in (sel.m0 - 1, sel.m0)
             if 1 <= m <= Nb and tau < 1.0]
    if sel.m < Nb:
        a, b = sel.phat[sel.order[sel.m - 1]], sel.phat[sel.order[sel.m]]
        cands.append((a - b) / a)
    return min(cands) if cands else 1.0


@pytest.mark.parametrize("case", list(CASES), ids=list(CASES))
def test_fused_headline_call_vs_oracle(A, case):
    wl, kw = CASES[case]
    q, k, v = _inputs(wl)
    BH, N, d = q.shape
    p = O.AsaParams(**kw)
    qd, kd, vd = PT.to_dev(q, k, v)
    o, lse, kv_idx, kv_cnt = A.blade_asa_fwd(qd, kd, vd, **kw)
    torch.cuda.synchronize()

    class Got:  # the fields check_mask reads
        pass
    got = Got()
    got.kv_idx, got.kv_cnt, got.mask = kv_idx, kv_cnt, None
    ref = O.asa_mask(q, k, p)                       # every unit
    stats = PT.check_mask(ref, got, p)
    assert stats["exempt"] <= stats["rows"] // 50, stats
    Nb = O.num_blocks(N, 128)
    idx_np, cnt_np = kv_idx.cpu().numpy(), kv_cnt.cpu().numpy()
    units = sorted({0, BH // 3, BH // 2, BH - 1})
    for u in units:
        margins = sorted(range(Nb), key=lambda i: _margin(ref.rows[u][i], float(kw["tau"])))
        qblocks = sorted({0, 1, Nb // 2, Nb - 1, *margins[:4]})
        o_ref, lse_ref = O.sparse_attention_unit(q[u], k[u], v[u], idx_np[u], cnt_np[u], 128,
                                                 O.default_scale(d), qblocks)
        PT.check_attention(o[u], lse[u], o_ref, lse_ref)


@pytest.mark.parametrize("wl,kw", [("wan", dict(tau=0.9, keep_min=51, keep_max=51)),
                                   ("cog", dict(tau=0.9, keep_min=7))])
def test_host_entry_point_fullsize(A, wl, kw):
    """blade_asa_fwd_host (the bench's e2e call) == blade_asa_fwd bit for bit
    at full size, so the oracle parity above carries over."""
    q, k, v = _inputs(wl)
    BH, N, d = q.shape
    qd, kd, vd = PT.to_dev(q, k, v)
    o_d, lse_d, _, cnt_d = A.blade_asa_fwd(qd, kd, vd, **kw)
    qp, kp, vp = (t.pin_memory() for t in (q, k, v))
    cnt = torch.empty((BH, O.num_blocks(N, 128)), dtype=torch.int32).pin_memory()
    o_h, lse_h = A.blade_asa_fwd_host(qp, kp, vp, kv_cnt=cnt, **kw)
    torch.cuda.synchronize()
    assert torch.equal(cnt, cnt_d.cpu())
    assert torch.equal(o_h.view(torch.int16), o_d.cpu().view(torch.int16))
    assert torch.equal(lse_h, lse_d.cpu())
