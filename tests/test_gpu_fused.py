"""blade_asa_fwd (mask + attention in one call, the attention a programmatic
dependent of the mask's fp64 refinement) equals blade_asa_mask followed by
blade_bsa_fwd bit for bit, with no row, a few rows and every row refined."""

import pytest
import torch

from paper_2508_10774_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A(cuda_dev):
    from paper_2508_10774_b200 import asa
    return asa


@pytest.mark.parametrize("guard", [0.0, 1e-3, 1e30])
@pytest.mark.parametrize("d,impl", [(128, 0), (64, 0), (128, 1), (64, 3), (64, 1)])
def test_fused_equals_two_calls(A, d, impl, guard):
    q, k, v = inputs.smooth(1, 3, 2000, d, (1, 1, 2000), ell=3.0, beta=9.0, seed=d)
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    kw = dict(tau=0.9, keep_min=2, keep_max=12, refine_guard=guard)
    o1, l1, m = A.asa_forward(qd, kd, vd, impl=impl, **kw)
    o2, l2, idx, cnt = A.blade_asa_fwd(qd, kd, vd, impl=impl, **kw)
    torch.cuda.synchronize()
    assert torch.equal(cnt, m.kv_cnt) and (cnt > 0).all()
    assert torch.equal(idx, m.kv_idx)
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    assert torch.equal(l1, l2)


def test_fused_repeated_calls_are_stable(A):
    q, k, v = (t.cuda() for t in inputs.make("tiny", "smooth"))
    outs = [A.blade_asa_fwd(q, k, v, tau=0.9, refine_guard=1e30) for _ in range(5)]
    torch.cuda.synchronize()
    for o, lse, idx, cnt in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(cnt, outs[0][3])


@pytest.mark.parametrize("N", [1, 129, 300, 1407])
@pytest.mark.parametrize("d", [64, 128])
def test_fused_edges_lpt(A, N, d):
    """Odd block counts (the two-block kernel's lone last block), a single
    token, tau mode so the LPT order is active, every row refined."""
    q, k, v = inputs.iid(1, 2, N, d, seed=N + d)
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    for guard in (0.0, 1e30):
        kw = dict(tau=0.8, keep_min=1, refine_guard=guard)
        o1, l1, m = A.asa_forward(qd, kd, vd, **kw)
        o2, l2, idx, cnt = A.blade_asa_fwd(qd, kd, vd, **kw)
        torch.cuda.synchronize()
        assert torch.equal(cnt, m.kv_cnt) and torch.equal(idx, m.kv_idx)
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
        assert torch.equal(l1, l2)


@pytest.mark.parametrize("guard", [0.0, 1e30])
@pytest.mark.parametrize("N,d,n,impl", [(2000, 128, 128, 0), (2000, 64, 100, 0), (1407, 128, 7, 1),
                                        (300, 64, 1000, 3), (2000, 64, 128, 1)])
def test_fused_gt_equals_separate_calls(A, N, d, n, impl, guard):
    """blade_asa_gt_fwd (MeanPool_n + mask + ASA_GT attention, PDL) equals
    blade_gt_pool + blade_asa_mask + blade_bsa_gt_fwd bit for bit; the MMA_SYNC
    impl is UNSUPPORTED for the global tokens."""
    q, k, v = inputs.smooth(1, 2, N, d, (1, 1, N), ell=3.0, beta=9.0, seed=N + d)
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    kw = dict(tau=0.85, keep_min=1, refine_guard=guard)
    o1, l1, m = A.asa_gt_forward(qd, kd, vd, window=n, impl=impl, **kw)
    kg1, vg1 = A.blade_gt_pool(kd, vd, window=n)
    o2, l2, idx, cnt, kg2, vg2 = A.blade_asa_gt_fwd(qd, kd, vd, window=n, impl=impl, **kw)
    torch.cuda.synchronize()
    assert torch.equal(cnt, m.kv_cnt) and torch.equal(idx, m.kv_idx)
    assert torch.equal(kg1, kg2) and torch.equal(vg1, vg2)
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    assert torch.equal(l1, l2)
    with pytest.raises(A.BladeError) as e:
        A.blade_asa_gt_fwd(qd, kd, vd, window=n, impl=A.ATTN_MMA_SYNC, **kw)
    assert e.value.status == A.BLADE_ERR_UNSUPPORTED


@pytest.mark.parametrize("d,impl", [(128, 0), (64, 0), (128, 1)])
def test_fused_many_ctas_mixed_refined_rows(A, d, impl):
    """More CTAs than SMs, a small N_b (several rows share one 128-B line of
    kv_idx) and a mix of refined and unrefined rows: CTAs that waited for the
    refine kernel must read their rewritten lists, not a stale L1 line pulled
    in by a CTA that did not wait (coherent list loads)."""
    q, k, v = inputs.smooth(1, 32, 1000, d, (1, 1, 1000), ell=3.0, beta=9.0, seed=77 + d)
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    kw = dict(tau=0.9, keep_min=1, refine_guard=1e-3)
    o1, l1, m = A.asa_forward(qd, kd, vd, impl=impl, **kw)
    n_ref = int(m.n_refined.item())
    assert 0 < n_ref < 32 * 8, n_ref
    for _ in range(3):
        o2, l2, idx, cnt = A.blade_asa_fwd(qd, kd, vd, impl=impl, **kw)
        torch.cuda.synchronize()
        assert torch.equal(cnt, m.kv_cnt) and torch.equal(idx, m.kv_idx)
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
        assert torch.equal(l1, l2)


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("keep", [None, 3])
def test_fused_persistent_many_items_per_cta(A, d, keep):
    """The AUTO attention is persistent (one CTA per SM walking the (unit,
    pair) items): 96 units x 4 pairs = 384 items, 2-3 per CTA, so TMEM, the
    K/V rings and every barrier phase carry across items, refined rows (whose
    CTA waits for K-mask.4) sit between unrefined ones, tau mode activates the
    LPT order (alternating rounds); the result must equal the separate calls
    and the non-persistent pair kernel (impl PAIR) bit for bit."""
    q, k, v = inputs.smooth(1, 96, 1000, d, (1, 1, 1000), ell=3.0, beta=9.0, seed=5 + d)
    qd, kd, vd = (t.cuda() for t in (q, k, v))
    kw = dict(tau=0.9, keep_min=1, refine_guard=1e-3) if keep is None else \
        dict(tau=0.9, keep_min=keep, keep_max=keep, refine_guard=1e-3)
    o1, l1, m = A.asa_forward(qd, kd, vd, **kw)
    n_ref = int(m.n_refined.item())
    assert 0 < n_ref < 96 * 8, n_ref
    o3 = torch.empty_like(qd)
    l3 = torch.empty_like(l1)
    A.blade_bsa_fwd(qd, kd, vd, m.kv_idx, m.kv_cnt, impl=A.ATTN_TCGEN05_PAIR, o=o3, lse=l3)
    for _ in range(2):
        o2, l2, idx, cnt = A.blade_asa_fwd(qd, kd, vd, **kw)
        torch.cuda.synchronize()
        assert torch.equal(cnt, m.kv_cnt) and torch.equal(idx, m.kv_idx)
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
        assert torch.equal(l1, l2)
    assert torch.equal(o1.view(torch.int16), o3.view(torch.int16))
    assert torch.equal(l1, l3)
