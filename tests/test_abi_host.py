"""Host-side checks of the C-ABI library (no GPU needed, no compute calls):
the library loads, exports every function include/blade_asa.h declares,
and its synchronous validation returns the documented status codes."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "blade_asa.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(blade_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def asa():
    from paper_2508_10774_b200 import asa as A
    return A


def test_header_declares_the_boundary():
    fns = _declared_functions()
    assert {"blade_asa_mask", "blade_bsa_fwd"} <= set(fns)


def test_library_exports_every_declared_symbol(asa):
    lib = ctypes.CDLL(asa.library_path())
    for name in _declared_functions():
        assert hasattr(lib, name), name
    assert set(asa.ABI_SYMBOLS) == set(_declared_functions())


def test_params_struct_layout(asa):
    # blade_asa_params_t: 4+4+4+4+4+4 (+0 pad) +8 +4+4 +8 +4+4 = 56 bytes
    assert ctypes.sizeof(asa.BladeAsaParams) == 56
    assert asa.BladeAsaParams.seed.offset == 24
    assert asa.BladeAsaParams.unit_offset.offset == 40


def test_status_strings_and_version(asa):
    lib = asa._lib
    for s in range(5):
        assert lib.blade_status_string(s)
    assert asa.version() >= 200
    # product build: the pair / one-block tcgen05 kernels only; the mma.sync and
    # three-S-buffer comparison kernels are -DBLADE_WITH_BASELINES-only
    assert asa.impl_built(asa.ATTN_AUTO) and asa.impl_built(asa.ATTN_TCGEN05_PAIR)
    assert asa.impl_built(asa.ATTN_TCGEN05)
    assert not asa.impl_built(asa.ATTN_MMA_SYNC) and not asa.impl_built(asa.ATTN_TCGEN05_TRIPLE)


def test_workspace_sizes(asa):
    lib = asa._lib
    p = asa.make_params(d=128, tau=0.9)
    w1 = lib.blade_asa_mask_workspace_size(12, 32760, 128, ctypes.byref(p))
    # Q_s + K_s + fp32 P_imp + fp64 refine stash for every row
    assert w1 >= 2 * 12 * 256 * 16 * 128 * 2 + 12 * 256 * 256 * 4 + 12 * 256 * 16 * 256 * 8
    assert lib.blade_asa_mask_workspace_size(12, 32760, 96, ctypes.byref(p)) == 0  # d unsupported
    assert lib.blade_bsa_fwd_workspace_size(12, 32760, 128, 128) >= 256
    assert lib.blade_bsa_fwd_workspace_size(12, 32760, 128, 64) == 0


def _mask_call(asa, q=1 << 20, k=1 << 20, BH=1, N=512, d=64, prm=None, kv_idx=1 << 20,
               kv_cnt=1 << 20, ws=1 << 20, wsb=1 << 40, sample_idx=None):
    prm = prm or asa.make_params(d=d)
    return asa._lib.blade_asa_mask(q, k, BH, N, d, ctypes.byref(prm), None, kv_idx, kv_cnt, None,
                                   sample_idx, None, ws, wsb, None)


def test_mask_validation_codes(asa):
    A = asa
    assert _mask_call(A, q=None) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, q=(1 << 20) + 2) == A.BLADE_ERR_INVALID_ARG          # misaligned
    assert _mask_call(A, kv_cnt=None) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, N=0) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, tau=0.0)) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, tau=1.5)) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, keep_min=0)) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, keep_min=5, keep_max=4)) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, samples=200)) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, sample_mode=2)) == A.BLADE_ERR_INVALID_ARG
    assert _mask_call(A, prm=A.make_params(d=64, block=64)) == A.BLADE_ERR_UNSUPPORTED
    assert _mask_call(A, prm=A.make_params(d=64, samples=8)) == A.BLADE_ERR_UNSUPPORTED
    assert _mask_call(A, d=80, prm=A.make_params(d=80)) == A.BLADE_ERR_UNSUPPORTED
    assert _mask_call(A, N=128 * 600) == A.BLADE_ERR_UNSUPPORTED               # N_b > 512
    assert _mask_call(A, ws=None) == A.BLADE_ERR_WORKSPACE
    assert _mask_call(A, wsb=16) == A.BLADE_ERR_WORKSPACE
    assert _mask_call(A, ws=(1 << 20) + 16) == A.BLADE_ERR_WORKSPACE


def test_attn_validation_codes(asa):
    A, lib = asa, asa._lib
    P = 1 << 20

    def call(q=P, o=P, BH=1, N=512, d=64, block=128, scale=0.125, impl=0, ws=P, wsb=1 << 40):
        return lib.blade_bsa_fwd(q, P, P, BH, N, d, block, scale, P, P, o, None, impl, ws, wsb,
                                 None)

    assert call(q=None) == A.BLADE_ERR_INVALID_ARG
    assert call(o=P + 8) == A.BLADE_ERR_INVALID_ARG
    assert call(scale=0.0) == A.BLADE_ERR_INVALID_ARG
    assert call(impl=7) == A.BLADE_ERR_INVALID_ARG
    assert call(block=64) == A.BLADE_ERR_UNSUPPORTED
    assert call(d=256) == A.BLADE_ERR_UNSUPPORTED
    assert call(ws=None) == A.BLADE_ERR_WORKSPACE


def test_keep_count_integer_rounding(asa):
    assert asa.keep_count(50_000, 256) == 13          # ceil(0.05 * 256)
    assert asa.keep_count(200_000, 256) == 52
    assert asa.keep_count(1, 4) == 1


def test_host_pipeline_validation_codes(asa):
    A, lib = asa, asa._lib
    P = 1 << 20
    prm = A.make_params(d=64)

    def call(q=P, o=P, BH=2, N=512, d=64, impl=0, chunk=0, ws=P, wsb=1 << 40, p=prm):
        return lib.blade_asa_fwd_host(q, P, P, BH, N, d, ctypes.byref(p), impl, chunk, o, None,
                                      None, ws, wsb, None)

    assert call(q=None) == A.BLADE_ERR_INVALID_ARG
    assert call(o=None) == A.BLADE_ERR_INVALID_ARG
    assert call(BH=0) == A.BLADE_ERR_INVALID_ARG
    assert call(chunk=-1) == A.BLADE_ERR_INVALID_ARG
    assert call(impl=9) == A.BLADE_ERR_INVALID_ARG
    assert call(p=A.make_params(d=64, tau=2.0)) == A.BLADE_ERR_INVALID_ARG
    assert call(d=80, p=A.make_params(d=80)) == A.BLADE_ERR_UNSUPPORTED
    assert call(ws=None) == A.BLADE_ERR_WORKSPACE
    assert call(wsb=16) == A.BLADE_ERR_WORKSPACE


def test_host_pipeline_workspace_scales_with_chunk(asa):
    lib = asa._lib
    p = asa.make_params(d=128)
    w1 = lib.blade_asa_fwd_host_workspace_size(12, 32760, 128, ctypes.byref(p), 1)
    w3 = lib.blade_asa_fwd_host_workspace_size(12, 32760, 128, ctypes.byref(p), 3)
    tok = 32760 * 128 * 2
    assert w1 >= 2 * 4 * tok  # two slots of Q, K, V, O for one unit
    assert w3 >= 2 * 4 * 3 * tok and w3 > w1
    assert lib.blade_asa_fwd_host_workspace_size(12, 32760, 128, ctypes.byref(p), 0) == w1


def test_gt_validation_codes(asa):
    A, lib = asa, asa._lib
    P = 1 << 20
    assert lib.blade_gt_pool(None, P, 1, 512, 64, 128, P, P, None) == A.BLADE_ERR_INVALID_ARG
    assert lib.blade_gt_pool(P, P, 1, 512, 64, 0, P, P, None) == A.BLADE_ERR_INVALID_ARG
    assert lib.blade_gt_pool(P, P, 1, 512, 64, 128, P + 4, P, None) == A.BLADE_ERR_INVALID_ARG
    assert lib.blade_gt_pool(P, P, 1, 512, 96, 128, P, P, None) == A.BLADE_ERR_UNSUPPORTED

    def call(kg=P, window=128, impl=0, d=64, ws=P):
        return lib.blade_bsa_gt_fwd(P, P, P, 1, 512, d, 128, 0.125, P, P, kg, P, window, P, None,
                                    impl, ws, 1 << 40, None)

    assert call(kg=None) == A.BLADE_ERR_INVALID_ARG
    assert call(window=0) == A.BLADE_ERR_INVALID_ARG
    assert call(impl=A.ATTN_MMA_SYNC) == A.BLADE_ERR_UNSUPPORTED
    assert call(d=256) == A.BLADE_ERR_UNSUPPORTED
    assert call(ws=None) == A.BLADE_ERR_WORKSPACE


@pytest.mark.parametrize("t,h,w,n_text", [(1, 16, 32, 0), (21, 30, 52, 0), (13, 30, 45, 226),
                                          (1, 4, 5, 0), (2, 7, 3, 2), (1, 1, 1, 0), (3, 9, 9, 0)])
def test_gilbert_order_host_matches_oracle(asa, t, h, w, n_text):
    """blade_gilbert_order is a host function: compare it with the oracle here."""
    from oracle import asa_oracle as O
    perm = asa.gilbert_order(t, h, w, n_text).numpy()
    assert (perm == O.gilbert_permutation(t, h, w, n_text)).all()


def test_gilbert_exhaustive_small_grids_match_oracle(asa):
    from oracle import asa_oracle as O
    for h in range(1, 20):
        for w in range(1, 20):
            assert (asa.gilbert_order(1, h, w).numpy() == O.gilbert_permutation(1, h, w)).all(), (h, w)


def test_gilbert_and_permute_validation(asa):
    A, lib = asa, asa._lib
    buf = (ctypes.c_int32 * 8)()
    assert lib.blade_gilbert_order(1, 2, 4, 0, buf, 7) == A.BLADE_ERR_INVALID_ARG
    assert lib.blade_gilbert_order(0, 2, 4, 0, buf, 0) == A.BLADE_ERR_INVALID_ARG
    assert lib.blade_gilbert_order(1, 2, 4, 0, None, 8) == A.BLADE_ERR_INVALID_ARG
    P = 1 << 20
    assert lib.blade_permute_tokens(P, 1, 16, 12, P, 0, P + 4096, None) == A.BLADE_ERR_INVALID_ARG
    assert lib.blade_permute_tokens(P, 1, 16, 64, P, 0, P, None) == A.BLADE_ERR_INVALID_ARG
