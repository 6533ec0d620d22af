"""Thin Python binding of the C ABI in include/blade_asa.h.

Argument marshalling only: every step of the ASA forward runs in the CUDA
kernels of ``lib/libblade_asa.so``.  torch supplies device memory and the
current stream.  Importing this module fails loudly if the library is
missing; there is no CPU or PyTorch fallback.

Python names match the ABI:  ``blade_asa_mask``, ``blade_bsa_fwd``.
``asa_forward`` chains the two (the whole hot path).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                         os.environ.get("BLADE_LIB", "libblade_asa.so"))
if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -m paper_2508_10774_b200.build` "
        "(there is no fallback path)")
_lib = ctypes.CDLL(_LIB_PATH)

BLADE_OK, BLADE_ERR_INVALID_ARG, BLADE_ERR_UNSUPPORTED, BLADE_ERR_WORKSPACE, BLADE_ERR_CUDA = range(5)
ATTN_AUTO, ATTN_TCGEN05, ATTN_MMA_SYNC, ATTN_TCGEN05_PAIR, ATTN_TCGEN05_TRIPLE = 0, 1, 2, 3, 4

ABI_SYMBOLS = ("blade_asa_mask_workspace_size", "blade_asa_mask", "blade_bsa_fwd_workspace_size",
               "blade_bsa_fwd", "blade_asa_fwd_workspace_size", "blade_asa_fwd",
               "blade_bsa_bwd_workspace_size", "blade_bsa_bwd",
               "blade_gt_pool", "blade_bsa_gt_fwd",
               "blade_bsa_gt_bwd_workspace_size", "blade_bsa_gt_bwd", "blade_asa_gt_fwd",
               "blade_gilbert_order", "blade_permute_tokens",
               "blade_asa_fwd_host_workspace_size", "blade_asa_fwd_host",
               "blade_status_string", "blade_version", "blade_attn_impl_built")


class BladeAsaParams(ctypes.Structure):
    """Mirror of blade_asa_params_t (field order and types must match)."""

    _fields_ = [("block", ctypes.c_int32), ("samples", ctypes.c_int32), ("tau", ctypes.c_float),
                ("keep_min", ctypes.c_int32), ("keep_max", ctypes.c_int32),
                ("scale", ctypes.c_float), ("seed", ctypes.c_uint64),
                ("sample_mode", ctypes.c_int32), ("share_qk", ctypes.c_int32),
                ("unit_offset", ctypes.c_int64), ("refine_guard", ctypes.c_float),
                ("reserved", ctypes.c_int32)]


_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
_lib.blade_asa_mask_workspace_size.restype = _sz
_lib.blade_asa_mask_workspace_size.argtypes = [_i64, _i32, _i32, ctypes.POINTER(BladeAsaParams)]
_lib.blade_asa_mask.restype = ctypes.c_int
_lib.blade_asa_mask.argtypes = [_vp, _vp, _i64, _i32, _i32, ctypes.POINTER(BladeAsaParams),
                                _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.blade_bsa_fwd_workspace_size.restype = _sz
_lib.blade_bsa_fwd_workspace_size.argtypes = [_i64, _i32, _i32, _i32]
_lib.blade_bsa_fwd.restype = ctypes.c_int
_lib.blade_bsa_fwd.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32, _i32, ctypes.c_float, _vp, _vp,
                               _vp, _vp, _i32, _vp, _sz, _vp]
_lib.blade_asa_fwd_workspace_size.restype = _sz
_lib.blade_asa_fwd_workspace_size.argtypes = [_i64, _i32, _i32, ctypes.POINTER(BladeAsaParams)]
_lib.blade_asa_fwd.restype = ctypes.c_int
_lib.blade_asa_fwd.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32, ctypes.POINTER(BladeAsaParams),
                               _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.blade_bsa_bwd_workspace_size.restype = _sz
_lib.blade_bsa_bwd_workspace_size.argtypes = [_i64, _i32, _i32, _i32]
_lib.blade_bsa_bwd.restype = ctypes.c_int
_lib.blade_bsa_bwd.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32,
                               ctypes.c_float, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.blade_gt_pool.restype = ctypes.c_int
_lib.blade_gt_pool.argtypes = [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp]
_lib.blade_bsa_gt_fwd.restype = ctypes.c_int
_lib.blade_bsa_gt_fwd.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32, _i32, ctypes.c_float, _vp,
                                  _vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp, _sz, _vp]
_lib.blade_bsa_gt_bwd_workspace_size.restype = _sz
_lib.blade_bsa_gt_bwd_workspace_size.argtypes = [_i64, _i32, _i32, _i32, _i32]
_lib.blade_bsa_gt_bwd.restype = ctypes.c_int
_lib.blade_bsa_gt_bwd.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i64, _i32, _i32,
                                  _i32, ctypes.c_float, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.blade_asa_gt_fwd.restype = ctypes.c_int
_lib.blade_asa_gt_fwd.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32, ctypes.POINTER(BladeAsaParams),
                                  _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.blade_gilbert_order.restype = ctypes.c_int
_lib.blade_gilbert_order.argtypes = [_i32, _i32, _i32, _i32, _vp, _i64]
_lib.blade_permute_tokens.restype = ctypes.c_int
_lib.blade_permute_tokens.argtypes = [_vp, _i64, _i32, _i32, _vp, _i32, _vp, _vp]
_lib.blade_asa_fwd_host_workspace_size.restype = _sz
_lib.blade_asa_fwd_host_workspace_size.argtypes = [_i64, _i32, _i32,
                                                   ctypes.POINTER(BladeAsaParams), _i32]
_lib.blade_asa_fwd_host.restype = ctypes.c_int
_lib.blade_asa_fwd_host.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32,
                                    ctypes.POINTER(BladeAsaParams), _i32, _i32, _vp, _vp, _vp,
                                    _vp, _sz, _vp]
_lib.blade_status_string.restype = ctypes.c_char_p
_lib.blade_status_string.argtypes = [ctypes.c_int]
_lib.blade_version.restype = _i32
_lib.blade_attn_impl_built.restype = _i32
_lib.blade_attn_impl_built.argtypes = [_i32]


class BladeError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {_lib.blade_status_string(status).decode()} (status {status})")
        self.status = status


def library_path() -> str:
    return _LIB_PATH


def version() -> int:
    return int(_lib.blade_version())


def impl_built(impl: int) -> bool:
    """Is attention implementation `impl` compiled into the library?"""
    return bool(_lib.blade_attn_impl_built(impl))


def default_scale(d: int) -> float:
    """fp32(1/sqrt(d)) (reading R-3)."""
    return float(torch.tensor(1.0 / math.sqrt(d), dtype=torch.float32))


def num_blocks(N: int, block: int = 128) -> int:
    return (N + block - 1) // block


def keep_count(ratio_ppm: int, Nb: int) -> int:
    """Fraction (parts per million) of N_b -> block count, integer ceil (>= 1)."""
    return max(1, (ratio_ppm * Nb + 999_999) // 1_000_000)


_workspaces: dict = {}


def _workspace(nbytes: int, device: torch.device, tag: str, stream=None) -> torch.Tensor:
    """Scratch for one entry point, cached per (device, tag, stream): two
    calls on different streams never share scratch (refine queue, Q_s/K_s,
    LPT order).  The buffer is allocated on ``stream`` (the caching
    allocator then only recycles it after work queued there), so a regrowth
    cannot hand memory still in use by an earlier launch to anyone else."""
    s = torch.cuda.current_stream(device) if stream is None else stream
    key = (device, tag, s.cuda_stream)
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        with torch.cuda.stream(s):
            buf = torch.empty(max(nbytes, 256) + 256, dtype=torch.uint8, device=device)
        _workspaces[key] = buf
    off = (-buf.data_ptr()) % 256
    return buf[off:off + max(nbytes, 256)]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _as_units(x: torch.Tensor, name: str) -> torch.Tensor:
    if x.dim() == 4:
        x = x.reshape(-1, x.shape[2], x.shape[3])
    if x.dim() != 3 or x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA bf16 [B,H,N,d] or [BH,N,d] tensor")
    return x


@dataclass
class MaskOut:
    kv_idx: torch.Tensor            # [BH, N_b, N_b] int32
    kv_cnt: torch.Tensor            # [BH, N_b] int32
    mask: torch.Tensor | None       # [BH, N_b, N_b] uint8
    p_imp: torch.Tensor | None      # [BH, N_b, N_b] fp32
    sample_idx: torch.Tensor | None # [BH, 2, N_b, k] int32
    n_refined: torch.Tensor         # [1] int32 (device)


def make_params(*, d: int, tau: float = 0.9, keep_min: int = 1, keep_max: int = 1 << 30,
                block: int = 128, samples: int = 16, scale: float | None = None, seed: int = 42,
                sample_mode: int = 0, share_qk: bool = False, unit_offset: int = 0,
                refine_guard: float = 0.0) -> BladeAsaParams:
    return BladeAsaParams(block, samples, tau, keep_min, keep_max,
                          default_scale(d) if scale is None else scale, seed & ((1 << 64) - 1),
                          sample_mode, int(bool(share_qk)), unit_offset, refine_guard, 0)


def blade_asa_mask(q: torch.Tensor, k: torch.Tensor, *, tau: float = 0.9, keep_min: int = 1,
                   keep_max: int = 1 << 30, block: int = 128, samples: int = 16,
                   scale: float | None = None, seed: int = 42, sample_mode: int = 0,
                   share_qk: bool = False, unit_offset: int = 0, refine_guard: float = 0.0,
                   want_mask: bool = True, want_pimp: bool = False, want_samples: bool = False,
                   sample_idx: torch.Tensor | None = None, out: MaskOut | None = None,
                   stream=None) -> MaskOut:
    """Alg. 1 on the GPU; see blade_asa.h for every argument."""
    q = _as_units(q, "q")
    k = _as_units(k, "k")
    BH, N, d = q.shape
    if k.shape != q.shape:
        raise ValueError("q and k shapes differ")
    prm = make_params(d=d, tau=tau, keep_min=keep_min, keep_max=keep_max, block=block,
                      samples=samples, scale=scale, seed=seed, sample_mode=sample_mode,
                      share_qk=share_qk, unit_offset=unit_offset, refine_guard=refine_guard)
    Nb = num_blocks(N, block)
    dev = q.device
    if out is None:
        if sample_mode == 2 and sample_idx is None:
            raise ValueError("sample_mode 2 needs sample_idx")
        out = MaskOut(
            kv_idx=torch.empty((BH, Nb, Nb), dtype=torch.int32, device=dev),
            kv_cnt=torch.empty((BH, Nb), dtype=torch.int32, device=dev),
            mask=torch.empty((BH, Nb, Nb), dtype=torch.uint8, device=dev) if want_mask else None,
            p_imp=torch.empty((BH, Nb, Nb), dtype=torch.float32, device=dev) if want_pimp else None,
            sample_idx=(sample_idx if sample_idx is not None else
                        torch.empty((BH, 2, Nb, samples), dtype=torch.int32, device=dev)
                        if want_samples else None),
            n_refined=torch.empty(1, dtype=torch.int32, device=dev))
    nbytes = _lib.blade_asa_mask_workspace_size(BH, N, d, ctypes.byref(prm))
    if nbytes == 0:  # let the call itself classify the arguments (no work is enqueued)
        st = _lib.blade_asa_mask(_ptr(q), _ptr(k), BH, N, d, ctypes.byref(prm), None,
                                 _ptr(out.kv_idx), _ptr(out.kv_cnt), None, None, None, None, 0,
                                 None)
        raise BladeError(st if st else BLADE_ERR_INVALID_ARG, "blade_asa_mask")
    ws = _workspace(nbytes, dev, "mask", stream)
    st = _lib.blade_asa_mask(_ptr(q), _ptr(k), BH, N, d, ctypes.byref(prm), _ptr(out.mask),
                             _ptr(out.kv_idx), _ptr(out.kv_cnt), _ptr(out.p_imp),
                             _ptr(out.sample_idx), _ptr(out.n_refined), _ptr(ws), ws.numel(),
                             _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_asa_mask")
    return out


def blade_bsa_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, kv_idx: torch.Tensor,
                  kv_cnt: torch.Tensor, *, scale: float | None = None, block: int = 128,
                  impl: int = ATTN_AUTO, want_lse: bool = True, o: torch.Tensor | None = None,
                  lse: torch.Tensor | None = None, stream=None):
    """Block-sparse attention forward over kept blocks -> (O, LSE)."""
    q = _as_units(q, "q")
    k = _as_units(k, "k")
    v = _as_units(v, "v")
    BH, N, d = q.shape
    Nb = num_blocks(N, block)
    for t, nm, shp in ((kv_idx, "kv_idx", (BH, Nb, Nb)), (kv_cnt, "kv_cnt", (BH, Nb))):
        if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous() or tuple(t.shape) != shp:
            raise ValueError(f"{nm} must be contiguous CUDA int32 of shape {shp}")
    if o is None:
        o = torch.empty_like(q)
    if lse is None and want_lse:
        lse = torch.empty((BH, N), dtype=torch.float32, device=q.device)
    nbytes = _lib.blade_bsa_fwd_workspace_size(BH, N, d, block)
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_bsa_fwd_workspace_size")
    ws = _workspace(nbytes, q.device, "attn", stream)
    st = _lib.blade_bsa_fwd(_ptr(q), _ptr(k), _ptr(v), BH, N, d, block,
                            default_scale(d) if scale is None else scale, _ptr(kv_idx),
                            _ptr(kv_cnt), _ptr(o), _ptr(lse), impl, _ptr(ws), ws.numel(),
                            _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_bsa_fwd")
    return o, lse


def blade_bsa_bwd(q, k, v, o, lse, do, kv_idx, kv_cnt, *, scale: float | None = None,
                  block: int = 128, dq=None, dk=None, dv=None, stream=None):
    """Gradients of the block-sparse attention -> (dQ, dK, dV) bf16."""
    q, k, v, o, do = (_as_units(x, n) for x, n in ((q, "q"), (k, "k"), (v, "v"), (o, "o"),
                                                    (do, "do")))
    BH, N, d = q.shape
    if lse.dtype != torch.float32 or not lse.is_cuda or tuple(lse.shape) != (BH, N):
        raise ValueError("lse must be CUDA fp32 [BH, N]")
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    nbytes = _lib.blade_bsa_bwd_workspace_size(BH, N, d, block)
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_bsa_bwd_workspace_size")
    ws = _workspace(nbytes, q.device, "bwd", stream)
    st = _lib.blade_bsa_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse.contiguous()), _ptr(do),
                            BH, N, d, block, default_scale(d) if scale is None else scale,
                            _ptr(kv_idx), _ptr(kv_cnt), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws),
                            ws.numel(), _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_bsa_bwd")
    return dq, dk, dv


def num_global_tokens(N: int, window: int) -> int:
    """N_g = ceil(N / n) (reading R-18)."""
    return (N + window - 1) // window


def blade_gt_pool(k: torch.Tensor, v: torch.Tensor, *, window: int = 128,
                  kg: torch.Tensor | None = None, vg: torch.Tensor | None = None, stream=None):
    """MeanPool_n of K and V -> (K_g, V_g) bf16 [BH, N_g, d]."""
    k = _as_units(k, "k")
    v = _as_units(v, "v")
    BH, N, d = k.shape
    Ng = num_global_tokens(N, window)
    if kg is None:
        kg = torch.empty((BH, Ng, d), dtype=torch.bfloat16, device=k.device)
    if vg is None:
        vg = torch.empty((BH, Ng, d), dtype=torch.bfloat16, device=k.device)
    st = _lib.blade_gt_pool(_ptr(k), _ptr(v), BH, N, d, window, _ptr(kg), _ptr(vg),
                            _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_gt_pool")
    return kg, vg


def blade_bsa_gt_fwd(q, k, v, kv_idx, kv_cnt, kg, vg, *, window: int = 128,
                     scale: float | None = None, block: int = 128, impl: int = ATTN_AUTO,
                     want_lse: bool = True, o=None, lse=None, stream=None):
    """ASA_GT attention: kept blocks plus every global token with the
    ln(n_w) bias, one softmax -> (O, LSE)."""
    q = _as_units(q, "q")
    k = _as_units(k, "k")
    v = _as_units(v, "v")
    BH, N, d = q.shape
    Ng = num_global_tokens(N, window)
    for t, nm in ((kg, "kg"), (vg, "vg")):
        if (t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous()
                or tuple(t.shape) != (BH, Ng, d)):
            raise ValueError(f"{nm} must be contiguous CUDA bf16 of shape {(BH, Ng, d)}")
    if o is None:
        o = torch.empty_like(q)
    if lse is None and want_lse:
        lse = torch.empty((BH, N), dtype=torch.float32, device=q.device)
    nbytes = _lib.blade_bsa_fwd_workspace_size(BH, N, d, block)
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_bsa_fwd_workspace_size")
    ws = _workspace(nbytes, q.device, "attn", stream)
    st = _lib.blade_bsa_gt_fwd(_ptr(q), _ptr(k), _ptr(v), BH, N, d, block,
                               default_scale(d) if scale is None else scale, _ptr(kv_idx),
                               _ptr(kv_cnt), _ptr(kg), _ptr(vg), window, _ptr(o), _ptr(lse),
                               impl, _ptr(ws), ws.numel(), _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_bsa_gt_fwd")
    return o, lse


def blade_bsa_gt_bwd(q, k, v, kg, vg, o, lse, do, kv_idx, kv_cnt, *, window: int = 128,
                     scale: float | None = None, block: int = 128, dq=None, dk=None, dv=None,
                     stream=None):
    """Gradients of ASA_GT attention (P:135 trained per P:158-161), through
    MeanPool_n to K and V -> (dQ, dK, dV) bf16."""
    q, k, v, o, do = (_as_units(x, n) for x, n in ((q, "q"), (k, "k"), (v, "v"), (o, "o"),
                                                    (do, "do")))
    kg, vg = _as_units(kg, "kg"), _as_units(vg, "vg")
    BH, N, d = q.shape
    if tuple(kg.shape) != (BH, num_global_tokens(N, window), d) or kg.shape != vg.shape:
        raise ValueError("kg, vg must be [BH, ceil(N/window), d]")
    if lse.dtype != torch.float32 or not lse.is_cuda or tuple(lse.shape) != (BH, N):
        raise ValueError("lse must be CUDA fp32 [BH, N]")
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    nbytes = _lib.blade_bsa_gt_bwd_workspace_size(BH, N, d, block, window)
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_bsa_gt_bwd_workspace_size")
    ws = _workspace(nbytes, q.device, "gt_bwd", stream)
    st = _lib.blade_bsa_gt_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(kg), _ptr(vg), window, _ptr(o),
                               _ptr(lse.contiguous()), _ptr(do), BH, N, d, block,
                               default_scale(d) if scale is None else scale, _ptr(kv_idx),
                               _ptr(kv_cnt), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(),
                               _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_bsa_gt_bwd")
    return dq, dk, dv


def asa_gt_forward(q, k, v, *, window: int = 128, tau: float = 0.9, keep_min: int = 1,
                   keep_max: int = 1 << 30, samples: int = 16, seed: int = 42,
                   unit_offset: int = 0, impl: int = ATTN_AUTO, stream=None, **mask_kw):
    """ASA_GT forward: MeanPool_n, mask generation (Alg. 1, unchanged by the
    global tokens, reading R-20), then attention.  Returns (O, LSE, MaskOut)."""
    kg, vg = blade_gt_pool(k, v, window=window, stream=stream)
    m = blade_asa_mask(q, k, tau=tau, keep_min=keep_min, keep_max=keep_max, samples=samples,
                       seed=seed, unit_offset=unit_offset, stream=stream, **mask_kw)
    o, lse = blade_bsa_gt_fwd(q, k, v, m.kv_idx, m.kv_cnt, kg, vg, window=window, impl=impl,
                              stream=stream)
    return o, lse, m


def gilbert_order(t: int, h: int, w: int, n_text: int = 0) -> torch.Tensor:
    """The Gilbert token order (blade_gilbert_order, computed on the host):
    int32 CPU tensor perm with perm[i] = raster index of the i-th token."""
    n = n_text + t * h * w
    perm = torch.empty(n, dtype=torch.int32)
    st = _lib.blade_gilbert_order(t, h, w, n_text, _ptr(perm), n)
    if st != BLADE_OK:
        raise BladeError(st, "blade_gilbert_order")
    return perm


def blade_permute_tokens(x: torch.Tensor, perm: torch.Tensor, *, inverse: bool = False,
                         out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Token-axis gather on the GPU: x[:, perm] (apply) or its inverse (undo)."""
    x = _as_units(x, "x")
    BH, N, d = x.shape
    if perm.dtype != torch.int32 or not perm.is_cuda or perm.numel() != N:
        raise ValueError("perm must be a CUDA int32 tensor of N entries")
    if out is None:
        out = torch.empty_like(x)
    st = _lib.blade_permute_tokens(_ptr(x), BH, N, d, _ptr(perm.contiguous()), int(inverse),
                                   _ptr(out), _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_permute_tokens")
    return out


def _as_host_units(x: torch.Tensor, name: str) -> torch.Tensor:
    if x.dim() == 4:
        x = x.reshape(-1, x.shape[2], x.shape[3])
    if x.dim() != 3 or x.dtype != torch.bfloat16 or x.is_cuda or not x.is_contiguous():
        raise ValueError(f"{name} must be a contiguous host (CPU) bf16 [B,H,N,d] or [BH,N,d] tensor")
    return x


def blade_asa_fwd_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, tau: float = 0.9,
                       keep_min: int = 1, keep_max: int = 1 << 30, samples: int = 16,
                       seed: int = 42, unit_offset: int = 0, impl: int = ATTN_AUTO,
                       chunk_units: int = 0, o: torch.Tensor | None = None,
                       lse: torch.Tensor | None = None, want_lse: bool = True,
                       kv_cnt: torch.Tensor | None = None, device: torch.device | None = None,
                       stream=None, **mask_kw):
    """The whole ASA forward on HOST (preferably pinned) tensors, chunked over
    units with copy/compute overlap (blade_asa_fwd_host).  Enqueued on
    ``stream`` of ``device``; outputs are valid once that stream completes.
    Returns (O, LSE) as host tensors."""
    q = _as_host_units(q, "q")
    k = _as_host_units(k, "k")
    v = _as_host_units(v, "v")
    BH, N, d = q.shape
    if k.shape != q.shape or v.shape != q.shape:
        raise ValueError("q, k, v shapes differ")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    prm = make_params(d=d, tau=tau, keep_min=keep_min, keep_max=keep_max, samples=samples,
                      seed=seed, unit_offset=unit_offset, **mask_kw)
    if o is None:
        o = torch.empty_like(q).pin_memory()
    if lse is None and want_lse:
        lse = torch.empty((BH, N), dtype=torch.float32).pin_memory()
    nbytes = _lib.blade_asa_fwd_host_workspace_size(BH, N, d, ctypes.byref(prm), chunk_units)
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_asa_fwd_host_workspace_size")
    ws = _workspace(nbytes, dev, "host", stream)
    st = _lib.blade_asa_fwd_host(_ptr(q), _ptr(k), _ptr(v), BH, N, d, ctypes.byref(prm), impl,
                                 chunk_units, _ptr(o), _ptr(lse), _ptr(kv_cnt), _ptr(ws),
                                 ws.numel(), _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_asa_fwd_host")
    return o, lse


def blade_asa_fwd(q, k, v, *, tau: float = 0.9, keep_min: int = 1, keep_max: int = 1 << 30,
                  samples: int = 16, seed: int = 42, unit_offset: int = 0, impl: int = ATTN_AUTO,
                  want_lse: bool = True, out=None, stream=None, **mask_kw):
    """The whole forward in one C call (mask, then attention launched as a
    programmatic dependent of the mask's fp64 refinement).  Returns
    (O, LSE, kv_idx, kv_cnt); ``out`` = (o, lse, kv_idx, kv_cnt) to reuse."""
    q = _as_units(q, "q")
    k = _as_units(k, "k")
    v = _as_units(v, "v")
    BH, N, d = q.shape
    prm = make_params(d=d, tau=tau, keep_min=keep_min, keep_max=keep_max, samples=samples,
                      seed=seed, unit_offset=unit_offset, **mask_kw)
    Nb = num_blocks(N)
    if out is None:
        out = (torch.empty_like(q),
               torch.empty((BH, N), dtype=torch.float32, device=q.device) if want_lse else None,
               torch.empty((BH, Nb, Nb), dtype=torch.int32, device=q.device),
               torch.empty((BH, Nb), dtype=torch.int32, device=q.device))
    o, lse, kv_idx, kv_cnt = out
    nbytes = _lib.blade_asa_fwd_workspace_size(BH, N, d, ctypes.byref(prm))
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_asa_fwd_workspace_size")
    ws = _workspace(nbytes, q.device, "fwd", stream)
    st = _lib.blade_asa_fwd(_ptr(q), _ptr(k), _ptr(v), BH, N, d, ctypes.byref(prm), impl,
                            _ptr(kv_idx), _ptr(kv_cnt), _ptr(o), _ptr(lse), _ptr(ws), ws.numel(),
                            _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_asa_fwd")
    return o, lse, kv_idx, kv_cnt


def blade_asa_gt_fwd(q, k, v, *, window: int = 128, tau: float = 0.9, keep_min: int = 1,
                     keep_max: int = 1 << 30, samples: int = 16, seed: int = 42,
                     unit_offset: int = 0, impl: int = ATTN_AUTO, want_lse: bool = True,
                     out=None, stream=None, **mask_kw):
    """The whole ASA_GT forward in one C call (MeanPool_n, mask, attention over
    the kept blocks and the global tokens as a programmatic dependent launch).
    Returns (O, LSE, kv_idx, kv_cnt, K_g, V_g); ``out`` = that tuple to reuse."""
    q = _as_units(q, "q")
    k = _as_units(k, "k")
    v = _as_units(v, "v")
    BH, N, d = q.shape
    prm = make_params(d=d, tau=tau, keep_min=keep_min, keep_max=keep_max, samples=samples,
                      seed=seed, unit_offset=unit_offset, **mask_kw)
    Nb, Ng = num_blocks(N), num_global_tokens(N, window)
    if out is None:
        out = (torch.empty_like(q),
               torch.empty((BH, N), dtype=torch.float32, device=q.device) if want_lse else None,
               torch.empty((BH, Nb, Nb), dtype=torch.int32, device=q.device),
               torch.empty((BH, Nb), dtype=torch.int32, device=q.device),
               torch.empty((BH, Ng, d), dtype=torch.bfloat16, device=q.device),
               torch.empty((BH, Ng, d), dtype=torch.bfloat16, device=q.device))
    o, lse, kv_idx, kv_cnt, kg, vg = out
    nbytes = _lib.blade_asa_fwd_workspace_size(BH, N, d, ctypes.byref(prm))
    if nbytes == 0:
        raise BladeError(BLADE_ERR_UNSUPPORTED, "blade_asa_fwd_workspace_size")
    ws = _workspace(nbytes, q.device, "fwd", stream)
    st = _lib.blade_asa_gt_fwd(_ptr(q), _ptr(k), _ptr(v), BH, N, d, ctypes.byref(prm), window,
                               impl, _ptr(kv_idx), _ptr(kv_cnt), _ptr(kg), _ptr(vg), _ptr(o),
                               _ptr(lse), _ptr(ws), ws.numel(), _stream(stream))
    if st != BLADE_OK:
        raise BladeError(st, "blade_asa_gt_fwd")
    return o, lse, kv_idx, kv_cnt, kg, vg


def asa_forward(q, k, v, *, tau: float = 0.9, keep_min: int = 1, keep_max: int = 1 << 30,
                samples: int = 16, seed: int = 42, unit_offset: int = 0,
                impl: int = ATTN_AUTO, stream=None, **mask_kw):
    """The whole ASA forward: mask generation then block-sparse attention.
    Returns (O, LSE, MaskOut)."""
    m = blade_asa_mask(q, k, tau=tau, keep_min=keep_min, keep_max=keep_max, samples=samples,
                       seed=seed, unit_offset=unit_offset, stream=stream, **mask_kw)
    o, lse = blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt, impl=impl, stream=stream)
    return o, lse, m
