"""Shared comparison helpers for the GPU parity tests (CUDA path vs oracle)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import asa_oracle as O

# BASELINE.json north_star tolerances for bf16 inputs
O_MAX_ABS = 2e-2
O_MEAN_ABS = 2e-3
LSE_ABS = 1e-3
TIE_EPS = 1e-6


def oracle_params(**kw) -> O.AsaParams:
    return O.AsaParams(**kw)


def check_mask(ref: O.MaskResult, got, p: O.AsaParams, units=None) -> dict:
    """Bit-exact kv lists / counts / mask outside the tie band (T1/T2),
    tie-band-valid inside it.  Returns stats."""
    kv_idx = got.kv_idx.cpu().numpy()
    kv_cnt = got.kv_cnt.cpu().numpy()
    mask = got.mask.cpu().numpy() if got.mask is not None else None
    BH, Nb, _ = kv_idx.shape
    lo, hi = O.clamp_bounds(Nb, p)
    exempt = mismatched_exempt = 0
    for u in (range(BH) if units is None else units):
        for i in range(Nb):
            sel = ref.rows[u][i]
            c = int(kv_cnt[u, i])
            kept = kv_idx[u, i, :c].tolist()
            assert (kv_idx[u, i, c:] == -1).all(), (u, i)
            assert kept == sorted(set(kept)), (u, i, kept)
            assert lo <= c <= hi, (u, i, c)
            if mask is not None:
                assert set(np.flatnonzero(mask[u, i]).tolist()) == set(kept), (u, i)
            te = O.tie_exemption(sel, float(p.tau), lo, hi, TIE_EPS)
            exempt += te["exempt"]
            why = O.check_row_against(sel, float(p.tau), lo, hi, kept, TIE_EPS)
            assert why is None, f"unit {u} row {i}: {why}"
            mismatched_exempt += kept != sel.kept
    return {"rows": (BH if units is None else len(units)) * Nb, "exempt": exempt,
            "exempt_differing": mismatched_exempt}


def check_attention(o_gpu, lse_gpu, o_ref, lse_ref, rows_mask=None) -> dict:
    """O: max abs <= 2e-2 and mean abs <= 2e-3; LSE: abs <= 1e-3."""
    o = o_gpu.float().cpu().numpy().astype(np.float64)
    lse = lse_gpu.cpu().numpy().astype(np.float64)
    sel = ~np.isnan(lse_ref) if rows_mask is None else rows_mask
    err = np.abs(o[sel] - o_ref[sel])
    lerr = np.abs(lse[sel] - lse_ref[sel])
    stats = {"o_max": float(err.max()), "o_mean": float(err.mean()),
             "lse_max": float(lerr.max()), "rows": int(sel.sum())}
    assert np.isfinite(o[sel]).all() and np.isfinite(lse[sel]).all()
    assert stats["o_max"] <= O_MAX_ABS, stats
    assert stats["o_mean"] <= O_MEAN_ABS, stats
    assert stats["lse_max"] <= LSE_ABS, stats
    return stats


def to_dev(*ts, device="cuda"):
    return [t.to(device).contiguous() for t in ts]


def lists_to_dev(kv_idx: np.ndarray, kv_cnt: np.ndarray, device="cuda"):
    return (torch.from_numpy(np.ascontiguousarray(kv_idx, np.int32)).to(device),
            torch.from_numpy(np.ascontiguousarray(kv_cnt, np.int32)).to(device))
