"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no sampling, probing,
selection or attention).  It only makes Q, K, V tensors with the shapes of
the paper's workloads (Table 7) and a documented value
distribution, so that ``oracle/`` and the CUDA path can
be fed identical bf16 data without sharing any code.

Recipes
-------
* ``iid``     Q, K, V ~ N(0, 1) iid.
* ``smooth``  a random-Fourier-feature field over the video token grid
              (t, y, x) ("spatially contiguous information"):
              F = sqrt(2/D) cos(pos W + phi), W ~ N(0, 1/ell^2) per axis,
              Q = beta F + sigma_n eps_q, K = beta F + sigma_n eps_k,
              V ~ N(0, 1); a leading block of ``n_text`` iid "text" tokens
              (CogVideoX: 226, BASELINE.json configs[2]).  Logits are then
              ~ beta^2/sqrt(d) * exp(-|dpos|^2 / 2 ell^2): localised
              attention, so tau-mode masks are sparse as in the paper.
* ``const``   constant rows (exact ties everywhere; adversarial).
* ``spike``   iid plus one key row of large norm aligned with all queries.

All draws use numpy's PCG64 with an explicit seed; values are rounded to
bf16 exactly once (torch round-to-nearest-even) and both sides read those
bf16 values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class Workload:
    name: str
    B: int
    H: int
    N: int
    d: int
    grid: tuple | None = None     # (t, y, x) video-token grid, t*y*x = N - n_text
    n_text: int = 0
    ell: float = 3.0              # smooth-field length scale, in tokens
    beta: float = 9.0             # smooth-field amplitude
    sigma_n: float = 0.1          # smooth-field noise


# BASELINE.json configs (shapes from P:582-588 Table 7; P:605 480x832).
WORKLOADS = {
    "tiny": Workload("tiny", 1, 1, 512, 64, grid=(1, 16, 32)),
    # 21 latent frames x 30 x 52 patches = 32760 (P:588, P:590 patch [1,2,2])
    "wan": Workload("wan2.1-1.3b-layer", 1, 12, 32760, 128, grid=(21, 30, 52),
                    beta=9.25),
    # 226 text + 13 x 30 x 45 = 17550 video tokens (BASELINE.json)
    "cog": Workload("cogvideox-5b-layer", 1, 48, 17776, 64, grid=(13, 30, 45),
                    n_text=226, beta=8.5),
    "wan_stack": Workload("wan2.1-1.3b-stack-b8", 8, 12, 32760, 128,
                          grid=(21, 30, 52), beta=9.25),
}


def _to_bf16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)


def iid(B: int, H: int, N: int, d: int, seed: int = 42):
    """Q, K, V ~ N(0, 1), bf16, shape [B*H, N, d] (contiguous units)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (B * H, N, d)
    return tuple(_to_bf16(rng.standard_normal(shape, dtype=np.float32)) for _ in range(3))


def grid_positions(grid: tuple) -> np.ndarray:
    """Raster-order (t, y, x) coordinates of a video token grid, [t*y*x, 3]."""
    t, y, x = grid
    tt, yy, xx = np.meshgrid(np.arange(t), np.arange(y), np.arange(x), indexing="ij")
    return np.stack([tt.ravel(), yy.ravel(), xx.ravel()], axis=1).astype(np.float32)


def smooth(B: int, H: int, N: int, d: int, grid: tuple, n_text: int = 0,
           ell: float = 3.0, beta: float = 9.0, sigma_n: float = 0.1,
           seed: int = 42):
    """Smooth-field Q, K and iid V, bf16 [B*H, N, d] (recipe in module doc)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pos = grid_positions(grid)
    assert pos.shape[0] + n_text == N, (grid, n_text, N)
    BH = B * H
    q = np.empty((BH, N, d), np.float32)
    k = np.empty((BH, N, d), np.float32)
    for u in range(BH):
        W = rng.standard_normal((3, d), dtype=np.float32) / np.float32(ell)
        phi = rng.uniform(0, 2 * np.pi, size=d).astype(np.float32)
        F = np.sqrt(np.float32(2.0 / d)) * np.cos(pos @ W + phi)
        if n_text:
            T = rng.standard_normal((n_text, d), dtype=np.float32) / np.sqrt(np.float32(d))
            F = np.concatenate([T, F], axis=0)
        q[u] = beta * F + sigma_n * rng.standard_normal((N, d), dtype=np.float32)
        k[u] = beta * F + sigma_n * rng.standard_normal((N, d), dtype=np.float32)
    v = rng.standard_normal((BH, N, d), dtype=np.float32)
    return _to_bf16(q), _to_bf16(k), _to_bf16(v)


def const(BH: int, N: int, d: int, value: float = 0.5, seed: int = 42):
    """Q = K = constant (every logit equal: exact ties), V iid."""
    rng = np.random.Generator(np.random.PCG64(seed))
    q = np.full((BH, N, d), value, np.float32)
    v = rng.standard_normal((BH, N, d), dtype=np.float32)
    return _to_bf16(q), _to_bf16(q.copy()), _to_bf16(v)


def spike(BH: int, N: int, d: int, seed: int = 42, row: int | None = None,
          amp: float = 4.0):
    """iid Q, K, V plus one key row = amp * sum of mean query direction."""
    q, k, v = (t.float().numpy() for t in iid(1, BH, N, d, seed))
    r = N // 2 if row is None else row
    for u in range(BH):
        dirn = q[u].mean(axis=0)
        k[u, r] = amp * dirn / (np.linalg.norm(dirn) + 1e-6) * np.sqrt(d)
    return _to_bf16(q), _to_bf16(k), _to_bf16(v)


def make(workload: str | Workload, recipe: str = "smooth", seed: int = 42,
         B: int | None = None):
    """Inputs for a named workload; returns (q, k, v) bf16 CPU [B*H, N, d]."""
    w = WORKLOADS[workload] if isinstance(workload, str) else workload
    Bv = w.B if B is None else B
    if recipe == "iid":
        return iid(Bv, w.H, w.N, w.d, seed)
    if recipe == "smooth":
        return smooth(Bv, w.H, w.N, w.d, w.grid, w.n_text, w.ell, w.beta,
                      w.sigma_n, seed)
    raise ValueError(recipe)


def unit_seed(base: int, u_global: int) -> int:
    """Seed of one (batch, head) unit: a function of the GLOBAL unit index
    only, so every sharding of a batch draws identical tensors per unit."""
    return (base * 1_000_003 + u_global) & ((1 << 63) - 1)


def smooth_device(units, N: int, d: int, grid: tuple, device, n_text: int = 0,
                  ell: float = 3.0, beta: float = 9.0, sigma_n: float = 0.1, seed: int = 42):
    """The ``smooth`` recipe drawn with torch's CUDA generator directly on the
    device (same distribution, different stream of random numbers than the
    numpy version), for workloads too large to generate on the host (the
    30-layer batch-8 stack, BASELINE.json configs[4]).  ``units`` is the range
    (or list) of GLOBAL unit indices to draw; unit u uses its own generator
    seeded with ``unit_seed(seed, u)``, so a rank drawing units [lo, hi) gets
    exactly the slice a single-GPU run draws.  Returns bf16 [len(units), N, d]
    q, k, v on ``device``."""
    if isinstance(units, int):
        units = range(units)
    units = list(units)
    g = torch.Generator(device=device)
    pos = torch.from_numpy(grid_positions(grid)).to(device)
    q = torch.empty((len(units), N, d), dtype=torch.bfloat16, device=device)
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    for n, u in enumerate(units):
        g.manual_seed(unit_seed(seed, u))
        W = torch.randn((3, d), generator=g, device=device) / ell
        phi = torch.rand(d, generator=g, device=device) * (2 * np.pi)
        F = (2.0 / d) ** 0.5 * torch.cos(pos @ W + phi)
        if n_text:
            T = torch.randn((n_text, d), generator=g, device=device) / d ** 0.5
            F = torch.cat([T, F], 0)
        q[n] = beta * F + sigma_n * torch.randn((N, d), generator=g, device=device)
        k[n] = beta * F + sigma_n * torch.randn((N, d), generator=g, device=device)
        v[n] = torch.randn((N, d), generator=g, device=device)
    return q, k, v
