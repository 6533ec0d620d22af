"""Plain fp64 CPU oracle for the ASA forward hot path (BLADE, arXiv 2508.10774).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or call
anything in ``oracle/``.  The product path (``paper_2508_10774_b200``) never
imports it and shares no code with it: no kernels, headers, helpers, tables or
constants.  The only thing both sides consume is the seeded input data made by
``paper_2508_10774_b200/inputs.py`` (which contains none of the method's
arithmetic).

Everything here follows the paper step by step, in its order and notation,
and is deliberately slow and unblocked.  Citations use ``P:<line>`` for
``PAPER.md`` lines and name the algorithm line; ``DESIGN.md §Readings`` lists
every reading taken where the paper is silent (R-1 ... R-16, mirroring
SURVEY §8(c) C-1 ... C-16).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  * sampler          - public splitmix64 outputs; survey KATs (tests/golden);
                       chi^2 uniformity; order-statistics rank law P:450-454.
  * probe (A4-A6)    - torch.softmax + torch max_pool2d on the sampled logits
                       (library routines); k=b exhaustive probe == dense
                       importance map P:117; uniform-logit factor b/k P:479;
                       Alg. 3 streaming form == two-pass form.
  * selection (A7-8) - SPEC worked examples; brute-force m0 with math.fsum;
                       numpy lexsort top-m; power-of-two scale invariance;
                       tau monotonicity; clamp safety.
  * attention (A9)   - torch scaled_dot_product_attention (fp64) with the
                       block mask expanded to a boolean token mask; LSE vs
                       torch.logsumexp; V=1 => O=1; V=0 => O=0; V=I => O=P.
  * composed mask    - asa_mask (Alg. 1) with k = b equals torch
                       dense softmax + max_pool2d(ceil_mode) followed
                       by a brute-force selection (math.fsum, numpy lexsort);
                       with k = 16 it equals the library probe on the
                       KAT-pinned samples of the global unit index followed
                       by the same selection (tests/test_oracle_mask_pin.py).
Every function of this module has at least one pin; none is "parity unpinned".
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# A1  block partition (Alg.1 l.2 "Partition Q, K into N_b = N/b blocks";
#     P:627 Alg.2 l.1 "Make length divisible by b: Pad").  Reading R-8: the pad
#     is logical; padded rows never enter sampling, softmax or attention.
# ---------------------------------------------------------------------------


def num_blocks(N: int, b: int) -> int:
    """N_b = ceil(N / b)  (T_r = ceil(S/b))."""
    return (N + b - 1) // b


def block_valid(N: int, b: int, i: int) -> int:
    """Number of real (un-padded) rows of block i."""
    return min(b, N - i * b)


def block_samples(N: int, b: int, k: int, i: int) -> int:
    """k_i = min(k, valid_i): a trailing block with fewer than k real rows
    contributes all of them (reading R-8)."""
    return min(k, block_valid(N, b, i))


# ---------------------------------------------------------------------------
# A2  random sampling of k tokens per block ("we sample k representative
#     tokens"; Alg.1 l.3 "Randomly sample k tokens from each block";
#     P:628-629 Alg.2 BlockSample).  The paper names no generator; reading R-1
#     fixes a counter-based hash so both implementations can replay it.
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def fmix64(z: int) -> int:
    """splitmix64 output finaliser (xor-shift 30, *0xBF58476D1CE4E5B9,
    xor-shift 27, *0x94D049BB133111EB, xor-shift 31), mod 2^64."""
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def sm(x: int, n: int) -> int:
    """sm(x, n) = fmix64(x + G*(n+1)): the n-th splitmix64 output of state x."""
    return fmix64((x + _GOLDEN * (n + 1)) & _M64)


def sample_key(seed: int, u: int, i: int, which: int) -> int:
    """Per-(unit, block, Q-or-K) stream key (reading R-1)."""
    return sm(sm(sm(seed & _M64, u), i), which)


def sample_offsets(seed: int, u: int, i: int, which: int, valid: int, k: int,
                   mode: int = 0) -> list[int]:
    """The in-block offsets sampled for block i of unit u, ascending.

    mode 0 (default, reading R-1): k_i = min(k, valid) distinct offsets,
      uniform without replacement: rank every offset o in [0, valid) by the
      pair (sm(key, o), o) and keep the k_i smallest.
    mode 1 (strided ablation): o_j = floor((2j+1)*valid/(2*k_i)).
    """
    k_i = min(k, valid)
    if mode == 1:
        return [((2 * j + 1) * valid) // (2 * k_i) for j in range(k_i)]
    if mode != 0:
        raise ValueError("mode must be 0 or 1 (mode 2 = caller-supplied)")
    key = sample_key(seed, u, i, which)
    ranked = sorted((sm(key, o), o) for o in range(valid))
    return sorted(o for _, o in ranked[:k_i])


# ---------------------------------------------------------------------------
# Parameters
# ---------------------------------------------------------------------------


@dataclass
class AsaParams:
    """The ABI parameter block, in plain Python (reading R-5/R-6 for tau and
    the clamps: integer keep_min/keep_max per row)."""

    block: int = 128          # b
    samples: int = 16         # k
    tau: float = 0.9          # threshold
    keep_min: int = 1         # lo           ("clamp m")
    keep_max: int = 1 << 30   # hi, clipped to N_b
    scale: float | None = None  # softmax scale; default fp32(1/sqrt(d)) (R-3)
    seed: int = 42            # P:603 Table 7 "Seed 42"
    sample_mode: int = 0      # 0 hash-random, 1 strided, 2 supplied
    share_qk: bool = False    # same offsets for Q and K
    unit_offset: int = 0      # global index of the first unit (sharding)


def default_scale(d: int) -> float:
    """fp32(1/sqrt(d)) widened to fp64 (reading R-3, "/ sqrt(d)")."""
    return float(np.float32(1.0 / math.sqrt(d)))


# ---------------------------------------------------------------------------
# A3-A6  probe: sampled attention and max-pool (Alg.1 l.4-5)
# ---------------------------------------------------------------------------


@dataclass
class UnitSamples:
    """Sampled row indices of one unit, block-major, ascending in each block."""

    rows_q: np.ndarray          # [N_k] absolute row index of each sampled query
    rows_k: np.ndarray          # [N_k] absolute row index of each sampled key
    blk_q: np.ndarray           # [N_k] block id of each sampled query row
    blk_k: np.ndarray           # [N_k] block id of each sampled key
    offsets_q: list = field(default_factory=list)   # per block, in-block offsets
    offsets_k: list = field(default_factory=list)


def draw_samples(N: int, p: AsaParams, u_global: int,
                 supplied: np.ndarray | None = None) -> UnitSamples:
    """BlockSample(Q_p, b, k) and BlockSample(K_p, b, k).

    ``supplied`` (mode 2) is an int array [2, N_b, k] of in-block offsets,
    -1 padded, [0] for Q and [1] for K."""
    b, k = p.block, p.samples
    Nb = num_blocks(N, b)
    oq, ok = [], []
    for i in range(Nb):
        valid = block_valid(N, b, i)
        if p.sample_mode == 2:
            k_i = block_samples(N, b, k, i)
            oq.append(sorted(int(x) for x in supplied[0, i, :k_i]))
            ok.append(sorted(int(x) for x in supplied[1, i, :k_i]))
        else:
            oq.append(sample_offsets(p.seed, u_global, i, 0, valid, k, p.sample_mode))
            ok.append(sample_offsets(p.seed, u_global, i, 0 if p.share_qk else 1,
                                     valid, k, p.sample_mode))
    rows_q = np.array([i * b + o for i in range(Nb) for o in oq[i]], dtype=np.int64)
    rows_k = np.array([i * b + o for i in range(Nb) for o in ok[i]], dtype=np.int64)
    blk_q = np.array([i for i in range(Nb) for _ in oq[i]], dtype=np.int64)
    blk_k = np.array([i for i in range(Nb) for _ in ok[i]], dtype=np.int64)
    return UnitSamples(rows_q, rows_k, blk_q, blk_k, oq, ok)


def row_softmax(L: np.ndarray) -> np.ndarray:
    """softmax over each row with the row max subtracted, fp64."""
    m = L.max(axis=1, keepdims=True)
    E = np.exp(L - m)
    return E / E.sum(axis=1, keepdims=True)


def probe_pimp(q_u: np.ndarray, k_u: np.ndarray, s: UnitSamples, Nb: int,
               scale: float) -> np.ndarray:
    """P_imp of one unit, two-pass definition.

    A3  Q_s, K_s = the sampled rows, block-major              (Alg.1 l.3)
    A4  L = Q_s K_s^T * scale  (fp64; bf16 products are exact) (Alg.1 l.4)
    A5  P~ = softmax(L) over all N_k sampled keys (reading R-2)
    A6  P_imp[i, j] = max over the k_i x k_j sub-block of P~   (Alg.1 l.5)
    """
    Qs = q_u[s.rows_q].astype(np.float64)
    Ks = k_u[s.rows_k].astype(np.float64)
    L = (Qs @ Ks.T) * scale
    Pt = row_softmax(L)
    # sampled rows are block-major, so block i owns one contiguous run of
    # rows (and block j one run of columns); every block has k_i >= 1 rows.
    q_starts = np.searchsorted(s.blk_q, np.arange(Nb))
    k_starts = np.searchsorted(s.blk_k, np.arange(Nb))
    row_max = np.maximum.reduceat(Pt, q_starts, axis=0)        # [Nb, N_k]
    return np.maximum.reduceat(row_max, k_starts, axis=1)      # [Nb, Nb]


def probe_pimp_streaming(q_u: np.ndarray, k_u: np.ndarray, s: UnitSamples,
                         Nb: int, scale: float) -> np.ndarray:
    """The same P_imp by Alg. 3 GetMaxPooledAttnMap, literally:
    running max M~, running sum l~, stash R~[:, j] = m_ij, then
    A[i, j] = max(e^{R~[:, j] - M~} / l~).  Used only to pin probe_pimp."""
    Qs = q_u[s.rows_q].astype(np.float64)
    Ks = k_u[s.rows_k].astype(np.float64)
    A = np.zeros((Nb, Nb), dtype=np.float64)
    for i in range(Nb):                                   # l.6
        Qi = Qs[s.blk_q == i]
        M = np.full(Qi.shape[0], -np.inf)                 # l.7  M~
        ell = np.zeros(Qi.shape[0])                       # l.8  l~
        R = np.full((Qi.shape[0], Nb), -np.inf)           # l.9  R~
        for j in range(Nb):                               # l.10
            Kj = Ks[s.blk_k == j]
            s_ij = (Qi @ Kj.T) * scale                    # l.11
            m_ij = s_ij.max(axis=1)                       # l.12
            P_ij = np.exp(s_ij - m_ij[:, None])
            l_ij = P_ij.sum(axis=1)                       # l.13
            m_new = np.maximum(M, m_ij)
            ell = np.exp(M - m_new) * ell + np.exp(m_ij - m_new) * l_ij  # l.14
            M = m_new                                     # l.15
            R[:, j] = m_ij
        for j in range(Nb):                               # l.17
            A[i, j] = (np.exp(R[:, j] - M) / ell).max()   # l.18-19
    return A


def dense_importance_map(q_u: np.ndarray, k_u: np.ndarray, b: int,
                         scale: float) -> np.ndarray:
    """The conceptual full importance: P = softmax(Q K^T / sqrt(d))
    over all N keys, then b x b max-pooling.  Only a test aid (pins the probe
    via k = b, P:117 vs P:146-147)."""
    N = q_u.shape[0]
    Nb = num_blocks(N, b)
    P = row_softmax((q_u.astype(np.float64) @ k_u.astype(np.float64).T) * scale)
    out = np.zeros((Nb, Nb))
    for i in range(Nb):
        for j in range(Nb):
            out[i, j] = P[i * b:(i + 1) * b, j * b:(j + 1) * b].max()
    return out


# ---------------------------------------------------------------------------
# A7-A8  selection and compaction (Alg.1 l.6-11)
# ---------------------------------------------------------------------------


@dataclass
class RowSelection:
    phat: np.ndarray      # normalised row
    order: list           # block ids, p-hat descending, ties by ascending id
    csum: list            # C_m for m = 1..N_b, sequential fp64 sums
    m0: int               # smallest m with C_m >= tau, else N_b
    m: int                # clamp(m0, lo, hi)
    kept: list            # kept block ids, ascending


def select_row(p_row: np.ndarray, tau: float, lo: int, hi: int) -> RowSelection:
    """One row of Alg. 1 l.7-10.

    l.7  p~_j = P_imp(i, j) / sum_k P_imp(i, k)   (sum ascending j, fp64)
    l.8  sort descending (reading R-7: ties -> lower block id first)
    l.9  smallest m with sum_{r<=m} s_r >= tau (reading R-4: '>=', Alg. 1,
         not 'exceed' of P:124; if never reached, m0 = N_b; tau = 1 gives
         m0 = N_b, "tau = 1 -> dense"), then clamp m to
         [lo, hi] (reading R-6: integer clamps)
    l.10 M[i, j] = 1 for the top m indices.
    """
    Nb = len(p_row)
    Z = 0.0
    for j in range(Nb):
        Z += float(p_row[j])
    phat = np.array([float(p_row[j]) / Z for j in range(Nb)])
    order = sorted(range(Nb), key=lambda j: (-phat[j], j))
    csum, c = [], 0.0
    for j in order:
        c += phat[j]
        csum.append(c)
    m0 = Nb
    if tau < 1.0:  # reading R-4: tau = 1 keeps all N_b blocks (exact mass of
        for r in range(Nb):  # positive scores reaches 1 only at N_b, whatever fp64 rounding says)
            if csum[r] >= tau:
                m0 = r + 1
                break
    m = min(max(m0, lo), hi)
    return RowSelection(phat, order, csum, m0, m, sorted(order[:m]))


def clamp_bounds(Nb: int, p: AsaParams) -> tuple[int, int]:
    """Integer clamps of Alg. 1 l.9 (reading R-6).  keep_min < 1 or
    keep_max < keep_min is an argument error (as at the C ABI); values above
    N_b clip to N_b."""
    if p.keep_min < 1 or p.keep_max < p.keep_min:
        raise ValueError(f"need 1 <= keep_min <= keep_max, got {p.keep_min}, {p.keep_max}")
    return min(p.keep_min, Nb), min(p.keep_max, Nb)


# ---------------------------------------------------------------------------
# Whole-unit and batched drivers
# ---------------------------------------------------------------------------


@dataclass
class MaskResult:
    mask: np.ndarray        # [BH, N_b, N_b] uint8
    kv_idx: np.ndarray      # [BH, N_b, N_b] int32, kept ascending, -1 tail
    kv_cnt: np.ndarray      # [BH, N_b] int32
    p_imp: np.ndarray       # [BH, N_b, N_b] fp64 raw max-pooled P_imp
    sample_idx: np.ndarray  # [BH, 2, N_b, k] int32 in-block offsets, -1 pad
    rows: list              # [BH][N_b] RowSelection


def to_f64(x) -> np.ndarray:
    """Widen bf16/fp32 torch or numpy data to fp64 exactly."""
    if hasattr(x, "detach"):
        x = x.detach().float().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def asa_mask(q, k, p: AsaParams, supplied_samples: np.ndarray | None = None,
             units: list | None = None) -> MaskResult:
    """Alg. 1 with Alg. 2/3 as the definition of
    P_imp, for every unit of q, k of shape [BH, N, d] (any float type;
    widened to fp64).  ``units`` restricts the work to a subset of local
    units (others are left zero / -1)."""
    q = to_f64(q)
    k = to_f64(k)
    BH, N, d = q.shape
    b, ks = p.block, p.samples
    Nb = num_blocks(N, b)
    scale = default_scale(d) if p.scale is None else float(p.scale)
    lo, hi = clamp_bounds(Nb, p)
    mask = np.zeros((BH, Nb, Nb), dtype=np.uint8)
    kv_idx = np.full((BH, Nb, Nb), -1, dtype=np.int32)
    kv_cnt = np.zeros((BH, Nb), dtype=np.int32)
    p_imp = np.zeros((BH, Nb, Nb), dtype=np.float64)
    sidx = np.full((BH, 2, Nb, ks), -1, dtype=np.int32)
    rows = [[None] * Nb for _ in range(BH)]
    for u in (range(BH) if units is None else units):
        sup = None if supplied_samples is None else supplied_samples[u]
        s = draw_samples(N, p, p.unit_offset + u, sup)
        for i in range(Nb):
            sidx[u, 0, i, :len(s.offsets_q[i])] = s.offsets_q[i]
            sidx[u, 1, i, :len(s.offsets_k[i])] = s.offsets_k[i]
        P = probe_pimp(q[u], k[u], s, Nb, scale)
        p_imp[u] = P
        for i in range(Nb):
            sel = select_row(P[i], float(p.tau), lo, hi)
            rows[u][i] = sel
            mask[u, i, sel.kept] = 1
            kv_idx[u, i, :sel.m] = sel.kept
            kv_cnt[u, i] = sel.m
    return MaskResult(mask, kv_idx, kv_cnt, p_imp, sidx, rows)


# ---------------------------------------------------------------------------
# A9  block-sparse attention ("binary sparse mask M is directly
#     integrated with a block-sparse attention kernel"); LSE by reading R-10.
# ---------------------------------------------------------------------------


def sparse_attention_unit(q_u, k_u, v_u, kv_idx_u, kv_cnt_u, b: int,
                          scale: float, qblocks=None):
    """For each query row r of q-block i:
        T     = union over kept j of [j*b, min((j+1)*b, N))
        LSE_r = ln sum_{t in T} exp(scale * q_r . k_t)
        O_r   = sum_{t in T} exp(scale * q_r . k_t - LSE_r) v_t
    in fp64.  Returns (O [N, d] fp64, LSE [N] fp64); rows of q-blocks not in
    ``qblocks`` are NaN."""
    q_u, k_u, v_u = to_f64(q_u), to_f64(k_u), to_f64(v_u)
    N, d = q_u.shape
    Nb = num_blocks(N, b)
    O = np.full((N, v_u.shape[1]), np.nan)
    LSE = np.full(N, np.nan)
    for i in (range(Nb) if qblocks is None else qblocks):
        r0, r1 = i * b, min((i + 1) * b, N)
        cols = np.concatenate([np.arange(j * b, min((j + 1) * b, N))
                               for j in kv_idx_u[i, :kv_cnt_u[i]]])
        S = (q_u[r0:r1] @ k_u[cols].T) * scale
        mx = S.max(axis=1, keepdims=True)
        E = np.exp(S - mx)
        ell = E.sum(axis=1, keepdims=True)
        O[r0:r1] = (E @ v_u[cols]) / ell
        LSE[r0:r1] = (mx + np.log(ell))[:, 0]
    return O, LSE


def sparse_attention(q, k, v, kv_idx, kv_cnt, b: int, scale: float | None = None,
                     units=None, qblocks=None):
    """A9 for [BH, N, d] inputs; returns fp64 O [BH, N, d], LSE [BH, N]."""
    q, k, v = to_f64(q), to_f64(k), to_f64(v)
    BH, N, d = q.shape
    scale = default_scale(d) if scale is None else float(scale)
    O = np.full(q.shape[:2] + (v.shape[2],), np.nan)
    LSE = np.full((BH, N), np.nan)
    for u in (range(BH) if units is None else units):
        O[u], LSE[u] = sparse_attention_unit(q[u], k[u], v[u], kv_idx[u],
                                             kv_cnt[u], b, scale, qblocks)
    return O, LSE


# ---------------------------------------------------------------------------
# Tie band (operational form of BASELINE.json's "bit-exact except where a
# block score lies within 1e-6 relative of the selection threshold"; reading
# R-14 / DESIGN.md §Tie band).
# ---------------------------------------------------------------------------


def tie_exemption(sel: RowSelection, tau: float, lo: int, hi: int,
                  eps: float = 1e-6) -> dict:
    """Classify one oracle row.  Returns {'exempt': bool, 'counts': set of
    accepted kv_cnt values, 'pivot_lo': p-hat lower bound for kept blocks,
    'pivot_hi': p-hat upper bound for dropped blocks}.

    T1 (cut ambiguity): |C_m' - tau| <= eps*tau for m' in {m0-1, m0} and the
        clamped count would change with the cut.
    T2 (membership ambiguity): m < N_b and p_(m) - p_(m+1) <= eps * p_(m).
    """
    Nb = len(sel.order)
    clamp = lambda x: min(max(x, lo), hi)
    counts = {sel.m}
    t1 = False
    for mp in ((sel.m0 - 1, sel.m0) if tau < 1.0 else ()):  # tau = 1: no cut (R-4)
        if 1 <= mp <= Nb and abs(sel.csum[mp - 1] - tau) <= eps * tau:
            for alt in (mp, mp + 1):
                if 1 <= alt <= Nb and clamp(alt) != sel.m:
                    counts.add(clamp(alt))
                    t1 = True
    sorted_p = [sel.phat[j] for j in sel.order]
    t2 = False
    for mm in counts:
        if mm < Nb and sorted_p[mm - 1] - sorted_p[mm] <= eps * sorted_p[mm - 1]:
            t2 = True
    return {"exempt": t1 or t2, "t1": t1, "t2": t2, "counts": counts,
            "sorted_p": sorted_p}


def check_row_against(sel: RowSelection, tau: float, lo: int, hi: int,
                      got_kept: list, eps: float = 1e-6) -> str | None:
    """Return None if a device row (its kept block ids) is acceptable for the
    oracle row ``sel`` under the tie band, else a reason string."""
    got_kept = sorted(int(j) for j in got_kept)
    if got_kept == sel.kept:
        return None
    te = tie_exemption(sel, tau, lo, hi, eps)
    if not te["exempt"]:
        return f"mismatch outside tie band: want {sel.kept} got {got_kept}"
    mm = len(got_kept)
    if mm not in te["counts"]:
        return f"count {mm} not in accepted {sorted(te['counts'])}"
    pivot = te["sorted_p"][mm - 1]
    kept = set(got_kept)
    for j in range(len(sel.phat)):
        pj = sel.phat[j]
        if j in kept and pj < (1 - eps) * pivot:
            return f"kept block {j} p={pj} below pivot {pivot}"
        if j not in kept and pj > (1 + eps) * pivot:
            return f"dropped block {j} p={pj} above pivot {pivot}"
    return None


# ---------------------------------------------------------------------------
# F1  ASA with global tokens, ASA_GT (P:135 Step 2.2 (2); Fig. 2
#     caption): K_aug = Concat(K, MeanPool_n(K)), V_aug likewise; the
#     original region keeps the binary block mask M, the pooled region
#     ("global tokens") is attended by every query with a fixed additive
#     pre-softmax bias ln(n).  Readings:
#       R-18  windows are consecutive runs of n tokens [w n, min((w+1) n, N));
#             N_g = ceil(N / n); a partial last window is the mean of its
#             n_w < n real tokens and carries bias ln(n_w) (= ln n for every
#             full window, "as if it represents the full importance of
#             its n constituent fine-grained tokens").
#       R-19  K_aug / V_aug are tensors of the input dtype (Concat needs one
#             dtype), so the pooled rows are the exact means rounded once to
#             bf16 (round-to-nearest-even).
#       R-20  the mask M (Alg. 1) is computed from Q and K only, unchanged;
#             global tokens join the same softmax, so LSE includes them.
# ---------------------------------------------------------------------------


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp64 values to the nearest bf16 value (8 significant bits, ties
    to even), returned as fp64.  One rounding step (no fp32 detour); bf16
    normal range only (|x| >= 2^-126 or 0), which the pooled means of bf16
    inputs of realistic size never leave."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                 # x = m 2^e, 0.5 <= |m| < 1
    r = np.round(m * 256.0)            # 8 significant bits; numpy rounds half to even
    return np.ldexp(r, e - 8)


def mean_pool_windows(x_u: np.ndarray, n: int):
    """MeanPool_n over the token axis (reading R-18): returns the
    pooled rows [N_g, d] (exact fp64 means, NOT yet rounded) and the window
    sizes n_w [N_g]."""
    x_u = to_f64(x_u)
    N = x_u.shape[0]
    Ng = (N + n - 1) // n
    pooled = np.empty((Ng, x_u.shape[1]))
    counts = np.empty(Ng, dtype=np.int64)
    for w in range(Ng):
        rows = x_u[w * n:min((w + 1) * n, N)]
        counts[w] = rows.shape[0]
        pooled[w] = rows.sum(axis=0) / rows.shape[0]
    return pooled, counts


def global_tokens(k_u, v_u, n: int):
    """The ASA_GT global tokens of one unit: (K_g, V_g, bias) with K_g, V_g
    the bf16-rounded window means (R-19) and bias_w = ln(n_w) (R-18)."""
    kg, counts = mean_pool_windows(k_u, n)
    vg, _ = mean_pool_windows(v_u, n)
    return round_to_bf16(kg), round_to_bf16(vg), np.log(counts.astype(np.float64))


def sparse_attention_gt_unit(q_u, k_u, v_u, kv_idx_u, kv_cnt_u, b: int, scale: float,
                             n: int, qblocks=None):
    """ASA_GT attention of one unit, fp64.  For query row r of q-block i:
        T     = union over kept j of [j*b, min((j+1)*b, N))     (mask M)
        s_t   = scale * q_r . k_t                 for t in T
        g_w   = scale * q_r . K_g[w] + ln(n_w)    for every window w
        LSE_r = ln( sum_{t in T} e^{s_t} + sum_w e^{g_w} )
        O_r   = sum_{t in T} e^{s_t - LSE_r} v_t + sum_w e^{g_w - LSE_r} V_g[w]
    Returns (O [N, d], LSE [N]); rows of q-blocks not in ``qblocks`` are NaN."""
    q_u, k_u, v_u = to_f64(q_u), to_f64(k_u), to_f64(v_u)
    N, d = q_u.shape
    Nb = num_blocks(N, b)
    kg, vg, bias = global_tokens(k_u, v_u, n)
    O = np.full((N, v_u.shape[1]), np.nan)
    LSE = np.full(N, np.nan)
    for i in (range(Nb) if qblocks is None else qblocks):
        r0, r1 = i * b, min((i + 1) * b, N)
        cols = np.concatenate([np.arange(j * b, min((j + 1) * b, N))
                               for j in kv_idx_u[i, :kv_cnt_u[i]]])
        S = (q_u[r0:r1] @ k_u[cols].T) * scale
        G = (q_u[r0:r1] @ kg.T) * scale + bias[None, :]
        A = np.concatenate([S, G], axis=1)
        Vaug = np.concatenate([v_u[cols], vg], axis=0)
        mx = A.max(axis=1, keepdims=True)
        E = np.exp(A - mx)
        ell = E.sum(axis=1, keepdims=True)
        O[r0:r1] = (E @ Vaug) / ell
        LSE[r0:r1] = (mx + np.log(ell))[:, 0]
    return O, LSE


def sparse_attention_gt(q, k, v, kv_idx, kv_cnt, b: int, n: int, scale: float | None = None,
                        units=None, qblocks=None):
    """ASA_GT attention for [BH, N, d] inputs; fp64 O [BH, N, d], LSE [BH, N]."""
    q, k, v = to_f64(q), to_f64(k), to_f64(v)
    BH, N, d = q.shape
    scale = default_scale(d) if scale is None else float(scale)
    O = np.full(q.shape[:2] + (v.shape[2],), np.nan)
    LSE = np.full((BH, N), np.nan)
    for u in (range(BH) if units is None else units):
        O[u], LSE[u] = sparse_attention_gt_unit(q[u], k[u], v[u], kv_idx[u], kv_cnt[u], b,
                                                scale, n, qblocks)
    return O, LSE


# ---------------------------------------------------------------------------
# F2  locality-preserving token rearrangement ("we employ a Gilbert
#     space-filling curve to reorder the tokens before blocking"; Alg. 1 l.1
#     P:143 "Rearrange tokens using Gilbert curve").  Readings:
#       R-21  the paper does not say 2-D or 3-D: each frame's h x w patch grid
#             is ordered by the 2-D generalised Hilbert ("Gilbert") curve,
#             frames stay in temporal order (frame-major), so every 128-token
#             block is a compact patch of one frame and the curve keeps exact
#             4-neighbour adjacency inside a frame;
#       R-22  leading text tokens (CogVideoX) keep their positions.
#     The curve is the recursive construction for arbitrary rectangles: split
#     the long side in two when the rectangle is more than 1.5x longer than
#     wide, else cut it into three parts (one step along the short side, the
#     long run, one step back), halves rounded so the sub-rectangles' major
#     sides are even where possible, which is what keeps consecutive cells
#     adjacent.  This is the published generalised-Hilbert ("gilbert2d")
#     recursion of J. Cerveny (github.com/jakubcerveny/gilbert, BSD-2-Clause),
#     the curve the paper names; it is pinned by the curve's
#     properties (tests/test_oracle_gilbert.py), not by the CUDA side, which
#     implements the same published recursion.
# ---------------------------------------------------------------------------


def _sgn(x: int) -> int:
    return (x > 0) - (x < 0)


def gilbert2d_cells(width: int, height: int) -> list:
    """(x, y) cells of a width x height grid in Gilbert-curve order, starting
    at (0, 0) and running along the longer side."""
    out = []

    def walk(x, y, ax, ay, bx, by):
        w, h = abs(ax + ay), abs(bx + by)
        dax, day, dbx, dby = _sgn(ax), _sgn(ay), _sgn(bx), _sgn(by)
        if h == 1:                      # a single row: walk it
            for _ in range(w):
                out.append((x, y))
                x, y = x + dax, y + day
            return
        if w == 1:                      # a single column
            for _ in range(h):
                out.append((x, y))
                x, y = x + dbx, y + dby
            return
        ax2, ay2, bx2, by2 = ax // 2, ay // 2, bx // 2, by // 2
        w2, h2 = abs(ax2 + ay2), abs(bx2 + by2)
        if 2 * w > 3 * h:               # long rectangle: two halves along the major axis
            if (w2 % 2) and (w > 2):
                ax2, ay2 = ax2 + dax, ay2 + day
            walk(x, y, ax2, ay2, bx, by)
            walk(x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by)
        else:                           # up, across, down
            if (h2 % 2) and (h > 2):
                bx2, by2 = bx2 + dbx, by2 + dby
            walk(x, y, bx2, by2, ax2, ay2)
            walk(x + bx2, y + by2, ax, ay, bx - bx2, by - by2)
            walk(x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby),
                 -bx2, -by2, -(ax - ax2), -(ay - ay2))

    if width >= height:                 # major axis x (length width), minor y
        walk(0, 0, width, 0, 0, height)
    else:                               # major axis y (length height), minor x
        walk(0, 0, 0, height, width, 0)
    return out


def gilbert_permutation(t: int, h: int, w: int, n_text: int = 0) -> np.ndarray:
    """perm[i] = raster index (text tokens first, then t-major, y, x) of the
    token placed at position i of the rearranged sequence (R-21, R-22)."""
    if min(t, h, w) < 1 or n_text < 0:
        raise ValueError("grid extents must be positive")
    cells = gilbert2d_cells(w, h)       # (x, y) along the frame
    frame = np.array([y * w + x for x, y in cells], dtype=np.int64)
    perm = [np.arange(n_text, dtype=np.int64)]
    for f in range(t):
        perm.append(n_text + f * h * w + frame)
    return np.concatenate(perm)


def apply_permutation(x, perm: np.ndarray) -> np.ndarray:
    """x'[.., i, :] = x[.., perm[i], :] (token axis = -2)."""
    return np.asarray(x)[..., perm, :]


def undo_permutation(x, perm: np.ndarray) -> np.ndarray:
    """Inverse of apply_permutation: y[.., perm[i], :] = x[.., i, :]."""
    x = np.asarray(x)
    y = np.empty_like(x)
    y[..., perm, :] = x
    return y


# ---------------------------------------------------------------------------
# F3  block-sparse attention backward (the student "generates its
#     trajectory using the ASA mechanism" and the loss "updates the student's
#     weights ... given these dynamic sparsity constraints", so gradients flow
#     through the masked attention of A9).  The vector-Jacobian product of
#     O = softmax_T(scale Q K^T) V restricted to the kept blocks T(r):
#       P_rt  = exp(scale q_r.k_t - LSE_r)             t in T(r), else 0
#       dV_t  = sum_r P_rt dO_r
#       dP_rt = dO_r . v_t
#       D_r   = sum_t P_rt dP_rt  (= dO_r . O_r)
#       dS_rt = P_rt (dP_rt - D_r)
#       dQ_r  = scale sum_t dS_rt k_t,   dK_t = scale sum_r dS_rt q_r
#     The mask M is a constant of the backward (Alg. 1's selection is not
#     differentiated; reading R-23).
# ---------------------------------------------------------------------------


def sparse_attention_backward_unit(q_u, k_u, v_u, do_u, kv_idx_u, kv_cnt_u, b: int,
                                   scale: float):
    """fp64 (dQ, dK, dV) of one unit, query block by query block."""
    q_u, k_u, v_u, do_u = to_f64(q_u), to_f64(k_u), to_f64(v_u), to_f64(do_u)
    N, d = q_u.shape
    Nb = num_blocks(N, b)
    dq, dk, dv = np.zeros_like(q_u), np.zeros_like(k_u), np.zeros_like(v_u)
    for i in range(Nb):
        r0, r1 = i * b, min((i + 1) * b, N)
        cols = np.concatenate([np.arange(j * b, min((j + 1) * b, N))
                               for j in kv_idx_u[i, :kv_cnt_u[i]]])
        S = (q_u[r0:r1] @ k_u[cols].T) * scale
        mx = S.max(axis=1, keepdims=True)
        E = np.exp(S - mx)
        P = E / E.sum(axis=1, keepdims=True)
        dO = do_u[r0:r1]
        dv[cols] += P.T @ dO
        dP = dO @ v_u[cols].T
        Dr = (P * dP).sum(axis=1, keepdims=True)
        dS = P * (dP - Dr)
        dq[r0:r1] += scale * (dS @ k_u[cols])
        dk[cols] += scale * (dS.T @ q_u[r0:r1])
    return dq, dk, dv


def sparse_attention_backward(q, k, v, do, kv_idx, kv_cnt, b: int, scale: float | None = None,
                              units=None):
    """F3 for [BH, N, d]: fp64 dQ, dK, dV (units not listed are NaN)."""
    q, k, v, do = to_f64(q), to_f64(k), to_f64(v), to_f64(do)
    scale = default_scale(q.shape[2]) if scale is None else float(scale)
    dq, dk, dv = (np.full(q.shape, np.nan) for _ in range(3))
    for u in (range(q.shape[0]) if units is None else units):
        dq[u], dk[u], dv[u] = sparse_attention_backward_unit(q[u], k[u], v[u], do[u], kv_idx[u],
                                                             kv_cnt[u], b, scale)
    return dq, dk, dv


def sparse_attention_gt_backward_unit(q_u, k_u, v_u, do_u, kv_idx_u, kv_cnt_u, b: int,
                                      scale: float, n: int):
    """fp64 (dQ, dK, dV) of ASA_GT attention (F1 + F3).
    The global tokens are K_g = round_bf16(MeanPool_n(K)) (R-19); the
    gradient passes through the mean (each token of window w receives 1/n_w
    of the pooled token's gradient) and through the bf16 rounding as the
    identity (straight-through: rounding has zero derivative almost
    everywhere, the training recipe treats K_aug as a function of K).  The
    mask is a constant (R-23).  Per query block i, with T = kept keys:
      A = [scale q K_T^T, scale q K_g^T + ln n_w],  P = softmax(A)
      dV_T += P_T^T dO,   dV_g = P_g^T dO
      dP = dO [V_T; V_g]^T,  dS = P (dP - rowsum(P dP))
      dQ += scale dS [K_T; K_g],  dK_T += scale dS_T^T q,  dK_g = scale dS_g^T q
    then dK[t] += dK_g[w(t)] / n_w, dV[t] += dV_g[w(t)] / n_w."""
    q_u, k_u, v_u, do_u = to_f64(q_u), to_f64(k_u), to_f64(v_u), to_f64(do_u)
    N, d = q_u.shape
    Nb = num_blocks(N, b)
    kg, vg, bias = global_tokens(k_u, v_u, n)
    Ng = kg.shape[0]
    dq, dk, dv = np.zeros_like(q_u), np.zeros_like(k_u), np.zeros_like(v_u)
    dkg, dvg = np.zeros((Ng, d)), np.zeros((Ng, d))
    for i in range(Nb):
        r0, r1 = i * b, min((i + 1) * b, N)
        cols = np.concatenate([np.arange(j * b, min((j + 1) * b, N))
                               for j in kv_idx_u[i, :kv_cnt_u[i]]])
        Kaug = np.concatenate([k_u[cols], kg], axis=0)
        Vaug = np.concatenate([v_u[cols], vg], axis=0)
        A = (q_u[r0:r1] @ Kaug.T) * scale
        A[:, len(cols):] += bias[None, :]
        P = np.exp(A - A.max(axis=1, keepdims=True))
        P /= P.sum(axis=1, keepdims=True)
        dO = do_u[r0:r1]
        dVaug = P.T @ dO
        dP = dO @ Vaug.T
        dS = P * (dP - (P * dP).sum(axis=1, keepdims=True))
        dq[r0:r1] += scale * (dS @ Kaug)
        dKaug = scale * (dS.T @ q_u[r0:r1])
        dk[cols] += dKaug[:len(cols)]
        dv[cols] += dVaug[:len(cols)]
        dkg += dKaug[len(cols):]
        dvg += dVaug[len(cols):]
    w_of = np.arange(N) // n
    counts = np.bincount(w_of, minlength=Ng).astype(np.float64)
    dk += dkg[w_of] / counts[w_of, None]
    dv += dvg[w_of] / counts[w_of, None]
    return dq, dk, dv


def sparse_attention_gt_backward(q, k, v, do, kv_idx, kv_cnt, b: int, n: int,
                                 scale: float | None = None, units=None):
    """F1 + F3 for [BH, N, d]: fp64 dQ, dK, dV of ASA_GT (units not listed are NaN)."""
    q, k, v, do = to_f64(q), to_f64(k), to_f64(v), to_f64(do)
    scale = default_scale(q.shape[2]) if scale is None else float(scale)
    dq, dk, dv = (np.full(q.shape, np.nan) for _ in range(3))
    for u in (range(q.shape[0]) if units is None else units):
        dq[u], dk[u], dv[u] = sparse_attention_gt_backward_unit(
            q[u], k[u], v[u], do[u], kv_idx[u], kv_cnt[u], b, scale, n)
    return dq, dk, dv
