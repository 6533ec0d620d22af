// select.cuh — one warp selects one row: PAPER.md Alg. 1 l.7-10.
//
//   l.7   p~_j = P_imp(i,j) / sum_k P_imp(i,k)                (fp64)
//   l.8   sort p~ descending, ties by ascending block id       (reading R-7)
//   l.9   m0 = smallest m with sum_{r<=m} s_r >= tau, else N_b; N_b for tau = 1 (R-4),
//         m  = clamp(m0, lo, hi)                               (reading R-6)
//   l.10  M[i, j] = 1 for the top m; compacted to ascending kv_idx
//
// The row lives in registers: a bitonic sort of P2 = 32*E (value, id) pairs,
// E per lane in lane-major order (position x = lane*E + e), so distances < E
// are in-register exchanges and larger ones are warp shuffles.  The sorted
// row is then lane-contiguous, which makes the cumulative sum a per-lane
// prefix plus one warp scan.  Returns whether the decision margin lies inside
// the refinement guard band (reading R-14).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

#ifndef BLADE_SEL_TOPK
#define BLADE_SEL_TOPK 1  // keep-ratio rows by a bitwise top-m search instead of a sort
#endif

namespace blade {

BLADE_DEVINL bool sel_before(double va, int ia, double vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

template <int E, typename T>
struct RowSelect {
  // vals: row values by block id (fp32 P_imp from the probe, or fp64 refined
  // values; any address space), Nb <= 32*E.  mask_row may be null.
  // keep_bits: shared-memory scratch of >= 16 words owned by this warp.
  __device__ static bool run(const T* vals, int Nb, double tau, int lo, int hi, double guard,
                             bool want_flag, uint8_t* mask_row, int32_t* kv_idx_row,
                             int32_t* kv_cnt_out, uint32_t* keep_bits) {
    const int lane = threadIdx.x & 31;
    double v[E];
    int id[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      v[e] = x < Nb ? double(vals[x]) : -1.0;  // pads sort last (values are >= 0)
      id[e] = x;
    }
    // l.7: Z (fixed-order lane partials + xor tree)
    double z = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) z += v[e] > 0.0 ? v[e] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] < Nb) v[e] = v[e] / z;
    // l.8: bitonic sort, descending in (value, -id)
    constexpr int P2 = 32 * E;
#pragma unroll
    for (int kb = 2; kb <= P2; kb <<= 1) {
#pragma unroll
      for (int jb = kb >> 1; jb > 0; jb >>= 1) {
        if (jb < E) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int pe = e ^ jb;
            if (pe > e) {
              const int x = lane * E + e;
              const bool up = (x & kb) == 0;  // this pair should end "before"-ordered
              const bool sw = up ? sel_before(v[pe], id[pe], v[e], id[e])
                                 : sel_before(v[e], id[e], v[pe], id[pe]);
              if (sw) {
                const double tv = v[e]; v[e] = v[pe]; v[pe] = tv;
                const int ti = id[e]; id[e] = id[pe]; id[pe] = ti;
              }
            }
          }
        } else {
          const int lm = jb / E;  // partner lane distance
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double ov = __shfl_xor_sync(0xffffffffu, v[e], lm);
            const int oi = __shfl_xor_sync(0xffffffffu, id[e], lm);
            const int x = lane * E + e;
            const bool lower = (lane & lm) == 0;  // x < partner position
            const bool up = (x & kb) == 0;
            // the lower position keeps the "before" element when up, else the other
            const bool mine_first = sel_before(v[e], id[e], ov, oi);
            const bool keep = (lower == up) ? mine_first : !mine_first;
            if (!keep) {
              v[e] = ov;
              id[e] = oi;
            }
          }
        }
      }
    }
    // l.9: cumulative sums over the lane-contiguous sorted row
    double part = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (lane * E + e < Nb) part += v[e];
    double incl = part;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    double c[E];
    double run = incl - part;
    int first = Nb + 1;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      run += (x < Nb) ? v[e] : 0.0;
      c[e] = run;  // C_{x+1}
      if (x < Nb && run >= tau && first > Nb) first = x + 1;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    // tau >= 1 keeps every block (reading R-4: exact cumulative mass of positive
    // scores reaches 1 only at N_b); else the first m with C_m >= tau
    const int m0 = (tau >= 1.0 || first > Nb) ? Nb : first;
    const int m = min(max(m0, lo), hi);

    bool flag = false;
    if (want_flag) {
      // fetch C at positions m0-1, m0-2 (C_{m0}, C_{m0-1}) and p at m-1, m
      auto getC = [&](int pos) -> double {  // C_{pos+1}; pos may be -1
        const int src = pos < 0 ? 0 : pos / E;
        double val = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (pos >= 0 && pos % E == e) val = c[e];
        val = __shfl_sync(0xffffffffu, val, src);
        return pos < 0 ? 0.0 : val;
      };
      auto getP = [&](int pos) -> double {
        const int src = pos / E;
        double val = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (pos % E == e) val = v[e];
        return __shfl_sync(0xffffffffu, val, src);
      };
      const double cm0 = getC(m0 - 1), cm1 = getC(m0 - 2);
      const double band = guard * tau;
      auto clampi = [&](int x) { return min(max(x, lo), hi); };
      const bool cut_matters = tau < 1.0 && (clampi(m0 - 1) != m || clampi(m0 + 1) != m);
      if (cut_matters && (fabs(cm0 - tau) <= band || (m0 >= 2 && fabs(cm1 - tau) <= band)))
        flag = true;
      if (m < Nb) {
        const double pm = getP(m - 1), pn = getP(m);
        if (pm - pn <= guard * pm) flag = true;
      }
    }
    // l.10: mask and ascending compaction through a bitmap of kept ids
    const int nwords = (Nb + 31) >> 5;
    if (lane < 16) keep_bits[lane] = 0u;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      if (x < m) atomicOr(&keep_bits[id[e] >> 5], 1u << (id[e] & 31));
    }
    __syncwarp();
    const uint32_t myw = lane < nwords ? keep_bits[lane] : 0u;
    const int cntw = __popc(myw);
    int pre = cntw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    pre -= cntw;
    {
      uint32_t w = myw;
      int pos = pre;
      while (w) {
        const int b = __ffs(w) - 1;
        w &= w - 1;
        kv_idx_row[pos++] = lane * 32 + b;
      }
    }
    for (int r = m + lane; r < Nb; r += 32) kv_idx_row[r] = -1;
    if (mask_row)
      for (int j = lane; j < Nb; j += 32) mask_row[j] = (keep_bits[j >> 5] >> (j & 31)) & 1u;
    if (lane == 0) *kv_cnt_out = m;
    __syncwarp();
    return flag;
  }
};


// Fast path for fp32 rows (the probe's output): the sort runs on 64-bit
// integer keys (fp32 bits of P << 32 | ~id), whose descending order is
// (P desc, id asc) — the order of p~ = P/Z, which shares P's order — so the
// network is pure integer compare/select; p~ is formed only after sorting.
template <int E>
struct RowSelectF32 {
  // Keep-ratio mode (lo == hi = m): the top m blocks need no cumulative sums
  // (the clamp fixes the count), so instead of sorting, the m-th largest
  // value is found by a bitwise search over the fp32 bits (non-negative
  // floats order like their bit patterns), ties at it taken by ascending id:
  // the same set, flag and output as the sort path below.
  __device__ static bool topk(const float* vals, int Nb, int m, double guard, bool want_flag,
                              uint8_t* mask_row, int32_t* kv_idx_row, int32_t* kv_cnt_out,
                              uint32_t* keep_bits) {
    const int lane = threadIdx.x & 31;
    uint32_t u[E];
    double z = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      const float pv = x < Nb ? vals[x] : 0.f;
      z += double(pv);
      u[e] = __float_as_uint(pv);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    auto count_ge = [&](uint32_t c) {
      int n = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) n += (lane * E + e < Nb && u[e] >= c) ? 1 : 0;
      return int(__reduce_add_sync(0xffffffffu, uint32_t(n)));
    };
    // T = the m-th largest value: the largest bit pattern with >= m values at or above it
    uint32_t T = 0u;
    for (int b = 31; b >= 0; --b) {
      const uint32_t c = T | (1u << b);
      if (count_ge(c) >= m) T = c;
    }
    const int g = T == 0xffffffffu ? 0 : count_ge(T + 1u);  // strictly above T
    const int need = m - g;                                  // ties at T to keep, by id
    int nt = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) nt += (lane * E + e < Nb && u[e] == T) ? 1 : 0;
    int pre = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    pre -= nt;  // ties at T in lower lanes (lower ids)
    bool flag = false;
    if (want_flag && m < Nb) {
      // p_(m) = T; p_(m+1) = T again when more than m values reach T, else the
      // largest value below T (the sort path's pm - pn <= guard pm on p~ = P / Z)
      uint32_t below = 0u;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (lane * E + e < Nb && u[e] < T) below = below > u[e] ? below : u[e];
      below = __reduce_max_sync(0xffffffffu, below);
      const bool tie = g + nt_total(nt) > m;
      const double inv_z = 1.0 / z;
      const double pm = double(__uint_as_float(T)) * inv_z;
      const double pn = double(__uint_as_float(tie ? T : below)) * inv_z;
      flag = pm - pn <= guard * pm;
    }
    const int nwords = (Nb + 31) >> 5;
    if (lane < 16) keep_bits[lane] = 0u;
    __syncwarp();
    int r = pre;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      if (x < Nb) {
        bool keep = u[e] > T;
        if (u[e] == T) keep = r++ < need;
        if (keep) atomicOr(&keep_bits[x >> 5], 1u << (x & 31));
      }
    }
    __syncwarp();
    const uint32_t myw = lane < nwords ? keep_bits[lane] : 0u;
    const int cntw = __popc(myw);
    int wp = cntw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wp, o);
      if (lane >= o) wp += y;
    }
    wp -= cntw;
    {
      uint32_t w = myw;
      int pos = wp;
      while (w) {
        const int b = __ffs(w) - 1;
        w &= w - 1;
        kv_idx_row[pos++] = lane * 32 + b;
      }
    }
    for (int rr = m + lane; rr < Nb; rr += 32) kv_idx_row[rr] = -1;
    if (mask_row)
      for (int j = lane; j < Nb; j += 32) mask_row[j] = (keep_bits[j >> 5] >> (j & 31)) & 1u;
    if (lane == 0) *kv_cnt_out = m;
    __syncwarp();
    return flag;
  }
  __device__ static int nt_total(int nt) {
    return int(__reduce_add_sync(0xffffffffu, uint32_t(nt)));
  }

  __device__ static bool run(const float* vals, int Nb, double tau, int lo, int hi, double guard,
                             bool want_flag, uint8_t* mask_row, int32_t* kv_idx_row,
                             int32_t* kv_cnt_out, uint32_t* keep_bits) {
#if BLADE_SEL_TOPK
    if (lo == hi)
      return topk(vals, Nb, lo, guard, want_flag, mask_row, kv_idx_row, kv_cnt_out, keep_bits);
#endif
    const int lane = threadIdx.x & 31;
    uint64_t key[E];
    double z = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      const float pv = x < Nb ? vals[x] : 0.f;
      z += double(pv);
      key[e] = x < Nb ? ((uint64_t(__float_as_uint(pv)) << 32) | uint64_t(~uint32_t(x))) : 0ull;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    constexpr int P2 = 32 * E;
#pragma unroll
    for (int kb = 2; kb <= P2; kb <<= 1) {
#pragma unroll
      for (int jb = kb >> 1; jb > 0; jb >>= 1) {
        if (jb < E) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int pe = e ^ jb;
            if (pe > e) {
              const bool up = ((lane * E + e) & kb) == 0;
              const uint64_t a = key[e], b = key[pe];
              const bool sw = up ? (b > a) : (a > b);
              key[e] = sw ? b : a;
              key[pe] = sw ? a : b;
            }
          }
        } else {
          const int lm = jb / E;
          const bool lower = (lane & lm) == 0;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, key[e], lm);
            const bool up = ((lane * E + e) & kb) == 0;
            const bool take_max = (lower == up);
            key[e] = take_max ? (o > key[e] ? o : key[e]) : (o < key[e] ? o : key[e]);
          }
        }
      }
    }
    const double inv_z = 1.0 / z;
    double v[E];
    double part = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      v[e] = x < Nb ? double(__uint_as_float(uint32_t(key[e] >> 32))) * inv_z : 0.0;
      part += v[e];
    }
    double incl = part;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    double c[E];
    double run = incl - part;
    int first = Nb + 1;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane * E + e;
      run += v[e];
      c[e] = run;
      if (x < Nb && run >= tau && first > Nb) first = x + 1;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    // tau >= 1 keeps every block (reading R-4: exact cumulative mass of positive
    // scores reaches 1 only at N_b); else the first m with C_m >= tau
    const int m0 = (tau >= 1.0 || first > Nb) ? Nb : first;
    const int m = min(max(m0, lo), hi);
    bool flag = false;
    if (want_flag) {
      auto pick = [&](const double (&arr)[E], int pos) -> double {
        double val = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
          if ((pos & (E - 1)) == e) val = arr[e];
        return __shfl_sync(0xffffffffu, val, pos < 0 ? 0 : pos / E);
      };
      const double cm0 = pick(c, m0 - 1);
      const double cm1 = m0 >= 2 ? pick(c, m0 - 2) : 0.0;
      const double band = guard * tau;
      auto clampi = [&](int x) { return min(max(x, lo), hi); };
      const bool cut_matters = tau < 1.0 && (clampi(m0 - 1) != m || clampi(m0 + 1) != m);
      if (cut_matters && (fabs(cm0 - tau) <= band || (m0 >= 2 && fabs(cm1 - tau) <= band)))
        flag = true;
      if (m < Nb) {
        const double pm = pick(v, m - 1), pn = pick(v, m);
        if (pm - pn <= guard * pm) flag = true;
      }
    }
    const int nwords = (Nb + 31) >> 5;
    if (lane < 16) keep_bits[lane] = 0u;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (lane * E + e < m) {
        const uint32_t id = ~uint32_t(key[e]);
        atomicOr(&keep_bits[id >> 5], 1u << (id & 31));
      }
    }
    __syncwarp();
    const uint32_t myw = lane < nwords ? keep_bits[lane] : 0u;
    const int cntw = __popc(myw);
    int pre = cntw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    pre -= cntw;
    {
      uint32_t w = myw;
      int pos = pre;
      while (w) {
        const int b = __ffs(w) - 1;
        w &= w - 1;
        kv_idx_row[pos++] = lane * 32 + b;
      }
    }
    for (int r = m + lane; r < Nb; r += 32) kv_idx_row[r] = -1;
    if (mask_row)
      for (int j = lane; j < Nb; j += 32) mask_row[j] = (keep_bits[j >> 5] >> (j & 31)) & 1u;
    if (lane == 0) *kv_cnt_out = m;
    __syncwarp();
    return flag;
  }
};

// Dispatch on the per-lane element count E = P2 / 32.
template <typename T>
__device__ __forceinline__ bool select_row(const T* vals, int Nb, double tau, int lo, int hi,
                                           double guard, bool want_flag, uint8_t* mask_row,
                                           int32_t* kv_idx_row, int32_t* kv_cnt_out,
                                           uint32_t* keep_bits) {
#define BLADE_SEL(E_)                                                                         \
  return std::conditional<std::is_same<T, float>::value, RowSelectF32<E_>,                    \
                          RowSelect<E_, T>>::type::run(vals, Nb, tau, lo, hi, guard, want_flag, mask_row, kv_idx_row, \
                               kv_cnt_out, keep_bits)
  if (Nb <= 32) BLADE_SEL(1);
  if (Nb <= 64) BLADE_SEL(2);
  if (Nb <= 128) BLADE_SEL(4);
  if (Nb <= 256) BLADE_SEL(8);
  BLADE_SEL(16);
#undef BLADE_SEL
}

}  // namespace blade
