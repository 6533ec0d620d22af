// mask_fused.cu — K-mask.2-3 (Alg. 1 l.4-10, with Alg. 3
// P:633-662 as the definition of P_imp) as ONE persistent kernel on sm_100a,
// launched as a programmatic dependent of K-mask.1 (sample_gather_kernel).
//
// The separate probe2 -> select kernels cost a full-grid drain, a 3 MB P_imp
// round trip through L2 and a probe of 2.6 waves of non-persistent CTAs whose
// prologues (TMEM allocation, Q_s load) and pooling epilogues left the tensor
// core idle.  Here one CTA per SM walks the work items (unit u, 128 sampled
// query rows) in static round-robin order:
//
//  A4-A6  the TMA warp streams the item's Q_s tile and every K_s tile; the
//         MMA warp issues S = Q_s K_s^T into two TMEM buffers (the next
//         item's first tiles run under this item's epilogue); the 16
//         statistics warps keep the running row max / sum (Alg. 3 l.12-15)
//         and the per-(row, key-block) max R in TMEM, then pool
//         P_imp[i, j] = max_{s in block i} e^{R_sj - M_s} / l_s (l.17-19)
//         into a double-buffered shared-memory slot.
//  A7-A8  in the item's epilogue one statistics warp per query block
//         selects its row from the slot (select.cuh: fp64 normalisation,
//         sort, cut at tau, clamp, compaction) and queues rows inside the
//         refinement guard band for K-mask.4, while the other statistics
//         warps start the next item (whose rows go to the other slot).
//
// Sampling (A1-A3) stays a separate high-occupancy kernel: it is latency
// bound (hash chains, row gathers) and ran ~2.5x longer as a first phase of
// this kernel with only 20 warps per SM to hide the latency.
//
// Warp roles: 0..15 statistics (and selection), 16 MMA issuer + TMEM
// allocator, 17 TMA producer (+ kMFSel dedicated selection warps, option).  TMEM: S0 [0,128) S1 [128,256) R [256, 256+N_b).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "select.cuh"
#include "tc_ptx.cuh"
#include "tma_host.h"

namespace blade {
namespace {

constexpr int kMFSoft = 16;                       // statistics warps
constexpr int kMFWarpMma = kMFSoft, kMFWarpTma = kMFSoft + 1;
// Selection (A7-A8) by dedicated warps (kMFSel = 2: 20 warps = 5 per SMSP keep
// 96 registers per thread; 22 warps cap it at 80 and the statistics loop
// spills) or, kMFSel = 0, by the statistics warps in the item's epilogue (one
// warp per query block, the others start the next item).  Dedicated warps
// measured slower: Cog's 6672 rows over 296 selection warps (~3 us per row)
// throttle the statistics warps (mask 0.254 vs 0.183 ms unfused).
#ifndef BLADE_MF_SELWARPS
#define BLADE_MF_SELWARPS 0
#endif
constexpr int kMFSel = BLADE_MF_SELWARPS;
constexpr int kMFWarpSel0 = kMFSoft + 2;
constexpr int kMFThreads = 32 * (kMFSoft + 2 + kMFSel);
constexpr int kMFMaxNb = 256;                     // R columns in TMEM
constexpr int kMFMaxRows = 8;                     // query blocks per item (k = 16)

template <int D>
struct MFCfg {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kPanels = D / 64;
  static constexpr int kPanel = 128 * 128;
  static constexpr int kRing = D == 128 ? 4 : 8;
  static constexpr int kOffRing = kTile;  // Q_s tile at 0
  static constexpr int kOffBar = kOffRing + kRing * kTile;
  // bar_q, bar_qfree, full[R], empty[R], bar_s[2], bar_f[2], bar_pooled[2], bar_selfree[2]
  static constexpr int kNumBar = 2 + 2 * kRing + 8;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;      // tmem slot (16 B)
  static constexpr int kOffM = kOffMisc + 16;                 // float  [4][128]
  static constexpr int kOffL = kOffM + 4 * 128 * 4;           // double [4][128]
  static constexpr int kOffP = kOffL + 4 * 128 * 8;           // float  [2][8][kMFMaxNb]
  static constexpr int kOffBits = kOffP + 2 * kMFMaxRows * kMFMaxNb * 4;  // u32 [warps][16]
  static constexpr int kOffNext = kOffBits + (kMFSoft + 2 + kMFSel) * 16 * 4;  // int [2]
  static constexpr int kSmem = kOffNext + 16 + 1024;
};

BLADE_DEVINL float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;\n" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}


struct SelectArgs {
  double tau, guard;
  int lo, hi, neg_flagged;
  float* p_imp_out;  // optional raw P_imp [BH, N_b, N_b]
  uint8_t* mask;     // optional
  int32_t* kv_idx;
  int32_t* kv_cnt;
  int* counters;     // [0] refine queue length (zeroed by K-mask.1)
  int32_t* flags;
  int* done;
};

template <int D, int KK>
__global__ void __launch_bounds__(kMFThreads, 1)
    mask_fused_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const SelectArgs sel, int N, int Nb, int b, int64_t BH, float scale_log2) {
  using C = MFCfg<D>;
  constexpr int G = 128 / KK;  // key blocks per 128-key tile
  constexpr int GH = G / 2;    // key blocks per warp column half
  constexpr int NQ = 128 / KK; // query blocks per work item
  static_assert(GH >= 1 && NQ <= kMFMaxRows, "KK in {16, 32, 64}");
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem;
  char* sRing = smem + C::kOffRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_qfree = bars + 1;
  uint64_t* bar_full = bars + 2;
  uint64_t* bar_empty = bar_full + C::kRing;
  uint64_t* bar_s = bar_empty + C::kRing;  // [2] S buffer written
  uint64_t* bar_f = bar_s + 2;             // [2] S buffer read out (8 warps)
  uint64_t* bar_pooled = bar_f + 2;        // [2] pooled rows of item n in sP[n & 1] (512 thr)
  uint64_t* bar_selfree = bar_pooled + 2;  // [2] sP[n & 1] selected, reusable (128 thr)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  float* smm = reinterpret_cast<float*>(smem + C::kOffM);
  double* sml = reinterpret_cast<double*>(smem + C::kOffL);
  float* sP = reinterpret_cast<float*>(smem + C::kOffP);
  uint32_t* sBits = reinterpret_cast<uint32_t*>(smem + C::kOffBits);
  int* sNext = reinterpret_cast<int*>(smem + C::kOffNext);  // [2] next row to select per slot

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NK = Nb * KK;
  const int ntiles = (NK + 127) / 128;
  const int64_t nitems = BH * ntiles;
  const int k_last = min(KK, N - (Nb - 1) * b);
  const int first_invalid = (Nb - 1) * KK + k_last;  // sampled columns >= this are padding

  if (warp == kMFWarpTma && lane == 0) {
    tc::mbar_init(bar_q, 1);
    tc::mbar_init(bar_qfree, 1);
    for (int s = 0; s < C::kRing; ++s) {
      tc::mbar_init(bar_full + s, 1);
      tc::mbar_init(bar_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(bar_s + t, 1);
      tc::mbar_init(bar_f + t, kMFSoft / 2);
      tc::mbar_init(bar_pooled + t, kMFSoft * 32);
      tc::mbar_init(bar_selfree + t, kMFSel > 0 ? kMFSel * 32 : 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == kMFWarpMma) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent of K-mask.1: Q_s / K_s and the zeroed refine queue
  // counter are complete and visible past this point
  asm volatile("griddepcontrol.wait;\n" ::: "memory");

  // A7-A8 for the query blocks of an item whose pooled rows sit in slot bs:
  // rows are claimed one at a time (selection warps; the statistics warps
  // join for their last item)
  auto select_rows = [&](int bs, int64_t u, int ib0, int nq) {
    const float* P = sP + bs * kMFMaxRows * kMFMaxNb;
    for (;;) {
      int ql = 0;
      if (lane == 0) ql = atomicAdd(sNext + bs, 1);
      ql = __shfl_sync(0xffffffffu, ql, 0);
      if (ql >= nq) break;
      const int64_t row = u * Nb + ib0 + ql;
      const bool flag = select_row(P + ql * kMFMaxNb, Nb, sel.tau, sel.lo, sel.hi, sel.guard, true,
                                   sel.mask ? sel.mask + row * Nb : nullptr, sel.kv_idx + row * Nb,
                                   sel.kv_cnt + row, sBits + warp * 16);
      if (flag && lane == 0) {
        const int slot = atomicAdd(&sel.counters[0], 1);
        sel.flags[slot] = int32_t(row);
        sel.done[slot] = 0;
        // blade_asa_fwd: provisional count (-1 - m) until K-mask.4 rewrites it
        if (sel.neg_flagged) sel.kv_cnt[row] = -1 - sel.kv_cnt[row];
      }
    }
  };

  if (warp == kMFWarpTma) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmQ);
      tc::tma_prefetch_desc(&tmK);
      int g = 0;
      for (int n = 0;; ++n) {
        const int64_t item = blockIdx.x + int64_t(n) * gridDim.x;
        if (item >= nitems) break;
        const int64_t u = item / ntiles;
        const int rt = int(item % ntiles);
        if (n > 0) tc::mbar_wait(bar_qfree, (n - 1) & 1);  // last S MMA of item n-1 done
        tc::mbar_arrive_expect_tx(bar_q, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(sQ + p * C::kPanel, &tmQ, bar_q, p * 64, rt * 128, int(u));
        for (int t = 0; t < ntiles; ++t, ++g) {
          const int s = g % C::kRing;
          tc::mbar_wait(bar_empty + s, ((g / C::kRing) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(bar_full + s, C::kTile);
          for (int p = 0; p < C::kPanels; ++p)
            tc::tma_load_3d(sRing + s * C::kTile + p * C::kPanel, &tmK, bar_full + s, p * 64,
                            t * 128, int(u));
        }
      }
    }
  } else if (warp == kMFWarpMma) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      const uint32_t qa = smem_u32(sQ), rb = smem_u32(sRing);
      int g = 0, T = 0;  // ring position, S tile count (buffer T & 1, use T >> 1)
      for (int n = 0;; ++n) {
        const int64_t item = blockIdx.x + int64_t(n) * gridDim.x;
        if (item >= nitems) break;
        tc::mbar_wait(bar_q, n & 1);
        tc::fence_after_sync();
        for (int t = 0; t < ntiles; ++t, ++g, ++T) {
          const int s = g % C::kRing, bsel = T & 1;
          tc::mbar_wait(bar_full + s, (g / C::kRing) & 1);
          if (T >= 2) tc::mbar_wait(bar_f + bsel, ((T >> 1) - 1) & 1);
          tc::fence_after_sync();
          const uint32_t kb = rb + s * C::kTile;
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
            tc::mma_ss(tmem + bsel * 128, tc::sw128_desc(qa + off, 16, 1024),
                       tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
          }
          tc::commit(bar_s + bsel);
          tc::commit(bar_empty + s);
        }
        tc::commit(bar_qfree);  // Q_s tile free once this item's MMAs complete
      }
    }
  } else {
    if (kMFSel > 0 && warp >= kMFWarpSel0) {
      // ===================== phase 3 (A7-A8): selection warps =====================
      const int sw = warp - kMFWarpSel0;
      for (int n = 0;; ++n) {
        const int64_t item = blockIdx.x + int64_t(n) * gridDim.x;
        if (item >= nitems) break;
        const int64_t u = item / ntiles;
        const int rt = int(item % ntiles);
        tc::mbar_wait(bar_pooled + (n & 1), (n >> 1) & 1);
        const float* P = sP + (n & 1) * kMFMaxRows * kMFMaxNb;
        const int ib0 = (rt * 128) / KK;
        const int nq = min(NQ, Nb - ib0);
        if (sel.p_imp_out) {  // optional raw P_imp output
          for (int x = sw * 32 + lane; x < nq * Nb; x += kMFSel * 32) {
            const int ql = x / Nb, j = x % Nb;
            sel.p_imp_out[(u * Nb + ib0 + ql) * int64_t(Nb) + j] = P[ql * kMFMaxNb + j];
          }
        }
        select_rows(n & 1, u, ib0, nq);
        tc::mbar_arrive(bar_selfree + (n & 1));  // every lane, after its last read of sP
      }
    } else {
    // ===================== phase 2: statistics and pooling =====
    const int par = warp >> 3, h = (warp >> 2) & 1, quad = warp & 3;
    const int grp = warp >> 2;  // (par, h): which of the four partial states
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    const int r = quad * 32 + lane;
    int last_n = -1;
    for (int n = 0;; ++n) {
      const int64_t item = blockIdx.x + int64_t(n) * gridDim.x;
      if (item >= nitems) break;
      last_n = n;
      const int64_t u = item / ntiles;
      const int rt = int(item % ntiles);
      const int Tb = n * ntiles;
      float* P = sP + (n & 1) * kMFMaxRows * kMFMaxNb;
      if (kMFSel > 0 && n >= 2)  // item n-2 selected
        tc::mbar_wait(bar_selfree + (n & 1), ((n >> 1) - 1) & 1);
      if (kMFSel > 0 && tid == 0) sNext[n & 1] = 0;  // published by the bar_pooled arrivals
      if (KK > 32)  // pooled rows by atomicMax over two quads: start from +0
        for (int x = tid; x < NQ * kMFMaxNb; x += kMFSoft * 32) P[x] = 0.f;
      float m_run = -INFINITY;
      double l_run = 0.0;
      for (int t = 0; t < ntiles; ++t) {
        const int T = Tb + t;
        if ((T & 1) != par) continue;
        tc::mbar_wait(bar_s + par, (T >> 1) & 1);
        tc::fence_after_sync();
        float s[64];
        {
          const uint32_t ta = tmem + lane_base + par * 128 + h * 64;
          uint32_t r0[32], r1[32];
          tc::ld_32x32b_x32(ta, r0);
          tc::ld_32x32b_x32(ta + 32, r1);
          tc::wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            s[e] = __uint_as_float(r0[e]);
            s[32 + e] = __uint_as_float(r1[e]);
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(bar_f + par);  // S buffer may be overwritten now
        const int col0 = t * 128 + h * 64;
        if (col0 + 64 > first_invalid) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (col0 + c >= first_invalid) s[c] = -INFINITY;
        }
        // R: per key-block max of the raw logits (Alg. 3 l.12/l.15)
        uint32_t rv[GH];
        float tmax = -INFINITY;
#pragma unroll
        for (int gg = 0; gg < GH; ++gg) {
          float gm = fmax3(s[gg * KK], s[gg * KK + 1], s[gg * KK + 2]);
#pragma unroll
          for (int c = 3; c + 1 < KK; c += 2) gm = fmax3(gm, s[gg * KK + c], s[gg * KK + c + 1]);
          if ((KK & 1) == 0) gm = fmaxf(gm, s[gg * KK + KK - 1]);
          tmax = fmaxf(tmax, gm);
          rv[gg] = __float_as_uint(gm);
        }
        const uint32_t rcol = tmem + lane_base + 256 + t * G + h * GH;
        if constexpr (GH == 4) {
          tc::st_32x32b_x4(rcol, reinterpret_cast<uint32_t(&)[4]>(rv));
        } else if constexpr (GH == 2) {
          tc::st_32x32b_x2(rcol, reinterpret_cast<uint32_t(&)[2]>(rv));
        } else {
          tc::st_32x32b_x1(rcol, reinterpret_cast<uint32_t(&)[1]>(rv));
        }
        // online row max / sum over this half tile (l.13-15)
        const float m_new = fmaxf(m_run, tmax);
        if (m_new != -INFINITY) {
          const float2 nm2 = make_float2(-m_new, -m_new);
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 x = mul2(add2(make_float2(s[c], s[c + 1]), nm2), sc2);
            s[c] = ex2(x.x);
            s[c + 1] = ex2(x.y);
          }
#pragma unroll
          for (int w = 32; w >= 2; w >>= 1)
#pragma unroll
            for (int c = 0; c < w; c += 2) {
              const float2 y = add2(make_float2(s[c], s[c + 1]), make_float2(s[c + w], s[c + w + 1]));
              s[c] = y.x;
              s[c + 1] = y.y;
            }
          s[0] += s[1];
          if (m_new != m_run) l_run *= double(ex2((m_run - m_new) * scale_log2));
          l_run += double(s[0]);
          m_run = m_new;
        }
      }
      tc::wait_st();
      // merge the four partial (M, l) of each row (the l.14 recurrence, once)
      smm[grp * 128 + r] = m_run;
      sml[grp * 128 + r] = l_run;
      tc::fence_before_sync();  // R columns written by every statistics warp, read below
      asm volatile("bar.sync 1, %0;\n" ::"n"(kMFSoft * 32) : "memory");
      tc::fence_after_sync();
      float M = -INFINITY;
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) M = fmaxf(M, smm[gg * 128 + r]);
      double L = 0.0;
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        const float mg = smm[gg * 128 + r];
        if (mg != -INFINITY) L += sml[gg * 128 + r] * double(ex2((mg - M) * scale_log2));
      }
      // pooling (l.17-19): v_sj = (R_sj - M_s) c - log2 l_s, P_imp = 2^(max_s v_sj)
      const int gr = rt * 128 + r;
      const int ib = gr / KK;
      const bool row_ok = gr < NK && (gr % KK) < min(KK, N - ib * b);
      const float lg = float(log2(L));
      const int qb_local = r / KK;  // query block of this row within the item
      for (int j0 = grp * 32; j0 < Nb; j0 += 128) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + 256 + j0, rr);
        tc::wait_ld();
        float pv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float v = row_ok ? (__uint_as_float(rr[e]) - M) * scale_log2 - lg : -INFINITY;
#pragma unroll
          for (int o = 1; o < KK && o < 32; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
          pv[e] = v;
        }
        const int nj = min(32, Nb - j0);
        if (KK > 32) {  // a block spans two quads: max of the two halves
          if (lane == 0)
            for (int e = 0; e < nj; ++e)
              atomicMax(reinterpret_cast<int*>(P + qb_local * kMFMaxNb + j0 + e),
                        __float_as_int(ex2(pv[e])));
        } else if ((lane % KK) == 0) {
          float* dst = P + qb_local * kMFMaxNb + j0;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e < nj) dst[e] = ex2(pv[e]);
        }
      }
      if (kMFSel > 0) tc::mbar_arrive(bar_pooled + (n & 1));  // every lane, after its sP writes
      tc::fence_before_sync();  // R reads done before the next item's R writes
      asm volatile("bar.sync 1, %0;\n" ::"n"(kMFSoft * 32) : "memory");
      tc::fence_after_sync();
      if constexpr (kMFSel == 0) {
        // A7-A8 in the epilogue: warps < nq select one query block each while
        // the others start the next item (its pooled rows go to the other slot)
        const int ib0 = (rt * 128) / KK;
        const int nq = min(NQ, Nb - ib0);
        if (sel.p_imp_out) {
          for (int x = tid; x < nq * Nb; x += kMFSoft * 32) {
            const int ql = x / Nb, j = x % Nb;
            sel.p_imp_out[(u * Nb + ib0 + ql) * int64_t(Nb) + j] = P[ql * kMFMaxNb + j];
          }
        }
        if (warp < nq) {
          const int64_t row = u * Nb + ib0 + warp;
          const bool flag = select_row(P + warp * kMFMaxNb, Nb, sel.tau, sel.lo, sel.hi,
                                       sel.guard, true, sel.mask ? sel.mask + row * Nb : nullptr,
                                       sel.kv_idx + row * Nb, sel.kv_cnt + row, sBits + warp * 16);
          if (flag && lane == 0) {
            const int slot = atomicAdd(&sel.counters[0], 1);
            sel.flags[slot] = int32_t(row);
            sel.done[slot] = 0;
            if (sel.neg_flagged) sel.kv_cnt[row] = -1 - sel.kv_cnt[row];
          }
        }
      }
    }
    if (kMFSel > 0 && last_n >= 0) {  // no item left: help select the last one's rows
      const int64_t item = blockIdx.x + int64_t(last_n) * gridDim.x;
      const int ib0 = int(item % ntiles) * 128 / KK;
      select_rows(last_n & 1, item / ntiles, ib0, min(NQ, Nb - ib0));
    }
    }  // statistics warps
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kMFWarpMma) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n > 0 ? n : 148;
}

template <int D, int KK>
cudaError_t launch_mf(const MaskProblem& p, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                      float* p_imp_out, const MaskFusedBufs& w, cudaStream_t stream) {
  CUtensorMap mq, mk;
  const int64_t NK = int64_t(p.Nb) * KK;
  if (!make_tile_map(&mq, w.qs, p.BH, NK, D) || !make_tile_map(&mk, w.ks, p.BH, NK, D))
    return cudaErrorNotSupported;
  constexpr int smem = MFCfg<D>::kSmem;
  auto kern = mask_fused_kernel<D, KK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  SelectArgs sl{p.tau, p.guard, p.lo, p.hi, p.neg_flagged, p_imp_out, mask, kv_idx, kv_cnt,
                w.counters, w.flags, w.done};
  const int64_t nitems = p.BH * ((NK + 127) / 128);
  const int sms = sm_count();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(nitems < sms ? nitems : sms));
  cfg.blockDim = dim3(kMFThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, mq, mk, sl, p.N, p.Nb, p.b, p.BH, p.scale * kLog2e);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

bool mask_fused_supported(const MaskProblem& p) {
#ifdef BLADE_MASK_UNFUSED  // A/B: the three-kernel K-mask.1-3 path
  return false;
#else
  return (p.d == 64 || p.d == 128) && (p.kk == 16 || p.kk == 32 || p.kk == 64) &&
         p.Nb <= kMFMaxNb;
#endif
}

cudaError_t launch_mask_fused(const MaskProblem& p, uint8_t* mask, int32_t* kv_idx,
                              int32_t* kv_cnt, float* p_imp_out, const MaskFusedBufs& w,
                              cudaStream_t stream) {
#define BLADE_MF(D_, K_)                                                                      \
  if (p.d == D_ && p.kk == K_)                                                                \
    return launch_mf<D_, K_>(p, mask, kv_idx, kv_cnt, p_imp_out, w, stream);
  BLADE_MF(128, 16) BLADE_MF(128, 32) BLADE_MF(128, 64)
  BLADE_MF(64, 16) BLADE_MF(64, 32) BLADE_MF(64, 64)
#undef BLADE_MF
  return cudaErrorNotSupported;
}

}  // namespace blade
