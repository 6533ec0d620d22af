// attn_tc2.cu — block-sparse attention forward for sm_100a, two query blocks
// per CTA ("Standard ASA ... integrated with a block-sparse
// attention kernel"; P:135 ASA_GT global tokens as extra tiles).
//
// Why two: with one query block per CTA the tensor core waits while the
// softmax of the same block runs (S(n+1) cannot be consumed before P(n)).
// Here each CTA owns query blocks A = 2x and B = 2x+1 of one unit, each with
// its own kept-block list, its own softmax warpgroup and its own S and O in
// TMEM; the MMA issuer alternates between them, so the tensor core computes
// B's P V and Q K^T while A's softmax runs, and vice versa (ping-pong):
//
//   tensor pipe:  S_A0 S_B0 | PV_A0 S_A1 | PV_B0 S_B1 | PV_A1 S_A2 | ...
//   softmax A:         [ A0 ]           [ A1 ]           [ A2 ]
//   softmax B:                [ B0 ]           [ B1 ]
//
// Warp roles (384 threads):
//   warps 0-3   softmax of block A (thread = query row = TMEM lane)
//   warps 4-7   softmax of block B
//   warp  8     tcgen05.mma issuer (one thread) + TMEM allocator
//   warp  9     TMA producer: Q_A, Q_B, then K tiles in consumption order
//   warp  10    TMA producer: V tiles in consumption order
//   warp  11    builds the item tables (I, A \ B, B \ A) before the roles start
//               (an issuer per block was measured 24 % slower: an issuing
//               thread blocks at the tensor pipe's pace either way)
// TMEM (512 columns): S_A [0,128) S_B [128,256) O_A [256, 256+d) O_B [256+d, 256+2d).
// P (bf16) overwrites the upper half of its S and is the TMEM A operand of
// P V; S(n+1) of a block is issued after P V(n) of that block (the tensor
// pipe executes a thread's MMAs in order), so the commit that signals S(n+1)
// also guarantees that P V(n) finished writing O (no separate wait before a
// rescale).  Q stays in shared memory (S = Q K^T is an SS MMA).
// K and V rings are shared by both blocks, filled in the order the MMA issuer
// consumes them.  Adjacent query blocks keep mostly the same key blocks (62 %
// of the lists on the Wan inputs), so each CTA first splits its two lists
// into the common part I = A n B and the exclusive parts A \ B, B \ A (warp
// 11, bitmaps in shared memory) and orders both blocks' items as
//   [global-token tiles] [I] [own exclusive blocks]:
// item k < n_S = n_GT + |I| is the same tile for A and B, loaded once into one
// ring slot and consumed by S_A(k), S_B(k) (K) and P V_A(k), P V_B(k) (V);
// later items alternate A B A B ... as before (the shorter list ends first).
// One TMA load and one shared-memory write then serve both blocks wherever
// their lists agree.  The order of a block's items only changes the fp32
// rounding of its online softmax (reading R-17).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"
#include "tma_host.h"

namespace blade {
namespace {

using attn::DefaultScale;
using attn::ex2_poly2;
using attn::GtArgs;

template <int D>
struct Cfg2 {
  static constexpr int kTile = 128 * D * 2;  // one Q / K / V tile
  static constexpr int kPanels = D / 64;     // 128-byte SW128 panels along d
  static constexpr int kPanel = 128 * 128;
#ifndef BLADE_ATTN2_RINGK128
#define BLADE_ATTN2_RINGK128 3  // 2 / 3 within noise on the Wan layer
#endif
#ifndef BLADE_ATTN2_RINGV128
#define BLADE_ATTN2_RINGV128 2
#endif
#ifndef BLADE_ATTN2_RINGK64
#define BLADE_ATTN2_RINGK64 6  // 6 / 6 for d = 64: Cog 1.0358 vs 1.0404 ms (5 / 4), 1.0372 (4 / 3)
#endif
#ifndef BLADE_ATTN2_RINGV64
#define BLADE_ATTN2_RINGV64 6
#endif
  static constexpr int kRingK = D == 128 ? BLADE_ATTN2_RINGK128 : BLADE_ATTN2_RINGK64;
  static constexpr int kRingV = D == 128 ? BLADE_ATTN2_RINGV128 : BLADE_ATTN2_RINGV64;
  static constexpr int kOffQ = 0;  // Q_A, Q_B
  static constexpr int kOffRingK = 2 * kTile;
  static constexpr int kOffRingV = kOffRingK + kRingK * kTile;
  static constexpr int kOffBar = kOffRingV + kRingV * kTile;
  // bar_q, kfull/kempty, vfull/vempty, per block: s, p, pv
  static constexpr int kNumBar = 1 + 2 * kRingK + 2 * kRingV + 3 * 2;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;  // tmem slot, n_I
  static constexpr int kOffTab = kOffMisc + 16;           // item tables, 3 x 256 B
  static constexpr int kOffBits = kOffTab + 3 * 256;      // list bitmaps, 2 x 8 words
  static constexpr int kSmem = kOffBits + 64 + 1024;      // + alignment slack
  static constexpr uint32_t kColO = 256;
};

constexpr int kThreads2 = 384;
constexpr int kShareMaxNb = 256;  // item tables hold 8-bit block ids

constexpr float kRescaleThreshold = 8.0f;  // log2 units
// Which of every 8 exponential pairs run on the FMA pipe (ex2_poly2) instead
// of MUFU: 1 in 8 for d = 64, none for d = 128 (interleaved A/B on B200:
// Cog 1.038 ms vs 1.045 (1 in 4) / 1.046 (none); Wan 1.166-1.171 vs 1.176
// (1 in 8) / 1.203-1.217 (1 in 4); 2 and 4 in 8 lose on both).
#ifdef BLADE_ATTN2_EMU_MASK
constexpr uint32_t kEmuMask2_64 = BLADE_ATTN2_EMU_MASK, kEmuMask2_128 = BLADE_ATTN2_EMU_MASK;
#else
constexpr uint32_t kEmuMask2_64 = 0x01, kEmuMask2_128 = 0x00;
#endif

// The item schedule of a CTA.  Items k < nS are shared by both blocks; later
// items alternate A, B (the shorter list simply ends earlier).  pos() is the
// position of block t's item k in the sequence the producers fill the rings
// with and the issuer drains them in.
struct Sched {
  int cntA, cntB;  // items per block (kept blocks + global-token tiles)
  int nS;          // shared items (0 for a lone last block)
  BLADE_DEVINL int pos(int t, int k) const {
    if (k < nS) return k;
    return nS + (min(k, cntA) - nS) + (min(k, cntB) - nS) + ((t == 1 && k < cntA) ? 1 : 0);
  }
  // calls f(t, k, shared) for every ring position in order
  template <typename F>
  BLADE_DEVINL void for_each(F&& f) const {
    const int m = cntA > cntB ? cntA : cntB;
    for (int k = 0; k < m; ++k) {
      if (k < nS) {
        f(0, k, true);
      } else {
        if (k < cntA) f(0, k, false);
        if (k < cntB) f(1, k, false);
      }
    }
  }
};

template <int D, bool kDefaultScale, bool kGT>
__global__ void __launch_bounds__(kThreads2, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV,
                    const __grid_constant__ CUtensorMap tmKg,
                    const __grid_constant__ CUtensorMap tmVg, const GtArgs gt, int N, int Nb,
                    float scale_log2_rt, const int32_t* __restrict__ kv_idx,
                    const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ O,
                    float* __restrict__ LSE, int pdl, const int32_t* __restrict__ order) {
  using C = Cfg2<D>;
  const float scale_log2 = kDefaultScale ? DefaultScale<D>::kScaleLog2 : scale_log2_rt;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem + C::kOffQ;
  char* sRingK = smem + C::kOffRingK;
  char* sRingV = smem + C::kOffRingV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_kempty = bar_kfull + C::kRingK;
  uint64_t* bar_vfull = bar_kempty + C::kRingK;
  uint64_t* bar_vempty = bar_vfull + C::kRingV;
  uint64_t* bar_s = bar_vempty + C::kRingV;  // [2] S of block t computed
  uint64_t* bar_p = bar_s + 2;               // [2] P of block t written (4 warp arrivals)
  uint64_t* bar_pv = bar_p + 2;              // [2] last P V of block t done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  int* s_nI = reinterpret_cast<int*>(smem + C::kOffMisc + 4);
  uint8_t* tabI = reinterpret_cast<uint8_t*>(smem + C::kOffTab);  // common blocks (A's order)
  uint8_t* tabX[2] = {tabI + 256, tabI + 512};                      // exclusive blocks of A, B
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + C::kOffBits);  // [2][8] list bitmaps

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // LPT order (blade_asa_fwd, tau mode): CTA b takes the b-th longest pair
  const int64_t item = order ? int64_t(__ldg(order + blockIdx.y * int64_t(gridDim.x) + blockIdx.x))
                             : blockIdx.y * int64_t(gridDim.x) + blockIdx.x;
  const int64_t u = item / gridDim.x;
  const int i0 = 2 * int(item % gridDim.x);     // block A; block B = i0 + 1 (if < Nb)
  const int nblk = (i0 + 1 < Nb) ? 2 : 1;
  const int ngt = kGT ? (gt.Ng + 127) / 128 : 0;
  int cf0 = kv_cnt[u * Nb + i0];
  int cf1 = nblk == 2 ? kv_cnt[u * Nb + i0 + 1] : 0;
  // a CTA that waited reads its lists through L2 (ld.global.cg): the refine
  // kernel rewrote them while this grid ran, and a line another CTA on this
  // SM pulled into L1 through the non-coherent path before could be stale
  const bool waited = pdl && (cf0 < 0 || cf1 < 0);
  auto ld_list = [waited](const int32_t* p) { return waited ? __ldcg(p) : __ldg(p); };
  if (waited) {  // a refined row (blade_asa_fwd): wait for K-mask.4
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    cf0 = __ldcg(kv_cnt + u * Nb + i0);
    cf1 = nblk == 2 ? __ldcg(kv_cnt + u * Nb + i0 + 1) : 0;
  }
  const int32_t* list0 = kv_idx + (u * Nb + i0) * Nb;
  const int32_t* list1 = list0 + Nb;
  const bool share = nblk == 2 && Nb <= kShareMaxNb;

  if (warp == 9 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRingK; ++s) {
      tc::mbar_init(bar_kfull + s, 1);
      tc::mbar_init(bar_kempty + s, 1);
    }
    for (int s = 0; s < C::kRingV; ++s) {
      tc::mbar_init(bar_vfull + s, 1);
      tc::mbar_init(bar_vempty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(bar_s + t, 1);
      tc::mbar_init(bar_p + t, 4);
      tc::mbar_init(bar_pv + t, 1);
    }
    tc::fence_barrier_init();
    // Q_A, Q_B right away: their latency overlaps the item-table build
    tc::tma_prefetch_desc(&tmQ);
    tc::mbar_arrive_expect_tx(bar_q, nblk * C::kTile);
    for (int t = 0; t < nblk; ++t)
      for (int p = 0; p < C::kPanels; ++p)
        tc::tma_load_3d(sQ + t * C::kTile + p * C::kPanel, &tmQ, bar_q, p * 64, (i0 + t) * 128,
                        int(u));
  }
  if (warp == 8) tc::tmem_alloc<512>(tmem_slot);
  if (warp == 11) {
    // ---- item tables: I = A n B in A's order, A \ B, B \ A (any list order) ----
    int nI = 0;
    if (share) {
      // both lists in registers (one L2 round trip), bitmaps, then the split
      int a[kShareMaxNb / 32], bl[kShareMaxNb / 32];
#pragma unroll
      for (int e = 0; e < kShareMaxNb / 32; ++e) {
        a[e] = 32 * e + lane < cf0 ? ld_list(list0 + 32 * e + lane) : -1;
        bl[e] = 32 * e + lane < cf1 ? ld_list(list1 + 32 * e + lane) : -1;
      }
      if (lane < 16) bits[lane] = 0u;
      __syncwarp();
#pragma unroll
      for (int e = 0; e < kShareMaxNb / 32; ++e) {
        if (a[e] >= 0) atomicOr(&bits[a[e] >> 5], 1u << (a[e] & 31));
        if (bl[e] >= 0) atomicOr(&bits[8 + (bl[e] >> 5)], 1u << (bl[e] & 31));
      }
      __syncwarp();
      const uint32_t lt = (1u << lane) - 1u;
      int nxa = 0, nxb = 0;
#pragma unroll
      for (int e = 0; e < kShareMaxNb / 32; ++e) {
        const int j = a[e];
        const bool in = j >= 0 && ((bits[8 + (j >> 5)] >> (j & 31)) & 1u);
        const uint32_t bi = __ballot_sync(0xffffffffu, in);
        const uint32_t bx = __ballot_sync(0xffffffffu, j >= 0 && !in);
        if (in) tabI[nI + __popc(bi & lt)] = uint8_t(j);
        else if (j >= 0) tabX[0][nxa + __popc(bx & lt)] = uint8_t(j);
        nI += __popc(bi);
        nxa += __popc(bx);
        const int jb = bl[e];
        const bool ex = jb >= 0 && !((bits[jb >> 5] >> (jb & 31)) & 1u);
        const uint32_t bxb = __ballot_sync(0xffffffffu, ex);
        if (ex) tabX[1][nxb + __popc(bxb & lt)] = uint8_t(jb);
        nxb += __popc(bxb);
      }
    }
    if (lane == 0) *s_nI = nI;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const int nI = *s_nI;
  const int cnt0 = cf0 + ngt, cnt1 = nblk == 2 ? cf1 + ngt : 0;
  const Sched sch{cnt0, cnt1, nblk == 2 ? ngt + nI : 0};
  // block id of block t's item k (k >= ngt; the first ngt items are the
  // global-token tiles): common blocks, then the block's own
  auto item_block = [&](int t, int k) -> int {
    const int f = k - ngt;
    if (!share) return ld_list((t ? list1 : list0) + f);
    return f < nI ? int(tabI[f]) : int(tabX[t][f - nI]);
  };
  // registers: the two softmax warpgroups hold a 128-column S row per thread;
  // the issuer / producer warpgroup needs few (2 x 128 x 216 + 128 x 56 <= 64K)
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 9 || warp == 10) {
      // ===================== TMA producers (warp 9: Q and K, warp 10: V) =====
      if (lane == 0) {
        const bool isK = warp == 9;
        if (isK) {
          tc::tma_prefetch_desc(&tmK);
          if (kGT) tc::tma_prefetch_desc(&tmKg);
        } else {
          tc::tma_prefetch_desc(&tmV);
          if (kGT) tc::tma_prefetch_desc(&tmVg);
        }
        const int R = isK ? C::kRingK : C::kRingV;
        char* ring = isK ? sRingK : sRingV;
        uint64_t* full = isK ? bar_kfull : bar_vfull;
        uint64_t* empty = isK ? bar_kempty : bar_vempty;
        const CUtensorMap* m = isK ? &tmK : &tmV;
        const CUtensorMap* mg = isK ? &tmKg : &tmVg;
        int g = 0;
        sch.for_each([&](int t, int k, bool) {
          const bool fine = !kGT || k >= ngt;
          const int row0 = fine ? item_block(t, k) * 128 : k * 128;
          const int s = g % R;
          tc::mbar_wait(empty + s, ((g / R) & 1) ^ 1);
          char* dst = ring + s * C::kTile;
          tc::mbar_arrive_expect_tx(full + s, C::kTile);
          for (int p = 0; p < C::kPanels; ++p)
            tc::tma_load_3d(dst + p * C::kPanel, fine ? m : mg, full + s, p * 64, row0, int(u));
          ++g;
        });
      }
    } else if (warp == 8) {
      // ===================== MMA issuer =====================
      if (lane == 0) {
        constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idO = tc::idesc_bf16(128, D, 0, 1);
        const uint32_t qbase = smem_u32(sQ), kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
        tc::mbar_wait(bar_q, 0);
        tc::fence_after_sync();
        auto issue_S = [&](int t, int k) {  // S_t = Q_t K^T of block t's item k
          const int g = sch.pos(t, k), s = g % C::kRingK;
          tc::mbar_wait(bar_kfull + s, (g / C::kRingK) & 1);
          tc::fence_after_sync();
          const uint32_t kb = kbase + s * C::kTile, qb = qbase + t * C::kTile;
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
            tc::mma_ss(tmem + t * 128, tc::sw128_desc(qb + off, 16, 1024),
                       tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
          }
          tc::commit(bar_s + t);
          // a shared tile is released after its second reader, S_B(k)
          if (k >= sch.nS || t == 1) tc::commit(bar_kempty + s);
        };
        auto issue_PV = [&](int t, int k) {  // O_t += P_t V of block t's item k
          const int g = sch.pos(t, k), s = g % C::kRingV;
          tc::mbar_wait(bar_vfull + s, (g / C::kRingV) & 1);
          tc::mbar_wait(bar_p + t, k & 1);
          tc::fence_after_sync();
          const uint32_t vb = vbase + s * C::kTile;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc::mma_ts(tmem + C::kColO + t * D, tmem + t * 128 + 64 + ks * 8,
                       tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO,
                       (k > 0 || ks > 0) ? 1 : 0);
          // only the last P V of a block is awaited (S(n) is issued after P
          // V(n-1) and tcgen05 ops of one thread complete in order): one
          // commit, so every phase of bar_pv has a waiter
          if (k + 1 == (t ? cnt1 : cnt0)) tc::commit(bar_pv + t);
          if (k >= sch.nS || t == 1) tc::commit(bar_vempty + s);
        };
        if (cnt0 > 0) issue_S(0, 0);
        if (cnt1 > 0) issue_S(1, 0);
        const int m = cnt0 > cnt1 ? cnt0 : cnt1;
        for (int k = 0; k < m; ++k) {
          if (k < cnt0) {
            issue_PV(0, k);
            if (k + 1 < cnt0) issue_S(0, k + 1);
          }
          if (k < cnt1) {
            issue_PV(1, k);
            if (k + 1 < cnt1) issue_S(1, k + 1);
          }
        }
        // drain: the last commits must land before the CTA's smem is released
        if (cnt0 > 0) tc::mbar_wait(bar_pv + 0, 0);
        if (cnt1 > 0) tc::mbar_wait(bar_pv + 1, 0);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::: "memory");
    // ===================== softmax of block t =====================
    const int t = warp >> 2, qw = warp & 3;
    const int cnt = t ? cnt1 : cnt0;
    const uint32_t lane_base = uint32_t(qw * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + C::kColO + t * D;
    const int r = qw * 32 + lane;
    float m_used = -INFINITY, l_sum = 0.f;
    for (int n = 0; n < cnt; ++n) {
      const bool fine = !kGT || n >= ngt;
      const int valid = fine ? N - item_block(t, n) * 128 : gt.Ng - n * 128;
      tc::mbar_wait(bar_s + t, n & 1);
      tc::fence_after_sync();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tS + c * 32, rr);
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(rr[e]);
      }
      tc::wait_ld();
      if (valid < 128) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c >= valid) s[c] = -INFINITY;
      }
      if (kGT && !fine) {  // + ln(n_w) on the pooled region, raw-score units
        const int last = gt.Ng - 1 - n * 128;
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] += c == last ? gt.bias_last : gt.bias_full;
      }
      float mx;
      {
        float t8[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float a = fmaxf(s[g], s[g + 8]);
#pragma unroll
          for (int c = g + 16; c < 128; c += 16) a = fmaxf(a, fmaxf(s[c], s[c + 8]));
          t8[g] = a;
        }
        mx = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                   fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7])));
      }
      const float mxs = mx * scale_log2;
      // warp-uniform (tcgen05.ld/st are .sync.aligned); always true for n = 0.
      // O_t is current: S_t(n) was issued after P V_t(n-1) and has completed.
      if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold)) {
        const float m_new = fmaxf(m_used, mxs);
        if (n > 0) {
          const float f = ex2(m_used - m_new);
          l_sum *= f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t rr[32];
            tc::ld_32x32b_x32(tO + c * 32, rr);
            tc::wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) * f);
            tc::st_32x32b_x32(tO + c * 32, rr);
          }
        }
        m_used = m_new;
      }
      float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
      const float2 sl2 = make_float2(scale_log2, scale_log2);
      const float2 nm = make_float2(-m_used, -m_used);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = fma2(make_float2(s[c * 32 + 2 * e], s[c * 32 + 2 * e + 1]), sl2, nm);
          float2 pp;
          if (((D == 64 ? kEmuMask2_64 : kEmuMask2_128) >> (e & 7)) & 1) {
            pp = ex2_poly2(x);
          } else {
            pp.x = ex2(x.x);
            pp.y = ex2(x.y);
          }
          acc4[e & 3] = add2(acc4[e & 3], pp);
          pk[e] = pack_bf16(pp.x, pp.y);
        }
        tc::st_32x32b_x16(tS + 64 + c * 16, pk);
      }
      const float2 acc = add2(add2(acc4[0], acc4[1]), add2(acc4[2], acc4[3]));
      l_sum += acc.x + acc.y;
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p + t);
    }
    if (cnt > 0) {
      // epilogue: O / l -> bf16, LSE
      tc::mbar_wait(bar_pv + t, 0);
      tc::fence_after_sync();
      const int row = (i0 + t) * 128 + r;
      const float inv = 1.f / l_sum;
      __nv_bfloat16* orow = O + (u * N + row) * int64_t(D);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tO + c * 32, rr);
        tc::wait_ld();
        if (row < N) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(rr[8 * e + 0]) * inv, __uint_as_float(rr[8 * e + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(rr[8 * e + 2]) * inv, __uint_as_float(rr[8 * e + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(rr[8 * e + 4]) * inv, __uint_as_float(rr[8 * e + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(rr[8 * e + 6]) * inv, __uint_as_float(rr[8 * e + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 32 + e * 8) = v;
          }
        }
      }
      if (row < N && LSE) LSE[u * N + row] = (m_used + log2f(l_sum)) * 0.69314718055994531f;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 8) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int D>
cudaError_t launch2_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                      const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                      const GtProblem* g, cudaStream_t stream, bool pdl,
                      const int32_t* order) {
  CUtensorMap mq, mk, mv, mkg, mvg;
  if (!make_tile_map(&mq, q, p.BH, p.N, D) || !make_tile_map(&mk, k, p.BH, p.N, D) ||
      !make_tile_map(&mv, v, p.BH, p.N, D))
    return cudaErrorNotSupported;
  GtArgs ga{0, 0.f, 0.f};
  if (g) {
    if (!make_tile_map(&mkg, g->kg, p.BH, g->Ng, D) || !make_tile_map(&mvg, g->vg, p.BH, g->Ng, D))
      return cudaErrorNotSupported;
    ga.Ng = g->Ng;
    ga.bias_full = logf(float(g->window)) / p.scale;
    ga.bias_last = logf(float(p.N - (g->Ng - 1) * g->window)) / p.scale;
  } else {
    mkg = mk;
    mvg = mv;
  }
  constexpr int smem = Cfg2<D>::kSmem;
  const bool dflt = p.scale == (D == 128 ? 0.088388346f : 0.125f);
  auto kern = g ? (dflt ? attn_tc2_kernel<D, true, true> : attn_tc2_kernel<D, false, true>)
                : (dflt ? attn_tc2_kernel<D, true, false> : attn_tc2_kernel<D, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned((p.Nb + 1) / 2), unsigned(p.BH));
  if (pdl) {  // programmatic dependent launch behind the refine kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads2);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mkg, mvg, ga, p.N, p.Nb, p.scale * kLog2e,
                           kv_idx, kv_cnt, reinterpret_cast<__nv_bfloat16*>(o), lse, 1, order);
    if (e != cudaSuccess) return e;
  } else {
    kern<<<grid, kThreads2, smem, stream>>>(mq, mk, mv, mkg, mvg, ga, p.N, p.Nb,
                                            p.scale * kLog2e, kv_idx, kv_cnt,
                                            reinterpret_cast<__nv_bfloat16*>(o), lse, 0, order);
  }
  e = cudaGetLastError();
  return e;
}

}  // namespace

cudaError_t launch_attn_tc2(const AttnProblem& p, const void* q, const void* k, const void* v,
                            const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                            cudaStream_t stream, const GtProblem* gt, bool pdl,
                            const int32_t* order) {
  if (p.d == 64) return launch2_d<64>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream, pdl, order);
  if (p.d == 128)
    return launch2_d<128>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream, pdl, order);
  return cudaErrorNotSupported;
}

}  // namespace blade
