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
//   warp  11    idle (an issuer per block was measured 24 % slower: an
//               issuing thread blocks at the tensor pipe's pace either way)
// TMEM (512 columns): S_A [0,128) S_B [128,256) O_A [256, 256+d) O_B [256+d, 256+2d).
// P (bf16) overwrites the upper half of its S and is the TMEM A operand of
// P V; S(n+1) of a block is issued after P V(n) of that block (the tensor
// pipe executes a thread's MMAs in order), so the commit that signals S(n+1)
// also guarantees that P V(n) finished writing O (no separate wait before a
// rescale).  Q stays in shared memory (S = Q K^T is an SS MMA).
// K and V rings are shared by both blocks, filled in the order the MMA issuer
// consumes them: A0 B0 A1 B1 ... (the shorter list simply ends earlier).
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
  // bar_q, kfull/kempty, vfull/vempty, per block: s, p, pv, sf, sl, slf
  static constexpr int kNumBar = 1 + 2 * kRingK + 2 * kRingV + 6 * 2;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  static constexpr int kSmem = kOffMisc + 16 + 1024;  // + alignment slack
  static constexpr uint32_t kColO = 256;
  // d = 64 leaves TMEM room for P outside S: P_t at [256 + 2d + 64t, +64), so
  // S_t(n+1) can be issued as soon as the softmax has read S_t(n).  Parity
  // green, but measured no faster on the Cog layer (1.05 vs 1.04 ms: the
  // softmax, not the S round trip, bounds d = 64), so off by default.
#ifndef BLADE_ATTN2_SEP_P
#define BLADE_ATTN2_SEP_P 0
#endif
  static constexpr bool kSepP = D == 64 && BLADE_ATTN2_SEP_P;
  static constexpr uint32_t kColP = 256 + 2 * D;
  // Half-tile S pipeline: S = Q K^T as two N = 64 MMAs (keys [0, 64) "early",
  // [64, 128) "late") into the two 64-column halves of the block's S region,
  // which alternate roles tile by tile: E_k (early S of tile k, then P(k))
  // and L_k (late S of tile k).  S_early(k+1) goes to L_k as soon as the
  // softmax has read S_late(k), so the softmax of tile k+1 starts on its first
  // half while the tensor core runs P V(k) and S_late(k+1) (into E_k, after
  // P V(k) has read P(k)).  The online max is lazy (threshold 2^8) per half;
  // a late-half rescale also rescales the already stored early-half P.
  // Parity green but slower (Wan 1.39-1.41 vs 1.155 ms, Cog 1.17 vs 1.04 ms,
  // interleaved A/B): two N = 64 S MMAs read Q twice, 96 instead of 64 KB of
  // shared memory per tile for S, and the d = 128 kernel is bound by shared-
  // memory bandwidth, so off by default.
#ifndef BLADE_ATTN2_HALF_S
#define BLADE_ATTN2_HALF_S 0
#endif
  static constexpr bool kHalfS = BLADE_ATTN2_HALF_S && !kSepP;
};

constexpr int kThreads2 = 384;

#ifdef BLADE_ATTN2_TRACE  // timing experiment: event timeline of one CTA
__device__ long long g_tr2[12][40];
#define TR2(ev, n)                                                                         \
  do {                                                                                     \
    if (blockIdx.x == 50 && blockIdx.y == 3 && (n) < 40) g_tr2[ev][n] = clock64();          \
  } while (0)
#else
#define TR2(ev, n) \
  do {             \
  } while (0)
#endif
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// Which of every 8 exponential pairs run on the FMA pipe (ex2_poly2) instead
// of MUFU: 1 in 8 for d = 64, none for d = 128 (interleaved A/B on B200:
// Cog 1.038 ms vs 1.045 (1 in 4) / 1.046 (none); Wan 1.166-1.171 vs 1.176
// (1 in 8) / 1.203-1.217 (1 in 4); 2 and 4 in 8 lose on both).
#ifdef BLADE_ATTN2_EMU_MASK
constexpr uint32_t kEmuMask2_64 = BLADE_ATTN2_EMU_MASK, kEmuMask2_128 = BLADE_ATTN2_EMU_MASK;
#else
// d = 64: the pattern of attn_tc2p.cu (pairs 1 and 5 of every 8), so the two
// kernels stay bit-identical
constexpr uint32_t kEmuMask2_64 = 0x22, kEmuMask2_128 = 0x00;
#endif

// Interleaved consumption order of the two blocks' items: A0 B0 A1 B1 ...
// (when one list is exhausted the other continues alone).  Calls f(t, k) for
// every item in order.
template <typename F>
BLADE_DEVINL void for_each_item(int cntA, int cntB, F&& f) {
  const int m = cntA > cntB ? cntA : cntB;
  for (int k = 0; k < m; ++k) {
    if (k < cntA) f(0, k);
    if (k < cntB) f(1, k);
  }
}

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
  uint64_t* bar_pv = bar_p + 2;              // [2] P V of block t done
  uint64_t* bar_sf = bar_pv + 2;             // [2] S of block t read out (kSepP, 4 warps)
  uint64_t* bar_sl = bar_sf + 2;             // [2] late half of S computed (kHalfS)
  uint64_t* bar_slf = bar_sl + 2;            // [2] late half of S read out (kHalfS, 4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

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
  const int cnt0 = cf0 + ngt, cnt1 = nblk == 2 ? cf1 + ngt : 0;
  const int32_t* list0 = kv_idx + (u * Nb + i0) * Nb;
  const int32_t* list1 = list0 + Nb;

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
      tc::mbar_init(bar_sf + t, 4);
      tc::mbar_init(bar_sl + t, 1);
      tc::mbar_init(bar_slf + t, 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 8) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  // registers: the two softmax warpgroups hold a 128-column S row per thread;
  // the issuer / producer warpgroup needs few (2 x 128 x 216 + 128 x 56 <= 64K)
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  if (warp == 9 || warp == 10) {
    // ===================== TMA producers (warp 9: Q and K, warp 10: V) =====
    if (lane == 0) {
      const bool isK = warp == 9;
      if (isK) {
        tc::tma_prefetch_desc(&tmQ);
        tc::tma_prefetch_desc(&tmK);
        if (kGT) tc::tma_prefetch_desc(&tmKg);
        tc::mbar_arrive_expect_tx(bar_q, nblk * C::kTile);
        for (int t = 0; t < nblk; ++t)
          for (int p = 0; p < C::kPanels; ++p)
            tc::tma_load_3d(sQ + t * C::kTile + p * C::kPanel, &tmQ, bar_q, p * 64,
                            (i0 + t) * 128, int(u));
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
      // the next block id of each list is loaded one item ahead, so the L2
      // latency of the list read overlaps the wait for a free slot
      int pre0 = cf0 > 0 ? ld_list(list0) : 0, pre1 = cf1 > 0 ? ld_list(list1) : 0;
      for_each_item(cnt0, cnt1, [&](int t, int k) {
        const int cf = t ? cf1 : cf0;
        const bool fine = !kGT || k < cf;
        const int jb = t ? pre1 : pre0;
        if (k + 1 < cf) {
          if (t) pre1 = ld_list(list1 + k + 1);
          else pre0 = ld_list(list0 + k + 1);
        }
        const int s = g % R;
        tc::mbar_wait(empty + s, ((g / R) & 1) ^ 1);
        TR2(isK ? 0 : 1, g);
        const CUtensorMap* mm = fine ? m : mg;
        const int row0 = fine ? jb * 128 : (k - cf) * 128;
        char* dst = ring + s * C::kTile;
#ifdef BLADE_ATTN2_SKIP_LOAD  // timing experiment only: MMA on stale smem
        (void)mm; (void)row0; (void)dst;
        tc::mbar_arrive(full + s);
#else
        tc::mbar_arrive_expect_tx(full + s, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(dst + p * C::kPanel, mm, full + s, p * 64, row0, int(u));
#endif
        ++g;
      });
    }
  } else if (warp == 8) {
    // ===================== MMA issuer =====================
    if (BLADE_ISSUER(lane)) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, D, 0, 1);
      const uint32_t qbase = smem_u32(sQ), kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
      int gk = 0, gv = 0;  // ring positions (interleaved order A0 B0 A1 B1 ...)
      tc::mbar_wait(bar_q, 0);
      tc::fence_after_sync();
      auto issue_S = [&](int t, int k) {  // S_t = Q_t K^T of block t's item k
        const int s = gk % C::kRingK;
        tc::mbar_wait(bar_kfull + s, (gk / C::kRingK) & 1);
        tc::fence_after_sync();
        TR2(2 + t, k);
        const uint32_t kb = kbase + s * C::kTile, qb = qbase + t * C::kTile;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          BLADE_MMA_SS(tmem + t * 128, tc::sw128_desc(qb + off, 16, 1024),
                     tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
        }
        BLADE_COMMIT(bar_s + t);
        BLADE_COMMIT(bar_kempty + s);
        ++gk;
      };
      auto issue_PV = [&](int t, int k) {  // O_t += P_t V of block t's item k
        const int s = gv % C::kRingV;
        tc::mbar_wait(bar_vfull + s, (gv / C::kRingV) & 1);
        TR2(8 + t, k);
        tc::mbar_wait(bar_p + t, k & 1);
        tc::fence_after_sync();
        TR2(4 + t, k);
        const uint32_t vb = vbase + s * C::kTile;
        const uint32_t pcol = C::kSepP ? C::kColP + t * 64 : t * 128 + 64;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          BLADE_MMA_TS(tmem + C::kColO + t * D, tmem + pcol + ks * 8,
                     tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO,
                     (k > 0 || ks > 0) ? 1 : 0);
        // bar_pv: with kSepP the softmax waits for every P V; otherwise only
        // the last one is awaited (S(n) is issued after P V(n-1), and tcgen05
        // ops of one thread complete in order), so only the last is committed
        // and every phase of the barrier has a waiter (compute-sanitizer
        // synccheck flags a phase nobody waits for)
        if (C::kSepP || k + 1 == (t ? cnt1 : cnt0)) BLADE_COMMIT(bar_pv + t);
        BLADE_COMMIT(bar_vempty + s);
        ++gv;
      };
      if constexpr (C::kHalfS) {
        constexpr uint32_t idS64 = tc::idesc_bf16(128, 64, 0, 0);
        int kslot[2] = {0, 0};
        // half h of S_t(k) (keys [64h, 64h+64)) into column half `dst` of S_t
        auto issue_Sh = [&](int t, int k, int h) {
          if (h == 0) {  // first use of item (t, k)'s K slot
            const int s = gk % C::kRingK;
            tc::mbar_wait(bar_kfull + s, (gk / C::kRingK) & 1);
            tc::fence_after_sync();
            kslot[t] = s;
            ++gk;
          }
          const int s = kslot[t];
          const uint32_t kb = kbase + s * C::kTile + h * 8192, qb = qbase + t * C::kTile;
          const uint32_t dst = t * 128 + ((k & 1) ^ h) * 64;  // early: E_k, late: L_k
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
            BLADE_MMA_SS(tmem + dst, tc::sw128_desc(qb + off, 16, 1024),
                       tc::sw128_desc(kb + off, 16, 1024), idS64, ks > 0);
          }
          BLADE_COMMIT(h ? bar_sl + t : bar_s + t);
          if (h) BLADE_COMMIT(bar_kempty + s);
        };
        auto issue_PVh = [&](int t, int k) {  // O_t += P_t(k) V, P_t(k) in E_k
          const int s = gv % C::kRingV;
          tc::mbar_wait(bar_vfull + s, (gv / C::kRingV) & 1);
          tc::mbar_wait(bar_p + t, k & 1);
          tc::fence_after_sync();
          const uint32_t vb = vbase + s * C::kTile;
          const uint32_t pcol = t * 128 + (k & 1) * 64;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            BLADE_MMA_TS(tmem + C::kColO + t * D, tmem + pcol + ks * 8,
                       tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO,
                       (k > 0 || ks > 0) ? 1 : 0);
          BLADE_COMMIT(bar_pv + t);
          BLADE_COMMIT(bar_vempty + s);
          ++gv;
        };
        for (int t = 0; t < 2; ++t)
          if ((t ? cnt1 : cnt0) > 0) {
            issue_Sh(t, 0, 0);
            issue_Sh(t, 0, 1);
          }
        const int m = cnt0 > cnt1 ? cnt0 : cnt1;
        for (int k = 0; k < m; ++k)
          for (int t = 0; t < 2; ++t) {
            const int c = t ? cnt1 : cnt0;
            if (k >= c) continue;
            if (k + 1 < c) {  // L_k free once the softmax has read S_late(k)
              tc::mbar_wait(bar_slf + t, k & 1);
              issue_Sh(t, k + 1, 0);
            }
            issue_PVh(t, k);
            if (k + 1 < c) issue_Sh(t, k + 1, 1);  // into E_k, after P V(k) read P(k)
          }
      } else {
      if (cnt0 > 0) issue_S(0, 0);
      if (cnt1 > 0) issue_S(1, 0);
      const int m = cnt0 > cnt1 ? cnt0 : cnt1;
      for (int k = 0; k < m; ++k) {
        if (C::kSepP) {
          // S(k+1) of both blocks as soon as their S(k) has been read out, then
          // the P V of item k: the tensor core computes S(k+1) while the
          // softmax turns S(k) into P(k)
          for (int t = 0; t < 2; ++t)
            if (k + 1 < (t ? cnt1 : cnt0)) {
              tc::mbar_wait(bar_sf + t, k & 1);
              issue_S(t, k + 1);
            }
          if (k < cnt0) issue_PV(0, k);
          if (k < cnt1) issue_PV(1, k);
        } else {
          if (k < cnt0) {
            issue_PV(0, k);
            if (k + 1 < cnt0) issue_S(0, k + 1);
          }
          if (k < cnt1) {
            issue_PV(1, k);
            if (k + 1 < cnt1) issue_S(1, k + 1);
          }
        }
      }
      }  // !kHalfS
      // drain: the last commits must land before the CTA's smem is released
      constexpr bool kPvEvery = C::kSepP || C::kHalfS;  // one bar_pv phase per item
      if (cnt0 > 0) tc::mbar_wait(bar_pv + 0, kPvEvery ? (cnt0 - 1) & 1 : 0);
      if (cnt1 > 0) tc::mbar_wait(bar_pv + 1, kPvEvery ? (cnt1 - 1) & 1 : 0);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::: "memory");
    // ===================== softmax of block t =====================
    const int t = warp >> 2, qw = warp & 3;
    const int cnt = t ? cnt1 : cnt0;
    const int cnt_fine = t ? cf1 : cf0;
    const int32_t* list = t ? list1 : list0;
    const uint32_t lane_base = uint32_t(qw * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + C::kColO + t * D;
    const int r = qw * 32 + lane;
    float m_used = -INFINITY, l_sum = 0.f;
    int jn = cnt_fine > 0 ? ld_list(list) : 0;  // block id, loaded one tile ahead
    if constexpr (C::kHalfS) {
      const float2 sl2 = make_float2(scale_log2, scale_log2);
      // rescale O_t (and l) by f; O_t must be current
      auto rescale_o = [&](float f) {
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t rr[32];
          tc::ld_32x32b_x32(tO + c * 32, rr);
          tc::wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) * f);
          tc::st_32x32b_x32(tO + c * 32, rr);
        }
      };
      // 64 scores of half h (keys [64h, 64h+64)) from TMEM column base `col`,
      // masked / biased; returns their max
      auto load_half = [&](uint32_t col, int h, int n, int jb, float (&x)[64]) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t rr[32];
          tc::ld_32x32b_x32(col + c * 32, rr);
#pragma unroll
          for (int e = 0; e < 32; ++e) x[c * 32 + e] = __uint_as_float(rr[e]);
        }
        tc::wait_ld();
        const bool fine = !kGT || n < cnt_fine;
        const int valid = (fine ? N - jb * 128 : gt.Ng - (n - cnt_fine) * 128) - 64 * h;
        if (valid < 64) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= valid) x[c] = -INFINITY;
        }
        if (kGT && !fine) {
          const int last = gt.Ng - 1 - (n - cnt_fine) * 128 - 64 * h;
#pragma unroll
          for (int c = 0; c < 64; ++c) x[c] += c == last ? gt.bias_last : gt.bias_full;
        }
        float t4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float m4 = fmaxf(x[g], x[g + 4]);
#pragma unroll
          for (int c = g + 8; c < 64; c += 8) m4 = fmaxf(m4, fmaxf(x[c], x[c + 4]));
          t4[g] = m4;
        }
        return fmaxf(fmaxf(t4[0], t4[1]), fmaxf(t4[2], t4[3]));
      };
      // P = 2^(s scale - m_used) of a half -> packed bf16 columns [32h, 32h+32) of E
      auto exp_store = [&](const float (&x)[64], uint32_t ecol, int h) {
        float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};
        const float2 nm = make_float2(-m_used, -m_used);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 xx = fma2(make_float2(x[c * 32 + 2 * e], x[c * 32 + 2 * e + 1]), sl2, nm);
            float2 pp;
            if (((D == 64 ? kEmuMask2_64 : kEmuMask2_128) >> (e & 7)) & 1) {
              pp = ex2_poly2(xx);
            } else {
              pp.x = ex2(xx.x);
              pp.y = ex2(xx.y);
            }
            acc4[e & 3] = add2(acc4[e & 3], pp);
            pk[e] = pack_bf16(pp.x, pp.y);
          }
          tc::st_32x32b_x16(ecol + 32 * h + c * 16, pk);
        }
        const float2 acc = add2(add2(acc4[0], acc4[1]), add2(acc4[2], acc4[3]));
        l_sum += acc.x + acc.y;
      };
      for (int n = 0; n < cnt; ++n) {
        const int jb = jn;
        if (n + 1 < cnt_fine) jn = ld_list(list + n + 1);
        const uint32_t E = tS + (n & 1) * 64, Lc = tS + ((n & 1) ^ 1) * 64;
        float x[64];
        // ---- early half (keys [0, 64)) in E_n
        tc::mbar_wait(bar_s + t, n & 1);
        tc::fence_after_sync();
        {
          const float mxs = load_half(E, 0, n, jb, x) * scale_log2;
          if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold)) {
            const float m_new = fmaxf(m_used, mxs);
            if (n > 0) {  // O_t current: P V(n-1) done
              tc::mbar_wait(bar_pv + t, (n - 1) & 1);
              tc::fence_after_sync();
              const float f = ex2(m_used - m_new);
              l_sum *= f;
              rescale_o(f);
            }
            m_used = m_new;
          }
        }
        exp_store(x, E, 0);
        // ---- late half (keys [64, 128)) in L_n
        tc::mbar_wait(bar_sl + t, n & 1);
        tc::fence_after_sync();
        {
          const float mxs = load_half(Lc, 1, n, jb, x) * scale_log2;
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(bar_slf + t);  // L_n may take S_early(n+1)
          if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold)) {
            // S_late(n) complete => P V(n-1) complete (issued before it)
            const float m_new = fmaxf(m_used, mxs);
            const float f = ex2(m_used - m_new);
            l_sum *= f;
            if (n > 0) rescale_o(f);
            tc::wait_st();
            {  // the early half's P, already stored with the old max
              uint32_t rr[32];
              tc::ld_32x32b_x32(E, rr);
              tc::wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const float2 v = unpack_bf16(rr[e]);
                rr[e] = pack_bf16(v.x * f, v.y * f);
              }
              tc::st_32x32b_x32(E, rr);
            }
            m_used = m_new;
          }
        }
        exp_store(x, E, 1);
        tc::wait_st();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(bar_p + t);
      }
    } else
    for (int n = 0; n < cnt; ++n) {
      const int jb = jn;
      if (n + 1 < cnt_fine) jn = ld_list(list + n + 1);
      tc::mbar_wait(bar_s + t, n & 1);
      tc::fence_after_sync();
      if (lane == 0 && qw == 0) TR2(6 + t, n);
#ifdef BLADE_ATTN2_SKIP_SOFTMAX  // timing experiment only: MMA / TMA pipeline alone
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0 && C::kSepP) tc::mbar_arrive(bar_sf + t);
      if (lane == 0) tc::mbar_arrive(bar_p + t);
      continue;
#endif
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tS + c * 32, rr);
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(rr[e]);
      }
      tc::wait_ld();
      if (C::kSepP) {  // S_t's columns may be overwritten by S_t(n+1) now
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(bar_sf + t);
      }
      const bool fine = !kGT || n < cnt_fine;
      const int valid = fine ? N - jb * 128 : gt.Ng - (n - cnt_fine) * 128;
      if (valid < 128) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c >= valid) s[c] = -INFINITY;
      }
      if (kGT && !fine) {  // + ln(n_w) on the pooled region, raw-score units
        const int last = gt.Ng - 1 - (n - cnt_fine) * 128;
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
      if (C::kSepP && n > 0) {  // P V_t(n-1) done: O_t current and P_t's columns free
        tc::mbar_wait(bar_pv + t, (n - 1) & 1);
        tc::fence_after_sync();
      }
      // warp-uniform (tcgen05.ld/st are .sync.aligned); always true for n = 0.
      // O_t is current (kSepP: waited above; else S_t(n) was issued after
      // P V_t(n-1) and has completed).
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
        tc::st_32x32b_x16(C::kSepP ? tmem + lane_base + C::kColP + t * 64 + c * 16
                                   : tS + 64 + c * 16,
                          pk);
      }
      const float2 acc = add2(add2(acc4[0], acc4[1]), add2(acc4[2], acc4[3]));
      l_sum += acc.x + acc.y;
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p + t);
      if (lane == 0 && qw == 0) TR2(10 + t, n);
    }
    if (cnt > 0) {
      // epilogue: O / l -> bf16, LSE
      tc::mbar_wait(bar_pv + t, (C::kSepP || C::kHalfS) ? (cnt - 1) & 1 : 0);
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
#ifdef BLADE_ATTN2_TRACE
  {
    static int calls = 0;
    long long h[12][40];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h, g_tr2, sizeof(h));
    if (++calls == 10) {
      const long long t0 = h[0][0];
      fprintf(stderr, "k : Kld Vld | S_A S_B | Vrdy_A PV_A Vrdy_B PV_B | smA_in smA_out smB_in smB_out (cycles)\n");
      for (int n = 0; n < 24; ++n)
        fprintf(stderr, "%2d: %6lld %6lld | %6lld %6lld | %6lld %6lld %6lld %6lld | %6lld %6lld %6lld %6lld\n", n,
                h[0][n] - t0, h[1][n] - t0, h[2][n] - t0, h[3][n] - t0, h[8][n] - t0, h[4][n] - t0,
                h[9][n] - t0, h[5][n] - t0, h[6][n] - t0, h[10][n] - t0, h[7][n] - t0, h[11][n] - t0);
    }
  }
#endif
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
