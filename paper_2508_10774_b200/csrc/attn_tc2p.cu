// attn_tc2p.cu — the pair kernel of attn_tc2.cu as a PERSISTENT kernel: one
// CTA per SM walks the (unit, query-block pair) items (PAPER.md P:133 block-
// sparse attention; ASA_GT global tokens P:135 as extra tiles).
//
// Why: the non-persistent pair kernel runs 10.4 waves on the Wan layer; every
// CTA pays TMEM allocation, barrier setup, the Q load and the first K/V tiles
// before its first MMA, and its epilogue (O out of TMEM, 64 KB stored) runs
// with the tensor core idle (~4 % of the kernel, plus 6.6 % idle SM time at
// the wave boundaries).  Here those overlap the neighbouring items: Q of item
// n+1 is loaded as soon as item n's last S MMA has consumed Q (bar_qfree), its
// first S MMAs run while the softmax warps still write item n's O, and the
// K/V rings, S/P barriers and TMEM stay live across items (phases counted
// globally).  The first P V of a block in item n+1 (accumulate = 0, it
// overwrites O_t) is issued only after that block's softmax warps arrived on
// bar_p for item n+1's first tile, i.e. after they read O_t out.
//
// Warp roles (384 threads), TMEM and the per-item schedule are those of
// attn_tc2.cu (default path: S in TMEM with P over its upper half, ping-pong
// of the two blocks' softmax warpgroups).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

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

#ifndef BLADE_ATTN2P_RK64
#define BLADE_ATTN2P_RK64 6  // d = 64 K / V ring slots (16 KB each)
#endif
#ifndef BLADE_ATTN2P_RV64
#define BLADE_ATTN2P_RV64 6
#endif
#ifndef BLADE_ATTN2P_PCHUNK
#define BLADE_ATTN2P_PCHUNK 1  // d = 128: P handed over in 1, 2 or 4 key chunks
#endif
#ifndef BLADE_ATTN2P_SEPP
#define BLADE_ATTN2P_SEPP 1  // d = 64: P outside S (below); Cog attention 0.920-0.926 vs 0.948 ms
#endif

constexpr int kThreadsP = 384;  // 8 softmax warps, MMA issuer, K / Q and V producers, spare

template <int D>
struct CfgP {
  static constexpr int kTile = 128 * D * 2;  // one Q / K / V tile
  static constexpr int kPanels = D / 64;     // 128-byte SW128 panels along d
  static constexpr int kPanel = 128 * 128;
  static constexpr int kRingK = D == 128 ? 3 : BLADE_ATTN2P_RK64;
  static constexpr int kRingV = D == 128 ? 2 : BLADE_ATTN2P_RV64;
  static constexpr int kOffQ = 0;  // Q_A, Q_B
  static constexpr int kOffRingK = 2 * kTile;
  static constexpr int kOffRingV = kOffRingK + kRingK * kTile;
  static constexpr int kOffBar = kOffRingV + kRingV * kTile;
  // bar_q, bar_qfree, kfull/kempty, vfull/vempty, per block: s, p, pv, sf, item queue full/empty
  static constexpr int kNumBar = 2 + 2 * kRingK + 2 * kRingV + 4 * 2 + 3 * 2 + 2 * 4;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;   // tmem slot (16 B)
  static constexpr int kOffItems = kOffMisc + 16;           // int [4] claimed item queue
  static constexpr int kSmem = kOffItems + 16 + 1024;       // + alignment slack
  static constexpr uint32_t kColO = 256;
  // registers: the kernel runs at 168, the four role warps drop to
  // kRegLow, the softmax warps take the rest
  static constexpr int kRegLow = 72;
  static constexpr int kRegHigh = 216;
  // d = 64 leaves TMEM room for P outside S: P_t at [256 + 2d + 64t, +64).
  // S_t(n+1) is then issued as soon as the softmax has read S_t(n) (bar_sf),
  // and the softmax waits for P V_t(n-1) only right before it stores P_t(n),
  // so a block's softmax runs tile after tile without the S round trip.
  static constexpr bool kSepP = D == 64 && BLADE_ATTN2P_SEPP;
  static constexpr uint32_t kColP = 256 + 2 * D;
  // P V of block t's tile issued chunk by chunk as the softmax stores P
  static constexpr int kPChunks = kSepP ? 1 : BLADE_ATTN2P_PCHUNK;
};
#ifndef BLADE_ATTN2P_QPREFETCH
#define BLADE_ATTN2P_QPREFETCH 1  // L2 prefetch of the next item's Q while its slot drains
#endif
constexpr float kRescaleThresholdP = 8.0f;  // log2 units
// exponential pairs on the FMA pipe (bit e of the mask: pair e of each 16-pair
// chunk of a row; as attn_tc2.cu), d = 64: pairs 1 and 5 of every 8 (with P in its own columns; Cog attention 0.891 vs 0.917 ms for 0x01,
// 0.998 for none, 0.894 for 0x11, 0.96 for 3 in 8, 1.02 for 0x55)
#ifndef BLADE_ATTN2P_EMU64
#define BLADE_ATTN2P_EMU64 0x2222
#endif
#ifndef BLADE_ATTN2P_EMU128
#define BLADE_ATTN2P_EMU128 0x00
#endif
constexpr uint32_t kEmuMaskP64 = BLADE_ATTN2P_EMU64, kEmuMaskP128 = BLADE_ATTN2P_EMU128;

// One item = query blocks A = 2x, B = 2x + 1 of one unit.
struct PairItem {
  int64_t u;
  int i0, nblk, cf0, cf1, cnt0, cnt1;
  const int32_t* list0;
  const int32_t* list1;
};

template <int D, bool kDefaultScale, bool kGT>
__global__ void __launch_bounds__(kThreadsP, 1)
    attn_tc2p_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmKg,
                     const __grid_constant__ CUtensorMap tmVg, const GtArgs gt, int N, int Nb,
                     int nitems, int* __restrict__ work, float scale_log2_rt,
                     const int32_t* __restrict__ kv_idx,
                     const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ O,
                     float* __restrict__ LSE, int pdl, const int32_t* __restrict__ order) {
  using C = CfgP<D>;
  const float scale_log2 = kDefaultScale ? DefaultScale<D>::kScaleLog2 : scale_log2_rt;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem + C::kOffQ;
  char* sRingK = smem + C::kOffRingK;
  char* sRingV = smem + C::kOffRingV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;          // Q tiles of the current item loaded
  uint64_t* bar_qfree = bars + 1;  // the item's last S MMA done: Q may be reloaded
  uint64_t* bar_kfull = bars + 2;
  uint64_t* bar_kempty = bar_kfull + C::kRingK;
  uint64_t* bar_vfull = bar_kempty + C::kRingK;
  uint64_t* bar_vempty = bar_vfull + C::kRingV;
  uint64_t* bar_s = bar_vempty + C::kRingV;  // [2] S of block t computed
  uint64_t* bar_p = bar_s + 2;               // [2] P of block t written (4 warp arrivals)
  uint64_t* bar_pv = bar_p + 2;              // [2] last P V of block t in an item done
  uint64_t* bar_sf = bar_pv + 2;             // [2] S_t read out by its 4 softmax warps (kSepP)
  uint64_t* bar_ph = bar_sf + 2;             // [2][3] P_t chunk c < kPChunks - 1 written (4 warps)
  uint64_t* bar_ifull = bar_ph + 6;          // [4] item queue slot written (warp 9)
  uint64_t* bar_iempty = bar_ifull + 4;      // [4] slot read by the other 10 warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  int* sItem = reinterpret_cast<int*>(smem + C::kOffItems);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int npair = (Nb + 1) / 2;
  const int ngt = kGT ? (gt.Ng + 127) / 128 : 0;
  // blade_asa_fwd: rows K-mask.4 recomputes carry a provisional negative count;
  // the first item of this CTA that meets one waits for that grid, and from
  // then on every list is read through L2 (ld.global.cg: K-mask.4 rewrote it
  // while this grid ran; a stale L1 line of an earlier item must not be used)
  bool waited = false;
  auto ld_list = [&waited](const int32_t* p) { return waited ? __ldcg(p) : __ldg(p); };
  // Items are claimed dynamically (warp 9 draws the next index from a global
  // counter and queues it in shared memory; the other roles take the queue
  // in order), so items of different length (tau mode) balance over the SMs
  // like the CTAs of a non-persistent grid; with an LPT order the longest
  // items are drawn first.  Returns false at the end-of-work sentinel.
  // consumers of queue entry n: a whole warp (one arrival after every lane
  // read the slot) or a single thread (the V producer's lane 0)
  auto take_item = [&](int n, bool whole_warp) -> int {
    const int slot = n & 3;
    tc::mbar_wait(bar_ifull + slot, (n >> 2) & 1);
    const int x = sItem[slot];
    if (whole_warp) __syncwarp();
    if (!whole_warp || lane == 0) tc::mbar_arrive(bar_iempty + slot);
    return x;
  };
  auto get_item = [&](int x, PairItem& it) -> bool {
    if (x < 0) return false;
    const int64_t id = order ? int64_t(__ldg(order + x)) : x;  // LPT: longest first
    it.u = id / npair;
    it.i0 = 2 * int(id % npair);
    it.nblk = (it.i0 + 1 < Nb) ? 2 : 1;
    const int32_t* cp = kv_cnt + it.u * Nb + it.i0;
    int c0 = waited ? __ldcg(cp) : cp[0];
    int c1 = it.nblk == 2 ? (waited ? __ldcg(cp + 1) : cp[1]) : 0;
    if (pdl && !waited && (c0 < 0 || c1 < 0)) {
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      waited = true;
      c0 = __ldcg(cp);
      c1 = it.nblk == 2 ? __ldcg(cp + 1) : 0;
    }
    it.cf0 = c0;
    it.cf1 = c1;
    it.cnt0 = c0 + ngt;
    it.cnt1 = it.nblk == 2 ? c1 + ngt : 0;
    it.list0 = kv_idx + (it.u * Nb + it.i0) * Nb;
    it.list1 = it.list0 + Nb;
    return true;
  };

  if (warp == 9 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    tc::mbar_init(bar_qfree, 1);
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
      for (int c = 0; c < 3; ++c) tc::mbar_init(bar_ph + 3 * t + c, 4);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(bar_ifull + i, 1);
      tc::mbar_init(bar_iempty + i, 10);  // V producer, MMA issuer, 8 softmax warps
    }
    tc::fence_barrier_init();
  }
  if (warp == 8) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 8) {
    // the CTA holds 384 x 168 registers: 128 x (168 - 72) freed here cover the
    // 256 x (216 - 168) the softmax warpgroups take (setmaxnreg.inc blocks
    // until the pool has them)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::kRegLow) : "memory");
    if (warp == 9 || warp == 10) {
      // ===================== TMA producers (warp 9: Q and K, warp 10: V) =====
      if (lane == 0) {
        const bool isK = warp == 9;
        if (isK) {
          tc::tma_prefetch_desc(&tmQ);
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
        int g = 0;  // ring position, continuous over the items
        PairItem it;
        for (int n = 0;; ++n) {
          int x;
          if (isK) {  // claim the next item and queue it for the other roles
            const int slot = n & 3;
            if (n >= 4) tc::mbar_wait(bar_iempty + slot, ((n >> 2) - 1) & 1);
            x = atomicAdd(work, 1);
            if (x >= nitems) x = -1;
            sItem[slot] = x;
            tc::mbar_arrive(bar_ifull + slot);
          } else {
            x = take_item(n, false);  // lane 0 of warp 10 only
          }
          if (!get_item(x, it)) break;
          if (isK) {  // Q_A, Q_B of this item, once the previous item's S MMAs are done
            if (n > 0) {  // meanwhile pull them into L2
              for (int t = 0; t < (BLADE_ATTN2P_QPREFETCH ? it.nblk : 0); ++t)
                for (int p = 0; p < C::kPanels; ++p)
                  tc::tma_prefetch_3d(&tmQ, p * 64, (it.i0 + t) * 128, int(it.u));
              tc::mbar_wait(bar_qfree, (n - 1) & 1);
            }
            tc::mbar_arrive_expect_tx(bar_q, it.nblk * C::kTile);
            for (int t = 0; t < it.nblk; ++t)
              for (int p = 0; p < C::kPanels; ++p)
                tc::tma_load_3d(sQ + t * C::kTile + p * C::kPanel, &tmQ, bar_q, p * 64,
                                (it.i0 + t) * 128, int(it.u));
          }
          int pre0 = it.cf0 > 0 ? ld_list(it.list0) : 0;
          int pre1 = it.cf1 > 0 ? ld_list(it.list1) : 0;
          const int mx = it.cnt0 > it.cnt1 ? it.cnt0 : it.cnt1;
          for (int k = 0; k < mx; ++k) {
            for (int t = 0; t < 2; ++t) {  // consumption order A0 B0 A1 B1 ...
              if (k >= (t ? it.cnt1 : it.cnt0)) continue;
              const int cf = t ? it.cf1 : it.cf0;
              const bool fine = !kGT || k < cf;
              const int jb = t ? pre1 : pre0;
              if (k + 1 < cf) {
                if (t) pre1 = ld_list(it.list1 + k + 1);
                else pre0 = ld_list(it.list0 + k + 1);
              }
              const int s = g % R;
              tc::mbar_wait(empty + s, ((g / R) & 1) ^ 1);
              tc::mbar_arrive_expect_tx(full + s, C::kTile);
              for (int p = 0; p < C::kPanels; ++p)
                tc::tma_load_3d(ring + s * C::kTile + p * C::kPanel, fine ? m : mg, full + s,
                                p * 64, fine ? jb * 128 : (k - cf) * 128, int(it.u));
              ++g;
            }
          }
        }
      }
    } else if (warp == 8) {
      // ===================== MMA issuer =====================
      if (BLADE_ISSUER(lane)) {
        constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idO = tc::idesc_bf16(128, D, 0, 1);
        const uint32_t qbase = smem_u32(sQ), kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
        int gk = 0, gv = 0;         // ring positions, continuous over the items
        int np[2] = {0, 0};         // bar_p phases consumed per block
        int gs[2] = {0, 0};         // S_t issued so far (kSepP: bar_sf phases)
        PairItem it;
        for (int n = 0; get_item(take_item(n, BLADE_MMA_WARP != 0), it); ++n) {
          tc::mbar_wait(bar_q, n & 1);
          tc::fence_after_sync();
          int s_left = it.cnt0 + it.cnt1;  // S MMAs of this item still to issue
          auto issue_S = [&](int t) {  // S_t = Q_t K^T of block t's next tile
            const int s = gk % C::kRingK;
            if (C::kSepP && gs[t] > 0) tc::mbar_wait(bar_sf + t, (gs[t] - 1) & 1);  // S_t read
            ++gs[t];
            tc::mbar_wait(bar_kfull + s, (gk / C::kRingK) & 1);
            tc::fence_after_sync();
            const uint32_t kb = kbase + s * C::kTile, qb = qbase + t * C::kTile;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
              const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
              BLADE_MMA_SS(tmem + t * 128, tc::sw128_desc(qb + off, 16, 1024),
                           tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
            }
            BLADE_COMMIT(bar_s + t);
            BLADE_COMMIT(bar_kempty + s);
            if (--s_left == 0) BLADE_COMMIT(bar_qfree);  // Q no longer read
            ++gk;
          };
          auto issue_PV = [&](int t, int k) {  // O_t += P_t V of block t's tile k
            const int s = gv % C::kRingV;
            tc::mbar_wait(bar_vfull + s, (gv / C::kRingV) & 1);
            const uint32_t vb = vbase + s * C::kTile;
            constexpr int kPer = 8 / C::kPChunks;  // MMAs (16 keys each) per chunk
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              if (ks % kPer == 0) {  // this chunk of P stored
                const int c = ks / kPer;
                tc::mbar_wait(c == C::kPChunks - 1 ? bar_p + t : bar_ph + 3 * t + c, np[t] & 1);
                tc::fence_after_sync();
              }
              BLADE_MMA_TS(tmem + C::kColO + t * D,
                           tmem + (C::kSepP ? C::kColP + t * 64 : t * 128 + 64) + ks * 8,
                           tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO,
                           (k > 0 || ks > 0) ? 1 : 0);
            }
            ++np[t];
            // without kSepP only the item's last P V is awaited (the epilogue):
            // S(k+1) is issued after P V(k) and one thread's tcgen05 ops
            // complete in order; with kSepP the softmax waits for every P V
            if (C::kSepP || k + 1 == (t ? it.cnt1 : it.cnt0)) BLADE_COMMIT(bar_pv + t);
            BLADE_COMMIT(bar_vempty + s);
            ++gv;
          };
          if (s_left == 0) BLADE_COMMIT(bar_qfree);  // an empty item still frees Q
          if (it.cnt0 > 0) issue_S(0);
          if (it.cnt1 > 0) issue_S(1);
          const int m = it.cnt0 > it.cnt1 ? it.cnt0 : it.cnt1;
          for (int k = 0; k < m; ++k) {
            if (C::kSepP) {
              // S(k+1) of both blocks as soon as S(k) has been read out, then
              // the P V of tile k
              if (k + 1 < it.cnt0) issue_S(0);
              if (k + 1 < it.cnt1) issue_S(1);
              if (k < it.cnt0) issue_PV(0, k);
              if (k < it.cnt1) issue_PV(1, k);
              continue;
            }
            if (k < it.cnt0) {
              issue_PV(0, k);
              if (k + 1 < it.cnt0) issue_S(0);
            }
            if (k < it.cnt1) {
              issue_PV(1, k);
              if (k + 1 < it.cnt1) issue_S(1);
            }
          }
        }
        // kSepP: consume the read-out of each block's last S (every mbarrier
        // phase that completes has a waiter)
        if (C::kSepP)
          for (int t = 0; t < 2; ++t)
            if (gs[t] > 0) tc::mbar_wait(bar_sf + t, (gs[t] - 1) & 1);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::kRegHigh) : "memory");
    // ===================== softmax of block t =====================
    // warp (t, qw): rows 32 qw .. 32 qw + 31 (TMEM lane quarter qw) of block t
    const int t = warp >> 2, qw = warp & 3;
    const uint32_t lane_base = uint32_t(qw * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + C::kColO + t * D;
    // P over the upper half of S_t, or (kSepP) in its own columns
    const uint32_t tP = C::kSepP ? tmem + lane_base + C::kColP + t * 64 : tS + 64;
    const int r = qw * 32 + lane;
    const float2 sl2 = make_float2(scale_log2, scale_log2);
    int ns = 0, npv = 0;  // bar_s / bar_pv phases consumed
    PairItem it;
    for (int item_n = 0; get_item(take_item(item_n, true), it); ++item_n) {
      const int cnt = t ? it.cnt1 : it.cnt0;
      const int cnt_fine = t ? it.cf1 : it.cf0;
      const int32_t* list = t ? it.list1 : it.list0;
      float m_used = -INFINITY, l_sum = 0.f;
      int jn = cnt_fine > 0 ? ld_list(list) : 0;  // block id, loaded one tile ahead
      for (int n = 0; n < cnt; ++n) {
        const int jb = jn;
        if (n + 1 < cnt_fine) jn = ld_list(list + n + 1);
        tc::mbar_wait(bar_s + t, ns & 1);
        ++ns;
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
        if (C::kSepP) {  // S_t's columns may be overwritten by S_t(n+1) now
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(bar_sf + t);
        }
        bool pv_done = !C::kSepP || n == 0;  // P V_t(n-1) complete (kSepP)
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
        // warp-uniform (tcgen05.ld/st are .sync.aligned); always true for n = 0.
        // O_t is current: S_t(n) was issued after P V_t(n-1) and has completed
        // (kSepP: waited for here).
        if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThresholdP)) {
          const float m_new = fmaxf(m_used, mxs);
          if (n > 0) {
            if (!pv_done) {
              tc::mbar_wait(bar_pv + t, npv & 1);
              ++npv;
              tc::fence_after_sync();
              pv_done = true;
            }
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
        const float2 nm = make_float2(-m_used, -m_used);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 x = fma2(make_float2(s[c * 32 + 2 * e], s[c * 32 + 2 * e + 1]), sl2, nm);
            float2 pp;
            if (((D == 64 ? kEmuMaskP64 : kEmuMaskP128) >> (e & 15)) & 1) {
              pp = ex2_poly2(x);
            } else {
              pp.x = ex2(x.x);
              pp.y = ex2(x.y);
            }
            acc4[e & 3] = add2(acc4[e & 3], pp);
            pk[e] = pack_bf16(pp.x, pp.y);
          }
          if (c == 0 && !pv_done) {  // kSepP: P_t's columns are free once P V_t(n-1) is done
            tc::mbar_wait(bar_pv + t, npv & 1);
            ++npv;
            tc::fence_after_sync();
          }
          tc::st_32x32b_x16(tP + c * 16, pk);
          constexpr int kCPer = 4 / C::kPChunks;  // 32-key store chunks per P chunk
          if (C::kPChunks > 1 && c % kCPer == kCPer - 1 && c < 3) {  // P V of this chunk may start
            tc::wait_st();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(bar_ph + 3 * t + c / kCPer);
          }
        }
        const float2 acc = add2(add2(acc4[0], acc4[1]), add2(acc4[2], acc4[3]));
        l_sum += acc.x + acc.y;
        tc::wait_st();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(bar_p + t);
      }
      if (cnt > 0) {
        // epilogue: O / l -> bf16, LSE.  The next item's first P V into O_t
        // waits for this warpgroup's bar_p arrival of its first tile, which
        // follows these O reads in program order.
        tc::mbar_wait(bar_pv + t, npv & 1);
        ++npv;
        tc::fence_after_sync();
        const int row = (it.i0 + t) * 128 + r;
        const float inv = 1.f / l_sum;
        __nv_bfloat16* orow = O + (it.u * N + row) * int64_t(D);
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
        if (row < N && LSE) LSE[it.u * N + row] = (m_used + log2f(l_sum)) * 0.69314718055994531f;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 8) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n > 0 ? n : 148;
}

template <int D>
cudaError_t launchp_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                      const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                      const GtProblem* g, cudaStream_t stream, bool pdl, const int32_t* order,
                      int* work, bool work_zeroed) {
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
  constexpr int smem = CfgP<D>::kSmem;
  static_assert(smem <= 227 * 1024, "dynamic shared memory per CTA");
  const bool dflt = p.scale == (D == 128 ? 0.088388346f : 0.125f);
  auto kern = g ? (dflt ? attn_tc2p_kernel<D, true, true> : attn_tc2p_kernel<D, false, true>)
                : (dflt ? attn_tc2p_kernel<D, true, false> : attn_tc2p_kernel<D, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int nitems = int((p.Nb + 1) / 2 * p.BH);  // BH <= 65535, Nb <= 512
  if (!work_zeroed) {  // the item counter
    e = cudaMemsetAsync(work, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
  }
  const int sms = num_sms();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(nitems < sms ? nitems : sms));
  cfg.blockDim = dim3(kThreadsP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;  // programmatic dependent launch behind the refine kernel
  e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mkg, mvg, ga, p.N, p.Nb, nitems, work,
                         p.scale * kLog2e, kv_idx, kv_cnt, reinterpret_cast<__nv_bfloat16*>(o),
                         lse, pdl ? 1 : 0, order);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_tc2p(const AttnProblem& p, const void* q, const void* k, const void* v,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                             int* work, bool work_zeroed, cudaStream_t stream,
                             const GtProblem* gt, bool pdl, const int32_t* order) {
  if (p.d == 64)
    return launchp_d<64>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream, pdl, order, work,
                         work_zeroed);
  if (p.d == 128)
    return launchp_d<128>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream, pdl, order, work,
                          work_zeroed);
  return cudaErrorNotSupported;
}

}  // namespace blade
