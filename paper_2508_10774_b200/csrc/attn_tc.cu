// attn_tc.cu — block-sparse attention forward for sm_100a on the 5th-gen
// tensor cores (tcgen05 + TMEM + TMA).  PAPER.md P:133 (Step 2.2 (1),
// "Standard ASA ... integrated with a block-sparse attention kernel").
//
// CTA = one query block (128 rows) of one unit, walking its kept-block list
// kv_idx[u, i, 0:kv_cnt).  Every CTA is independent, so content-adaptive
// lists of any length and order cost nothing extra.  Warp roles:
//   warps 0-3  softmax (thread = query row = TMEM lane)
//   warp  4    tcgen05.mma issuer (one thread) + TMEM allocator
//   warp  5    TMA producer (one thread): Q once, then K_j into the K ring
//   warp  6    TMA producer (one thread): V_j into the V ring
//   warp  7    idle (completes the second warpgroup)
// TMEM (512 columns): S_0 [0,128) S_1 [128,256) O [256, 256+d) Q [256+d, +d/2).
// Q is copied into TMEM once, so S = Q K^T takes its A operand from TMEM and
// the tensor core streams only K and V from shared memory (an SS MMA at
// M = N = 128 would need the whole 128 B/clk of smem bandwidth by itself).
// S is double-buffered, so S(n+1) = Q K(n+1)^T is computed while the softmax
// works on S(n); P(n) (bf16) overwrites the upper half of S(n)'s buffer and
// feeds the P V MMA straight from TMEM.  MMA issue order:
//   S(0) S(1) | PV(0) S(2) | PV(1) S(3) | ...
// The softmax is bound by the FMA and MUFU pipes, so the default softmax
// scale is baked in (immediate-form FFMA), arithmetic is packed fp32x2; exponentials can run
// partly as an FMA-pipe polynomial (BLADE_ATTN_EMU_MASK; off by default: fewer instructions
// measured faster than balancing the pipes).  O is rescaled lazily (only
// when a row max grows by more than 2^8).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"
#include "attn_common.cuh"
#include "tma_host.h"

namespace blade {
namespace {

using attn::DefaultScale;
using attn::ex2_poly2;
using attn::GtArgs;

template <int D>
struct Cfg {
  static constexpr int kTile = 128 * D * 2;          // Q tile / K slot / V slot bytes
  static constexpr int kPanels = D / 64;             // 128-byte SW128 panels along d
  static constexpr int kPanel = 128 * 128;           // 128 rows x 128 B
#ifndef BLADE_ATTN_KRING
#define BLADE_ATTN_KRING 3
#endif
#ifndef BLADE_ATTN_VRING
#define BLADE_ATTN_VRING 3
#endif
  // separate K and V rings: a K slot frees as soon as its S MMA completes,
  // a V slot only after P V, so sharing one ring starves the K prefetch
  static constexpr int kRingK = D == 128 ? BLADE_ATTN_KRING : 2 * BLADE_ATTN_KRING;
  static constexpr int kRingV = D == 128 ? BLADE_ATTN_VRING : 2 * BLADE_ATTN_VRING;
  static constexpr int kOffRingK = kTile;
  static constexpr int kOffRingV = kOffRingK + kRingK * kTile;
  static constexpr int kOffBar = kOffRingV + kRingV * kTile;
  // the Q tile's smem is free once Q sits in TMEM: it becomes one more V slot
  static constexpr int kRingVx = kRingV + 1;
  static constexpr int kNumBar = 1 + 2 * kRingK + 2 * kRingVx + 5 + 1;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  // row-max exchange between the two column halves of a row (bf16, rounded
  // up): [S buffer][half][row]; reused for the final l exchange (fp32)
  static constexpr int kOffXch = kOffMisc + 16;
  static constexpr int kSmem = kOffXch + 1024 + 1024;  // + alignment slack
  static constexpr uint32_t kColO = 256;
  static constexpr uint32_t kColQ = 256 + D;  // Q in TMEM (bf16 pairs): D / 2 columns
};

// Softmax warps: kSplit x 4.  With kSplit = 2 each query row is shared by two
// warps (one per 64-column half of S, same TMEM lane quarter): twice the
// warps to hide the softmax's latency chain (ld -> max -> exp -> st -> arrive)
// at the cost of one row-max exchange per tile.
#ifndef BLADE_ATTN_SPLIT
#define BLADE_ATTN_SPLIT 1  // 2 measured slower on B200 (Wan 1.252 vs 1.231 ms, Cog 1.221 vs 1.133 ms)
#endif
constexpr int kSplit = BLADE_ATTN_SPLIT;
constexpr int kSoftWarps = 4 * kSplit;
constexpr int kMmaWarp = kSoftWarps;      // tcgen05.mma issuer + TMEM allocator
constexpr int kLoadKWarp = kSoftWarps + 1;  // TMA: Q, then K
constexpr int kLoadVWarp = kSoftWarps + 2;  // TMA: V
constexpr int kThreads = 32 * (kSoftWarps + 3);
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P may reach 2^8 before O is rescaled
// which of every 8 exponential PAIRS run on the FMA pipe (bit k: pair k)
#ifndef BLADE_ATTN_EMU_MASK
#define BLADE_ATTN_EMU_MASK 0x00  // none: measured 3 % faster than 1 in 4 (0x11) on the Wan layer
#endif
constexpr uint32_t kEmuMask = BLADE_ATTN_EMU_MASK;

#ifdef BLADE_TC_DEBUG
#define TC_DBG(i, v)          \
  do {                        \
    if (dbg_on) dbg[i] = (v); \
  } while (0)
#else
#define TC_DBG(i, v) \
  do {               \
  } while (0)
#endif

#ifdef BLADE_ATTN_TRACE  // timing experiment: event timeline of one CTA
__device__ long long g_tr[8][64];
#define TR(ev, n, cond)                                                               \
  do {                                                                                \
    if ((cond) && blockIdx.x == 100 && blockIdx.y == 5 && (n) < 64) g_tr[ev][n] = clock64(); \
  } while (0)
#else
#define TR(ev, n, cond) \
  do {                  \
  } while (0)
#endif
#ifdef BLADE_ATTN_TIMING  // timing experiment: per-role cycle accounting
__device__ unsigned long long g_tm[10];
#define TM_ADD(i, v) atomicAdd(&g_tm[i], (unsigned long long)(v))
#endif

template <int D, bool kDefaultScale, bool kGT>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmKg,
                   const __grid_constant__ CUtensorMap tmVg, const GtArgs gt, int N, int Nb,
                   float scale_log2_rt, const int32_t* __restrict__ kv_idx,
                   const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ O,
                   float* __restrict__ LSE, volatile int* dbg, int pdl,
                   const int32_t* __restrict__ order) {
  using C = Cfg<D>;
  const float scale_log2 = kDefaultScale ? DefaultScale<D>::kScaleLog2 : scale_log2_rt;
#ifdef BLADE_TC_DEBUG
  const bool dbg_on = dbg != nullptr && blockIdx.x == 0 && blockIdx.y == 0;
#endif
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem;
  char* sRingK = smem + C::kOffRingK;
  char* sRingV = smem + C::kOffRingV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_kempty = bar_kfull + C::kRingK;
  uint64_t* bar_vfull = bar_kempty + C::kRingK;
  uint64_t* bar_vempty = bar_vfull + C::kRingVx;
  uint64_t* bar_s = bar_vempty + C::kRingVx;    // [2] S buffer computed
  uint64_t* bar_p = bar_s + 2;                  // [2] P written (4 warp arrivals)
  uint64_t* bar_pv = bar_p + 2;                 // one completion per P V MMA
  uint64_t* bar_qt = bar_pv + 1;                // Q copied into TMEM (4 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef BLADE_ATTN_TIMING
  const long long t_cta0 = clock64();
#endif
  // LPT order (blade_asa_fwd, tau mode): CTA b takes the b-th longest row
  const int64_t row_id = order ? int64_t(__ldg(order + blockIdx.y * int64_t(gridDim.x) + blockIdx.x))
                               : blockIdx.y * int64_t(Nb) + blockIdx.x;
  const int i = int(row_id % Nb);
  const int64_t u = row_id / Nb;
  int cnt_fine = kv_cnt[row_id];
  // a CTA that waited reads its list through L2 (ld.global.cg): see attn_tc2.cu
  const bool waited = pdl && cnt_fine < 0;
  auto ld_list = [waited](const int32_t* p) { return waited ? __ldcg(p) : __ldg(p); };
  if (waited) {  // refined row (blade_asa_fwd): wait for K-mask.4's final list
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    cnt_fine = __ldcg(kv_cnt + row_id);
  }
  // items: the kept blocks, then (ASA_GT) the global-token tiles
  const int cnt = cnt_fine + (kGT ? (gt.Ng + 127) / 128 : 0);
  const int32_t* list = kv_idx + row_id * Nb;

  if (warp == kLoadKWarp && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRingK; ++s) {
      tc::mbar_init(bar_kfull + s, 1);
      tc::mbar_init(bar_kempty + s, 1);
    }
    for (int s = 0; s < C::kRingVx; ++s) {
      tc::mbar_init(bar_vfull + s, 1);
      tc::mbar_init(bar_vempty + s, 1);
    }
    tc::mbar_init(bar_s + 0, 1);
    tc::mbar_init(bar_s + 1, 1);
    tc::mbar_init(bar_p + 0, kSoftWarps);
    tc::mbar_init(bar_p + 1, kSoftWarps);
    tc::mbar_init(bar_pv, 1);
    tc::mbar_init(bar_qt, 4);
    tc::fence_barrier_init();
  }
  if (warp == kMmaWarp) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kLoadKWarp || warp == kLoadVWarp) {
    // ===================== TMA producers (warp 5: Q and K, warp 6: V) ========
    if (lane == 0) {
      const bool isK = warp == kLoadKWarp;
      if (isK) {
        tc::tma_prefetch_desc(&tmQ);
        tc::tma_prefetch_desc(&tmK);
        if (kGT) tc::tma_prefetch_desc(&tmKg);
        tc::mbar_arrive_expect_tx(bar_q, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(sQ + p * C::kPanel, &tmQ, bar_q, p * 64, i * 128, int(u));
      } else {
        tc::tma_prefetch_desc(&tmV);
        if (kGT) tc::tma_prefetch_desc(&tmVg);
      }
      const int R = isK ? C::kRingK : C::kRingVx;
      char* ring = isK ? sRingK : sRingV;
      uint64_t* full = isK ? bar_kfull : bar_vfull;
      uint64_t* empty = isK ? bar_kempty : bar_vempty;
      const CUtensorMap* m = isK ? &tmK : &tmV;
#ifndef BLADE_ATTN_L2_PREFETCH
#define BLADE_ATTN_L2_PREFETCH 0
#endif
      // warm L2 for the first blocks, then keep BLADE_ATTN_L2_PREFETCH blocks
      // ahead of the ring: a block's first touch comes from HBM
      for (int n = 0; n < BLADE_ATTN_L2_PREFETCH && n < cnt_fine; ++n)
        for (int p = 0; p < C::kPanels; ++p) tc::tma_prefetch_3d(m, p * 64, list[n] * 128, int(u));
      int jn = cnt_fine > 0 ? ld_list(list) : 0;  // block id, loaded one item ahead
      for (int n = 0; n < cnt; ++n) {
        const int jb = jn;
        if (n + 1 < cnt_fine) jn = ld_list(list + n + 1);
        const int s = n % R;
        TC_DBG(0, n);
        if (BLADE_ATTN_L2_PREFETCH > 0 && n + BLADE_ATTN_L2_PREFETCH < cnt_fine)
          for (int p = 0; p < C::kPanels; ++p)
            tc::tma_prefetch_3d(m, p * 64, list[n + BLADE_ATTN_L2_PREFETCH] * 128, int(u));
#ifdef BLADE_ATTN_TIMING
        const long long te0 = clock64();
#endif
        tc::mbar_wait(empty + s, ((n / R) & 1) ^ 1);
#ifdef BLADE_ATTN_TIMING
        if (n >= R) TM_ADD(isK ? 8 : 9, clock64() - te0);
#endif
        TR(isK ? 0 : 1, n, true);
#ifdef BLADE_ATTN_SKIP_KV_LOAD  // timing experiment only: MMA on stale smem
        tc::mbar_arrive(full + s);
#else
        char* dst = ring + s * C::kTile;
        if (!isK && s == C::kRingV) {  // the Q tile's slot: only after Q is in TMEM
          if (n == C::kRingV) tc::mbar_wait(bar_qt, 0);
          dst = sQ;
        }
        tc::mbar_arrive_expect_tx(full + s, C::kTile);
        const bool fine = !kGT || n < cnt_fine;
        const CUtensorMap* mm = fine ? m : (isK ? &tmKg : &tmVg);
        const int row0 = fine ? jb * 128 : (n - cnt_fine) * 128;
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(dst + p * C::kPanel, mm, full + s, p * 64, row0, int(u));
#endif
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer =====================
    if (BLADE_ISSUER(lane)) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, D, 0, 1);
      const uint32_t kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
      auto take = [&](uint64_t* full, int R, int n) -> uint32_t {  // slot of item n, waited for
        const uint32_t s = n % R;
#ifdef BLADE_ATTN_TIMING
        const long long tf0 = clock64();
#endif
        tc::mbar_wait(full + s, (n / R) & 1);
#ifdef BLADE_ATTN_TIMING
        TM_ADD(n < 2 ? 7 : 4, clock64() - tf0);
#endif
        tc::fence_after_sync();
        return s;
      };
      auto issue_S = [&](int n) {  // S(n) into buffer n & 1
        const int buf = n & 1;
        const uint32_t s = take(bar_kfull, C::kRingK, n);
        TR(2, n, true);
        const uint32_t kb = kbase + s * C::kTile;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          // A = Q from TMEM (16 d-values = 8 columns per k-step): the tensor core
          // then reads only K from shared memory, which keeps the S MMA off the
          // smem-bandwidth limit
          BLADE_MMA_TS(tmem + buf * 128, tmem + C::kColQ + ks * 8, tc::sw128_desc(kb + off, 16, 1024),
                     idS, ks > 0);
        }
        BLADE_COMMIT(bar_s + buf);
        BLADE_COMMIT(bar_kempty + s);
      };
      TC_DBG(1, 1);
      tc::mbar_wait(bar_qt, 0);
      tc::fence_after_sync();
      issue_S(0);
      if (cnt > 1) issue_S(1);
      for (int n = 0; n < cnt; ++n) {
        const int buf = n & 1;
        const uint32_t s = take(bar_vfull, C::kRingVx, n);
        TR(3, n, true);
        TC_DBG(1, 100 + n);
#ifdef BLADE_ATTN_TIMING
        const long long tp0 = clock64();
#endif
        tc::mbar_wait(bar_p + buf, (n >> 1) & 1);
#ifdef BLADE_ATTN_TIMING
        TM_ADD(3, clock64() - tp0);
#endif
        tc::fence_after_sync();
        TR(4, n, true);
        const uint32_t vb = s < uint32_t(C::kRingV) ? vbase + s * C::kTile : smem_u32(sQ);
#ifndef BLADE_ATTN_SKIP_PV  // timing experiment only
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          BLADE_MMA_TS(tmem + C::kColO, tmem + buf * 128 + 64 + ks * 8,
                     tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO,
                     (n > 0 || ks > 0) ? 1 : 0);
#endif
        BLADE_COMMIT(bar_pv);
        BLADE_COMMIT(bar_vempty + s);
        if (n + 2 < cnt) issue_S(n + 2);
      }
      // drain: the last commits must land before the CTA's smem is released
      tc::mbar_wait(bar_pv, (cnt - 1) & 1);
      TC_DBG(1, 5001);
    }
  } else if (warp < kSoftWarps) {
    // ===================== softmax =====================
    // warp = (half h, lane quarter qw): rows 32 qw + lane, S columns
    // [h CW, (h+1) CW) of each tile, O columns [h D/kSplit, (h+1) D/kSplit)
    constexpr int CW = 128 / kSplit;    // S columns per thread
    constexpr int DW = D / kSplit;      // O columns per thread
    const int qw = warp & 3, h = warp >> 2;
    const uint32_t lane_base = uint32_t(qw * 32) << 16;
    const uint32_t tO = tmem + lane_base + C::kColO + h * DW;
    const int r = qw * 32 + lane;  // row within the query block
    uint16_t* xch = reinterpret_cast<uint16_t*>(smem + C::kOffXch);  // [2][2][128]
    if (h == 0) {  // Q row (this thread's) from the swizzled smem tile into TMEM columns
      tc::mbar_wait(bar_q, 0);
#pragma unroll
      for (int p = 0; p < C::kPanels; ++p) {
        uint32_t q32[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = *reinterpret_cast<const uint4*>(sQ + p * C::kPanel + r * 128 +
                                                          ((c ^ (r & 7)) << 4));
          q32[4 * c + 0] = v.x;
          q32[4 * c + 1] = v.y;
          q32[4 * c + 2] = v.z;
          q32[4 * c + 3] = v.w;
        }
        tc::st_32x32b_x32(tmem + lane_base + C::kColQ + p * 32, q32);
      }
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_qt);
    }
    float m_used = -INFINITY, l_sum = 0.f;
    int jn = cnt_fine > 0 ? ld_list(list) : 0;  // block id, loaded one tile ahead
    for (int n = 0; n < cnt; ++n) {
      const int buf = n & 1;
      const int jb = jn;
      if (n + 1 < cnt_fine) jn = ld_list(list + n + 1);
      const uint32_t tS = tmem + lane_base + buf * 128;
      if (lane == 0) TC_DBG(2 + (warp & 3), 10 * n + 1);
#ifdef BLADE_ATTN_TIMING
      const long long tw0 = clock64();
#endif
      tc::mbar_wait(bar_s + buf, (n >> 1) & 1);
      tc::fence_after_sync();
      TR(5, n, warp == 0 && lane == 0);
#ifdef BLADE_ATTN_TIMING
      const long long tw1 = clock64();
#endif
#ifdef BLADE_ATTN_SKIP_SOFTMAX  // timing experiment only: MMA/TMA pipeline alone
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p + buf);
      continue;
#endif
      float s[CW];
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tS + h * CW + c * 32, rr);
        tc::wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(rr[e]);
      }
      const bool fine = !kGT || n < cnt_fine;
      // keys of the (possibly partial) last block / global-token tile
      const int valid = (fine ? N - jb * 128 : gt.Ng - (n - cnt_fine) * 128) - h * CW;
      if (valid < CW) {
#pragma unroll
        for (int c = 0; c < CW; ++c)
          if (c >= valid) s[c] = -INFINITY;
      }
      if (kGT && !fine) {  // + ln(n_w) on the pooled region, raw-score units
        const int last = gt.Ng - 1 - (n - cnt_fine) * 128 - h * CW;  // column of the last window
#pragma unroll
        for (int c = 0; c < CW; ++c) s[c] += c == last ? gt.bias_last : gt.bias_full;
      }
      // row max as a tree (a linear chain would serialise the ALU latencies)
      float mx;
      {
        float t8[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float a = fmaxf(s[g], s[g + 8]);
#pragma unroll
          for (int c = g + 16; c < CW; c += 16) a = fmaxf(a, fmaxf(s[c], s[c + 8]));
          t8[g] = a;
        }
        mx = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                   fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7])));
      }
      if (kSplit == 2) {
        // both halves must use the same offset: exchange the half-row maxima
        // as bf16 rounded towards +inf, and both take the max of the two
        // rounded values (any offset >= the row max is exact for softmax).
        // The barrier also orders this half's S loads before the partner's P
        // stores into the upper S columns.
        const uint16_t mine = __bfloat16_as_ushort(__float2bfloat16_ru(mx));
        xch[(buf * 2 + h) * 128 + r] = mine;
        tc::fence_before_sync();  // order the tcgen05.ld above before the partner's st
        asm volatile("bar.sync %0, 64;" ::"r"(1 + qw) : "memory");
        tc::fence_after_sync();
        const uint16_t other = xch[(buf * 2 + (h ^ 1)) * 128 + r];
        mx = fmaxf(__bfloat162float(__ushort_as_bfloat16(mine)),
                   __bfloat162float(__ushort_as_bfloat16(other)));
      }
      const float mxs = mx * scale_log2;
      // warp-uniform (tcgen05.ld/st are .sync.aligned); always true for n = 0;
      // identical in both halves (same rows, same values)
      if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold)) {
        const float m_new = fmaxf(m_used, mxs);
        if (n > 0) {
          const float f = ex2(m_used - m_new);
          l_sum *= f;
          tc::mbar_wait(bar_pv, (n - 1) & 1);  // P V (n-1) has finished writing O
          tc::fence_after_sync();
#pragma unroll
          for (int c = 0; c < DW / 32; ++c) {
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
                        make_float2(0.f, 0.f)};  // independent partial sums (ILP)
      const float2 sl2 = make_float2(scale_log2, scale_log2);
      const float2 nm = make_float2(-m_used, -m_used);
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = fma2(make_float2(s[c * 32 + 2 * e], s[c * 32 + 2 * e + 1]), sl2, nm);
          float2 pp;
          if ((kEmuMask >> (e & 7)) & 1) {
            pp = ex2_poly2(x);
          } else {
            pp.x = ex2(x.x);
            pp.y = ex2(x.y);
          }
          acc4[e & 3] = add2(acc4[e & 3], pp);
          pk[e] = pack_bf16(pp.x, pp.y);
        }
        // P (bf16 pairs) of S columns [32 c', 32 c' + 32) -> TMEM columns 64 + 16 c'
        tc::st_32x32b_x16(tS + 64 + (h * (CW / 32) + c) * 16, pk);
      }
      const float2 acc = add2(add2(acc4[0], acc4[1]), add2(acc4[2], acc4[3]));
      l_sum += acc.x + acc.y;
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p + buf);
      TR(6, n, warp == 0 && lane == 0);
#ifdef BLADE_ATTN_TIMING
      if (lane == 0) {
        const long long tw2 = clock64();
        TM_ADD(0, tw1 - tw0);
        TM_ADD(1, tw2 - tw1);
        TM_ADD(2, 1);
      }
#endif
    }
    // epilogue: O / l -> bf16, LSE
    if (lane == 0) TC_DBG(2 + (warp & 3), 9000);
    if (kSplit == 2) {  // l = l_0 + l_1 (the exchange buffers are free after this barrier)
      float* xl = reinterpret_cast<float*>(smem + C::kOffXch);  // [2][128]
      asm volatile("bar.sync %0, 64;" ::"r"(1 + qw) : "memory");
      xl[h * 128 + r] = l_sum;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + qw) : "memory");
      l_sum = xl[r] + xl[128 + r];
    }
    tc::mbar_wait(bar_pv, (cnt - 1) & 1);
    tc::fence_after_sync();
    const int row = i * 128 + r;
    const float inv = 1.f / l_sum;
    __nv_bfloat16* orow = O + (u * N + row) * int64_t(D) + h * DW;
#pragma unroll
    for (int c = 0; c < DW / 32; ++c) {
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
    if (h == 0 && row < N && LSE)
      LSE[u * N + row] = (m_used + log2f(l_sum)) * 0.69314718055994531f;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
  if (tid == 0) TC_DBG(11, 777);
#ifdef BLADE_ATTN_TIMING
  if (tid == 0) {
    TM_ADD(5, clock64() - t_cta0);
    TM_ADD(6, 1);
  }
#endif
}

template <int D>
cudaError_t launch_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                     const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                     const GtProblem* g, cudaStream_t stream, bool pdl, const int32_t* order) {
  CUtensorMap mq, mk, mv, mkg, mvg;
  if (!make_tile_map(&mq, q, p.BH, p.N, D) || !make_tile_map(&mk, k, p.BH, p.N, D) ||
      !make_tile_map(&mv, v, p.BH, p.N, D))
    return cudaErrorNotSupported;
  GtArgs ga{0, 0.f, 0.f};
  if (g) {
    if (!make_tile_map(&mkg, g->kg, p.BH, g->Ng, D) || !make_tile_map(&mvg, g->vg, p.BH, g->Ng, D))
      return cudaErrorNotSupported;
    const int n_last = p.N - (g->Ng - 1) * g->window;
    ga.Ng = g->Ng;
    ga.bias_full = logf(float(g->window)) / p.scale;
    ga.bias_last = logf(float(n_last)) / p.scale;
  } else {
    mkg = mk;
    mvg = mv;
  }
  constexpr int smem = Cfg<D>::kSmem;
  const bool dflt = p.scale == (D == 128 ? 0.088388346f : 0.125f);
  auto kern = g ? (dflt ? attn_tc_kernel<D, true, true> : attn_tc_kernel<D, false, true>)
                : (dflt ? attn_tc_kernel<D, true, false> : attn_tc_kernel<D, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(p.Nb), unsigned(p.BH));
  int* dbg_dev = nullptr;
#ifdef BLADE_TC_DEBUG
  // CTA (0,0) writes role progress to mapped host memory; the launcher waits
  // up to 5 s and dumps the progress (then exits) if the kernel hangs.
  static int* dbg_host = nullptr;
  if (!dbg_host) cudaHostAlloc(&dbg_host, 64 * sizeof(int), cudaHostAllocMapped);
  memset(dbg_host, 0xff, 64 * sizeof(int));
  cudaHostGetDevicePointer(&dbg_dev, dbg_host, 0);
#endif
  if (pdl) {  // programmatic dependent launch behind the refine kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mkg, mvg, ga, p.N, p.Nb, p.scale * kLog2e,
                           kv_idx, kv_cnt, reinterpret_cast<__nv_bfloat16*>(o), lse,
                           static_cast<volatile int*>(dbg_dev), 1, order);
    if (e != cudaSuccess) return e;
  } else {
    kern<<<grid, kThreads, smem, stream>>>(
        mq, mk, mv, mkg, mvg, ga, p.N, p.Nb, p.scale * kLog2e, kv_idx, kv_cnt,
        reinterpret_cast<__nv_bfloat16*>(o), lse, dbg_dev, 0, order);
  }
  e = cudaGetLastError();
#ifdef BLADE_ATTN_TRACE
  {
    static int calls = 0;
    long long h[8][64];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h, g_tr, sizeof(h));
    if (++calls == 10) {
      const long long t0 = h[0][0];
      fprintf(stderr, "n: Kissue Vissue Ktake Vtake Pready(MMA) SMstart SMdone (cycles from first K issue)\n");
      for (int n = 0; n < 24; ++n)
        fprintf(stderr, "%2d: %7lld %7lld %7lld %7lld %7lld %7lld %7lld\n", n, h[0][n] - t0,
                h[1][n] - t0, h[2][n] - t0, h[3][n] - t0, h[4][n] - t0, h[5][n] - t0, h[6][n] - t0);
    }
  }
#endif
#ifdef BLADE_ATTN_TIMING
  {
    static int calls = 0;
    unsigned long long z[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, h[10];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h, g_tm, sizeof(h));
    cudaMemcpyToSymbol(g_tm, z, sizeof(z));
    if (++calls % 20 == 0 && h[2] && h[6])
      fprintf(stderr,
              "attn timing: softmax wait-S %.0f, compute %.0f cyc/tile/warp; MMA wait-P %.0f, "
              "wait-data %.0f cyc/item (first two items of a CTA: %.0f cyc per CTA); CTA %.0f "
              "cyc, %.1f tiles/CTA; loader wait-empty K %.0f V %.0f cyc/item\n",
              double(h[0]) / h[2], double(h[1]) / h[2], double(h[3]) / (h[2] / 4.0),
              double(h[4]) / (h[2] / 2.0 - 4.0 * h[6]), double(h[7]) / h[6],
              double(h[5]) / h[6], h[2] / 4.0 / h[6], double(h[8]) / (h[2] / 4.0),
              double(h[9]) / (h[2] / 4.0));
  }
#endif
#ifdef BLADE_TC_DEBUG
  if (e == cudaSuccess) {
    for (int it = 0; it < 500 && cudaStreamQuery(stream) == cudaErrorNotReady; ++it) usleep(10000);
    if (cudaStreamQuery(stream) == cudaErrorNotReady) {
      fprintf(stderr, "attn_tc HANG: load=%d mma=%d softmax=[%d %d %d %d] end=%d\n", dbg_host[0],
              dbg_host[1], dbg_host[2], dbg_host[3], dbg_host[4], dbg_host[5], dbg_host[11]);
      fflush(stderr);
      _exit(3);
    }
  }
#endif
  return e;
}

}  // namespace

size_t attn_tc_workspace(const AttnProblem&) { return 256; }

cudaError_t launch_attn_tc(const AttnProblem& p, const void* q, const void* k, const void* v,
                           const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                           char*, size_t, cudaStream_t stream, const GtProblem* gt, bool pdl,
                           const int32_t* order) {
  if (p.d == 64) return launch_d<64>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream, pdl, order);
  if (p.d == 128) return launch_d<128>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream, pdl, order);
  return cudaErrorNotSupported;
}

}  // namespace blade
