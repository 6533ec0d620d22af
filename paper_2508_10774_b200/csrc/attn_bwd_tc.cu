// attn_bwd_tc.cu — the block-sparse attention backward on the 5th-gen tensor
// cores (F3; reading R-23): dQ (forward lists) and
// dK / dV (transposed lists) kernels.
//
// CTA = one query block i (128 rows) of one unit, walking its kept blocks j
// (the forward's list).  Per item, with P = exp(scale S - LSE):
//   S  = Q K_j^T                (SS MMA, TMEM cols [0,128))
//   dP = dO V_j^T               (SS MMA, TMEM cols [128,256))
//   dS = P (dP - D)             (4 warps, thread = row = TMEM lane; dS (bf16)
//                                is written over the low half of dP)
//   dQ += dS K_j                (TS MMA: A = dS in TMEM, B = K_j MN-major;
//                                TMEM cols [256, 256+d))
// Warp roles: 0-3 elementwise, 4 MMA issuer + TMEM allocator, 5 TMA (Q, dO
// once, then K tiles), 6 TMA (V tiles).  MMA order per item n:
//   [S(n) read out] S(n+1) | [dS(n) written] dQ(n) dP(n+1)
// so S(n+1) runs while the warps turn dP(n) into dS(n); dP(n+1) overwrites
// dS(n) only after dQ(n) (one thread's MMAs execute in order).  K_j stays in
// its slot until dQ(n) has read it.
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

template <int D>
struct BCfg {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kPanels = D / 64;
  static constexpr int kPanel = 128 * 128;
  static constexpr int kRingK = D == 128 ? 3 : 4;
  static constexpr int kRingV = D == 128 ? 2 : 4;
  static constexpr int kOffQ = 0, kOffDO = kTile;
  static constexpr int kOffRingK = 2 * kTile;
  static constexpr int kOffRingV = kOffRingK + kRingK * kTile;
  static constexpr int kOffBar = kOffRingV + kRingV * kTile;
  // bar_q, kfull/kempty, vfull/vempty, sc, dp, sf, ds, dq
  static constexpr int kNumBar = 1 + 2 * kRingK + 2 * kRingV + 5;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  static constexpr int kSmem = kOffMisc + 16 + 1024;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256;
};

// EWG elementwise warpgroups split each 128-column tile into 128/EWG-column
// groups (thread = row = TMEM lane, as before).  EWG = 2 for d = 64, where the
// elementwise work (exponentials, dS) outweighs the tensor work per item; P /
// dS then go to TMEM columns of their own (no group overwrites columns another
// group has not read yet): dQ kernel [384, 448), dK/dV kernel [384, 512).
// Warps: 0..4 EWG-1 elementwise, 4 EWG MMA, 4 EWG + 1 / + 2 TMA.
template <int EWG>
constexpr int bwd_threads() { return 32 * (4 * EWG + 3); }
#ifndef BLADE_BWD_EWG64
#define BLADE_BWD_EWG64 2  // A/B on Cog: 3.28 ms (2) vs 3.54 (1) vs 3.38 (4)
#endif
// Which of every 8 exponential pairs of P run on the FMA pipe
// (attn::ex2_poly2, rel. error < 7.5e-5, below the bf16 rounding of P).
#ifndef BLADE_BWD_EMU_MASK
#define BLADE_BWD_EMU_MASK 0x01  // 1 in 8: Cog 3.280 ms vs 3.315 (1 in 4), 3.332 (none), 3.43 (1 in 2)
#endif
BLADE_DEVINL float2 bwd_ex2_pair(float2 x, int pair) {
  if ((BLADE_BWD_EMU_MASK >> (pair & 7)) & 1) return attn::ex2_poly2(x);
  return make_float2(ex2(x.x), ex2(x.y));
}

// ASA_GT (attn_bwd.cu header): the global tokens as extra 128-row items.
struct BwdGtArgs {
  int Ng = 0, ngt = 0;        // global tokens, 128-row tiles of them
  float bfull2 = 0.f, blast2 = 0.f;  // ln(n) log2e, ln(n_last) log2e
  int qps = 0;                // dK/dV of the global tokens: query blocks per split
  float* part = nullptr;      // fp32 partials [2][splits][BH][ngt*128][D]
  int64_t part_stride = 0;    // floats between the dK and dV partials
};

// log2-domain bias of global token w (-inf past N_g: P = 0)
BLADE_DEVINL float gt_bias2(const BwdGtArgs& g, int w) {
  return w < g.Ng - 1 ? g.bfull2 : (w == g.Ng - 1 ? g.blast2 : -INFINITY);
}

template <int D, bool kGT, int EWG>
__global__ void __launch_bounds__(bwd_threads<EWG>(), 1)
    bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmKg,
                     const __grid_constant__ CUtensorMap tmVg, const BwdGtArgs gt,
                     int N, int Nb, float scale, const float* __restrict__ LSE,
                     const float* __restrict__ Dv, const int32_t* __restrict__ kv_idx,
                     const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ dQ) {
  using C = BCfg<D>;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem + C::kOffQ;
  char* sDO = smem + C::kOffDO;
  char* sRingK = smem + C::kOffRingK;
  char* sRingV = smem + C::kOffRingV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_kempty = bar_kfull + C::kRingK;
  uint64_t* bar_vfull = bar_kempty + C::kRingK;
  uint64_t* bar_vempty = bar_vfull + C::kRingV;
  uint64_t* bar_sc = bar_vempty + C::kRingV;  // S(n) computed
  uint64_t* bar_dp = bar_sc + 1;              // dP(n) computed
  uint64_t* bar_sf = bar_dp + 1;              // S(n) read out (4 warps)
  uint64_t* bar_ds = bar_sf + 1;              // dS(n) written (4 warps)
  uint64_t* bar_dq = bar_ds + 1;              // dQ(n) accumulated
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kEW = 4 * EWG, kWMma = kEW, kWTmaK = kEW + 1, kWTmaV = kEW + 2;
  constexpr int CW = 128 / EWG;                               // columns per group
  constexpr uint32_t kColDS = EWG == 1 ? C::kColDP : 384;     // packed bf16 dS
  const int i = blockIdx.x;
  const int64_t u = blockIdx.y;
  const int cnt = kv_cnt[u * Nb + i];
  const int32_t* list = kv_idx + (u * Nb + i) * Nb;
  const int total = cnt + (kGT ? gt.ngt : 0);  // kept blocks, then global-token tiles

  if (warp == kWTmaK && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRingK; ++s) {
      tc::mbar_init(bar_kfull + s, 1);
      tc::mbar_init(bar_kempty + s, 1);
    }
    for (int s = 0; s < C::kRingV; ++s) {
      tc::mbar_init(bar_vfull + s, 1);
      tc::mbar_init(bar_vempty + s, 1);
    }
    tc::mbar_init(bar_sc, 1);
    tc::mbar_init(bar_dp, 1);
    tc::mbar_init(bar_sf, kEW);
    tc::mbar_init(bar_ds, kEW);
    tc::mbar_init(bar_dq, 1);
    tc::fence_barrier_init();
  }
  if (warp == kWMma) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWTmaK || warp == kWTmaV) {
    // ===================== TMA producers =====================
    if (lane == 0) {
      const bool isK = warp == kWTmaK;
      if (isK) {
        tc::tma_prefetch_desc(&tmQ);
        tc::tma_prefetch_desc(&tmDO);
        tc::tma_prefetch_desc(&tmK);
        tc::mbar_arrive_expect_tx(bar_q, 2 * C::kTile);
        for (int p = 0; p < C::kPanels; ++p) {
          tc::tma_load_3d(sQ + p * C::kPanel, &tmQ, bar_q, p * 64, i * 128, int(u));
          tc::tma_load_3d(sDO + p * C::kPanel, &tmDO, bar_q, p * 64, i * 128, int(u));
        }
      } else {
        tc::tma_prefetch_desc(&tmV);
      }
      const int R = isK ? C::kRingK : C::kRingV;
      char* ring = isK ? sRingK : sRingV;
      uint64_t* full = isK ? bar_kfull : bar_vfull;
      uint64_t* empty = isK ? bar_kempty : bar_vempty;
      int jn = cnt > 0 ? __ldg(list) : 0;
      for (int n = 0; n < total; ++n) {
        const int jb = n < cnt ? jn : n - cnt;
        if (n + 1 < cnt) jn = __ldg(list + n + 1);
        const CUtensorMap* m = (kGT && n >= cnt) ? (isK ? &tmKg : &tmVg) : (isK ? &tmK : &tmV);
        const int s = n % R;
        tc::mbar_wait(empty + s, ((n / R) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(full + s, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(ring + s * C::kTile + p * C::kPanel, m, full + s, p * 64, jb * 128,
                          int(u));
      }
    }
  } else if (warp == kWMma) {
    // ===================== MMA issuer =====================
    if (BLADE_ISSUER(lane) && total > 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idQ = tc::idesc_bf16(128, D, 0, 1);
      const uint32_t qa = smem_u32(sQ), da = smem_u32(sDO);
      const uint32_t kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
      tc::mbar_wait(bar_q, 0);
      tc::fence_after_sync();
      auto ss = [&](uint32_t d_col, uint32_t a, uint32_t b) {  // D = A B^T, K = d
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          BLADE_MMA_SS(tmem + d_col, tc::sw128_desc(a + off, 16, 1024),
                     tc::sw128_desc(b + off, 16, 1024), idS, ks > 0);
        }
      };
      auto issue_S = [&](int n) {
        const int s = n % C::kRingK;
        tc::mbar_wait(bar_kfull + s, (n / C::kRingK) & 1);
        tc::fence_after_sync();
        ss(C::kColS, qa, kbase + s * C::kTile);
        BLADE_COMMIT(bar_sc);
      };
      auto issue_dP = [&](int n) {
        const int s = n % C::kRingV;
        tc::mbar_wait(bar_vfull + s, (n / C::kRingV) & 1);
        tc::fence_after_sync();
        ss(C::kColDP, da, vbase + s * C::kTile);
        BLADE_COMMIT(bar_dp);
        BLADE_COMMIT(bar_vempty + s);
      };
      issue_S(0);
      issue_dP(0);
      for (int n = 0; n < total; ++n) {
        if (n + 1 < total) {
          tc::mbar_wait(bar_sf, n & 1);  // S(n) is in registers: its columns are free
          issue_S(n + 1);
        }
        tc::mbar_wait(bar_ds, n & 1);
        tc::fence_after_sync();
        const uint32_t kb = kbase + (n % C::kRingK) * C::kTile;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          BLADE_MMA_TS(tmem + C::kColDQ, tmem + kColDS + ks * 8,
                     tc::sw128_desc(kb + ks * 2048, C::kPanel, 1024), idQ,
                     (n > 0 || ks > 0) ? 1 : 0);
        // only the last dQ MMA is awaited (tcgen05 ops of one thread complete
        // in order): one commit, one phase, every phase has a waiter
        if (n + 1 == total) BLADE_COMMIT(bar_dq);
        BLADE_COMMIT(bar_kempty + (n % C::kRingK));
        if (n + 1 < total) issue_dP(n + 1);
      }
      tc::mbar_wait(bar_dq, 0);
    }
  } else if (warp < kEW) {
    // ===================== elementwise: P, dS =====================
    const int hg = warp / 4, quad = warp & 3;  // column group, TMEM lane quarter
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    const int r = quad * 32 + lane;
    const int c0 = hg * CW;                    // first column of this group
    const int row = i * 128 + r;
    const float sl2 = scale * kLog2e;
    const float lse2 = row < N ? LSE[u * N + row] * kLog2e : INFINITY;  // P = 0 past N
    const float dr = row < N ? Dv[u * N + row] : 0.f;
    int jn = cnt > 0 ? __ldg(list) : 0;
    for (int n = 0; n < total; ++n) {
      const int jb = jn;
      if (n + 1 < cnt) jn = __ldg(list + n + 1);
      tc::mbar_wait(bar_sc, n & 1);
      tc::fence_after_sync();
      float p[CW];
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + C::kColS + c0 + c * 32, rr);
#pragma unroll
        for (int e = 0; e < 32; ++e) p[c * 32 + e] = __uint_as_float(rr[e]);
      }
      tc::wait_ld();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_sf);
      if (!kGT || n < cnt) {
        const int valid = N - jb * 128 - c0;  // keys of a partial last block
#pragma unroll
        for (int c = 0; c < CW; c += 2) {
          const float2 x = bwd_ex2_pair(fma2(make_float2(p[c], p[c + 1]), make_float2(sl2, sl2),
                                             make_float2(-lse2, -lse2)), c / 2);
          p[c] = c < valid ? x.x : 0.f;
          p[c + 1] = c + 1 < valid ? x.y : 0.f;
        }
      } else {  // global tokens w0 + c: + ln n_w
        const int w0 = (n - cnt) * 128 + c0;
#pragma unroll
        for (int c = 0; c < CW; ++c) p[c] = ex2(fmaf(p[c], sl2, gt_bias2(gt, w0 + c) - lse2));
      }
      tc::mbar_wait(bar_dp, n & 1);
      tc::fence_after_sync();
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + C::kColDP + c0 + c * 32, rr);
        tc::wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float d0 = p[c * 32 + 2 * e] * (__uint_as_float(rr[2 * e]) - dr);
          const float d1 = p[c * 32 + 2 * e + 1] * (__uint_as_float(rr[2 * e + 1]) - dr);
          pk[e] = pack_bf16(d0, d1);
        }
        // dS of keys [32c, 32c+32) -> packed columns [16c, 16c+16) of the dP
        // region: columns this thread has already read
        tc::st_32x32b_x16(tmem + lane_base + kColDS + c0 / 2 + c * 16, pk);
      }
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_ds);
    }
    // epilogue: dQ * scale -> bf16
    if (total > 0) {
      tc::mbar_wait(bar_dq, 0);
      tc::fence_after_sync();
    }
    __nv_bfloat16* out = dQ + (u * N + row) * int64_t(D);
    if (total == 0) {  // no kept block (never produced by blade_asa_mask): dQ = 0
      if (row < N && hg == 0)
        for (int c = 0; c < D; c += 8) *reinterpret_cast<uint4*>(out + c) = make_uint4(0, 0, 0, 0);
    } else
#pragma unroll
    for (int c = hg; c < D / 32; c += EWG) {
      uint32_t rr[32];
      tc::ld_32x32b_x32(tmem + lane_base + C::kColDQ + c * 32, rr);
      tc::wait_ld();
      if (row < N) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint4 v;
          const float z = scale;
          v.x = pack_bf16(__uint_as_float(rr[8 * e + 0]) * z, __uint_as_float(rr[8 * e + 1]) * z);
          v.y = pack_bf16(__uint_as_float(rr[8 * e + 2]) * z, __uint_as_float(rr[8 * e + 3]) * z);
          v.z = pack_bf16(__uint_as_float(rr[8 * e + 4]) * z, __uint_as_float(rr[8 * e + 5]) * z);
          v.w = pack_bf16(__uint_as_float(rr[8 * e + 6]) * z, __uint_as_float(rr[8 * e + 7]) * z);
          *reinterpret_cast<uint4*>(out + c * 32 + e * 8) = v;
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kWMma) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------
// dK, dV: CTA = one key block j (128 keys), walking the query blocks i that
// keep it (the transposed lists).  Per item, with P^T = exp(scale S^T - LSE):
//   S^T  = K_j Q_i^T            (SS, TMEM [0,128): rows = keys, cols = queries)
//   dP^T = V_j dO_i^T           (SS, TMEM [128,256))
//   P^T (bf16) over the low half of S^T; dV += P^T dO_i   (TS, TMEM [256, 256+d))
//   dS^T = P^T (dP^T - D) (bf16) over the low half of dP^T;
//   dK += dS^T Q_i                                         (TS, TMEM [256+d, 256+2d))
// MMA order: S(0) dP(0) | [P(n)] dV(n) S(n+1) | [dS(n)] dK(n) dP(n+1)
// Q_i and dO_i share one ring slot, freed after dK(n).  LSE_i and D_i are
// staged in shared memory by the elementwise warps (a column per query).
// ---------------------------------------------------------------------------
template <int D>
struct KCfg {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kPanels = D / 64;
  static constexpr int kPanel = 128 * 128;
  static constexpr int kRing = D == 128 ? 2 : 3;  // slots of (Q_i, dO_i)
  static constexpr int kOffK = 0, kOffV = kTile;
  static constexpr int kOffRing = 2 * kTile;
  static constexpr int kOffBar = kOffRing + kRing * 2 * kTile;
  // bar_kv, full/empty, sc, dp, p, ds, dk
  static constexpr int kNumBar = 1 + 2 * kRing + 5;
  static constexpr int kOffLD = kOffBar + kNumBar * 8 + 16;     // [2][2][128] floats
  static constexpr int kSmem = kOffLD + 2 * 2 * 128 * 4 + 1024;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D;
};

// kGT: the "key block" j is a 128-row tile of global tokens (tmK/tmV map
// K_g/V_g), every query block attends it, blockIdx.z splits the query blocks
// (gt.qps each) and the sums go to fp32 partials gt.part (attn_bwd.cu reduces
// them and spreads dK_g/n_w, dV_g/n_w over the windows).
template <int D, bool kGT, int EWG>
__global__ void __launch_bounds__(bwd_threads<EWG>(), 1)
    bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
                       const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const BwdGtArgs gt, int N, int Nb, float scale, const float* __restrict__ LSE,
                       const float* __restrict__ Dv, const int32_t* __restrict__ q_idx,
                       const int32_t* __restrict__ q_cnt, __nv_bfloat16* __restrict__ dK,
                       __nv_bfloat16* __restrict__ dV) {
  using C = KCfg<D>;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sK = smem + C::kOffK;
  char* sV = smem + C::kOffV;
  char* sRing = smem + C::kOffRing;  // slot s: Q at s * 2 kTile, dO at + kTile
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_kv = bars;
  uint64_t* bar_full = bars + 1;
  uint64_t* bar_empty = bar_full + C::kRing;
  uint64_t* bar_sc = bar_empty + C::kRing;  // S^T(n) and dP^T(n) computed (2 commits)
  uint64_t* bar_dp = bar_sc + 1;
  uint64_t* bar_p = bar_dp + 1;             // P^T(n) written (4 warps)
  uint64_t* bar_ds = bar_p + 1;             // dS^T(n) written (4 warps)
  uint64_t* bar_dk = bar_ds + 1;            // dK(n) accumulated
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffBar + C::kNumBar * 8);
  float* sLD = reinterpret_cast<float*>(smem + C::kOffLD);  // [buf][0: lse2, 1: D][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kEW = 4 * EWG, kWMma = kEW, kWTma = kEW + 1;
  constexpr int CW = 128 / EWG;
  static_assert(EWG == 1 || 256 + 2 * D <= 384, "separate P / dS columns need d = 64");
  constexpr uint32_t kColP = EWG == 1 ? C::kColS : 384;      // packed bf16 P^T
  constexpr uint32_t kColDSt = EWG == 1 ? C::kColDP : 448;   // packed bf16 dS^T
  const int j = blockIdx.x;
  const int64_t u = blockIdx.y;
  const int i_first = kGT ? int(blockIdx.z) * gt.qps : 0;
  const int cnt = kGT ? max(0, min(Nb, i_first + gt.qps) - i_first) : q_cnt[u * Nb + j];
  const int32_t* list = kGT ? nullptr : q_idx + (u * Nb + j) * Nb;
  auto qblock = [&](int n) { return kGT ? i_first + n : __ldg(list + n); };

  if (warp == kWTma && lane == 0) {
    tc::mbar_init(bar_kv, 1);
    for (int s = 0; s < C::kRing; ++s) {
      tc::mbar_init(bar_full + s, 1);
      tc::mbar_init(bar_empty + s, 1);
    }
    tc::mbar_init(bar_sc, 1);
    tc::mbar_init(bar_dp, 1);
    tc::mbar_init(bar_p, kEW);
    tc::mbar_init(bar_ds, kEW);
    tc::mbar_init(bar_dk, 1);
    tc::fence_barrier_init();
  }
  if (warp == kWMma) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWTma) {
    // ===================== TMA producer: K_j, V_j once; (Q_i, dO_i) ring =====
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmQ);
      tc::tma_prefetch_desc(&tmDO);
      tc::mbar_arrive_expect_tx(bar_kv, 2 * C::kTile);
      for (int p = 0; p < C::kPanels; ++p) {
        tc::tma_load_3d(sK + p * C::kPanel, &tmK, bar_kv, p * 64, j * 128, int(u));
        tc::tma_load_3d(sV + p * C::kPanel, &tmV, bar_kv, p * 64, j * 128, int(u));
      }
      int in = cnt > 0 ? qblock(0) : 0;
      for (int n = 0; n < cnt; ++n) {
        const int ib = in;
        if (n + 1 < cnt) in = qblock(n + 1);
        const int s = n % C::kRing;
        tc::mbar_wait(bar_empty + s, ((n / C::kRing) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(bar_full + s, 2 * C::kTile);
        char* dst = sRing + s * 2 * C::kTile;
        for (int p = 0; p < C::kPanels; ++p) {
          tc::tma_load_3d(dst + p * C::kPanel, &tmQ, bar_full + s, p * 64, ib * 128, int(u));
          tc::tma_load_3d(dst + C::kTile + p * C::kPanel, &tmDO, bar_full + s, p * 64, ib * 128,
                          int(u));
        }
      }
    }
  } else if (warp == kWMma) {
    // ===================== MMA issuer =====================
    if (BLADE_ISSUER(lane) && cnt > 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idG = tc::idesc_bf16(128, D, 0, 1);
      const uint32_t ka = smem_u32(sK), va = smem_u32(sV), rb = smem_u32(sRing);
      tc::mbar_wait(bar_kv, 0);
      tc::fence_after_sync();
      auto ss = [&](uint32_t d_col, uint32_t a, uint32_t b) {  // D = A B^T over d
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          BLADE_MMA_SS(tmem + d_col, tc::sw128_desc(a + off, 16, 1024),
                     tc::sw128_desc(b + off, 16, 1024), idS, ks > 0);
        }
      };
      auto ts = [&](uint32_t d_col, uint32_t a_col, uint32_t b, bool acc) {  // D += A(TMEM) B
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          BLADE_MMA_TS(tmem + d_col, tmem + a_col + ks * 8,
                     tc::sw128_desc(b + ks * 2048, C::kPanel, 1024), idG, (acc || ks > 0) ? 1 : 0);
      };
      auto slot_q = [&](int n) { return rb + (n % C::kRing) * 2 * C::kTile; };
      auto wait_full = [&](int n) {
        tc::mbar_wait(bar_full + (n % C::kRing), (n / C::kRing) & 1);
        tc::fence_after_sync();
      };
      wait_full(0);
      ss(C::kColS, ka, slot_q(0));                 // S^T(0)
      BLADE_COMMIT(bar_sc);
      ss(C::kColDP, va, slot_q(0) + C::kTile);     // dP^T(0)
      BLADE_COMMIT(bar_dp);
      for (int n = 0; n < cnt; ++n) {
        tc::mbar_wait(bar_p, n & 1);
        tc::fence_after_sync();
        ts(C::kColDV, kColP, slot_q(n) + C::kTile, n > 0);  // dV += P^T dO_i
        if (n + 1 < cnt) {
          wait_full(n + 1);
          ss(C::kColS, ka, slot_q(n + 1));         // S^T(n+1) (after dV(n) read P^T(n))
          BLADE_COMMIT(bar_sc);
        }
        tc::mbar_wait(bar_ds, n & 1);
        tc::fence_after_sync();
        ts(C::kColDK, kColDSt, slot_q(n), n > 0);  // dK += dS^T Q_i
        if (n + 1 == cnt) BLADE_COMMIT(bar_dk);  // only the last is awaited (see bar_dq)
        BLADE_COMMIT(bar_empty + (n % C::kRing));
        if (n + 1 < cnt) {
          ss(C::kColDP, va, slot_q(n + 1) + C::kTile);  // dP^T(n+1) (after dK(n) read dS^T(n))
          BLADE_COMMIT(bar_dp);
        }
      }
      tc::mbar_wait(bar_dk, 0);
    }
  } else if (warp < kEW) {
    // ===================== elementwise: P^T, dS^T (thread = key row) ========
    const int hg = warp / 4, quad = warp & 3;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    const int r = quad * 32 + lane;
    const int c0 = hg * CW;
    const float sl2 = scale * kLog2e;
    const float brow = kGT ? gt_bias2(gt, j * 128 + r) : 0.f;  // ln n_w of this key row
    int in = cnt > 0 ? qblock(0) : 0;
    for (int n = 0; n < cnt; ++n) {
      const int ib = in;
      if (n + 1 < cnt) in = qblock(n + 1);
      float* L = sLD + (n & 1) * 256;
      if (hg == 0) {  // stage LSE_i (log2 domain) and D_i: query column r
        const int qrow = ib * 128 + r;
        L[r] = qrow < N ? LSE[u * N + qrow] * kLog2e : INFINITY;  // P = 0 past N
        L[128 + r] = qrow < N ? Dv[u * N + qrow] : 0.f;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kEW * 32) : "memory");
      tc::mbar_wait(bar_sc, n & 1);
      tc::fence_after_sync();
      float p[CW];
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + C::kColS + c0 + c * 32, rr);
#pragma unroll
        for (int e = 0; e < 32; ++e) p[c * 32 + e] = __uint_as_float(rr[e]);
      }
      tc::wait_ld();
#pragma unroll
      for (int c = 0; c < CW; c += 2) {
        const float* Lc = L + c0;
        const float2 x = bwd_ex2_pair(
            fma2(make_float2(p[c], p[c + 1]), make_float2(sl2, sl2),
                 kGT ? make_float2(brow - Lc[c], brow - Lc[c + 1]) : make_float2(-Lc[c], -Lc[c + 1])),
            c / 2);
        p[c] = x.x;
        p[c + 1] = x.y;
      }
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {  // P^T (bf16) -> packed columns
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(p[c * 32 + 2 * e], p[c * 32 + 2 * e + 1]);
        tc::st_32x32b_x16(tmem + lane_base + kColP + c0 / 2 + c * 16, pk);
      }
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p);
      tc::mbar_wait(bar_dp, n & 1);
      tc::fence_after_sync();
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + C::kColDP + c0 + c * 32, rr);
        tc::wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int q0 = c * 32 + 2 * e;
          const float d0 = p[q0] * (__uint_as_float(rr[2 * e]) - L[128 + c0 + q0]);
          const float d1 = p[q0 + 1] * (__uint_as_float(rr[2 * e + 1]) - L[128 + c0 + q0 + 1]);
          pk[e] = pack_bf16(d0, d1);
        }
        tc::st_32x32b_x16(tmem + lane_base + kColDSt + c0 / 2 + c * 16, pk);
      }
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_ds);
    }
    // epilogue: dK * scale, dV -> bf16 (key rows; zero if no query keeps j)
    if (cnt > 0) {
      tc::mbar_wait(bar_dk, 0);
      tc::fence_after_sync();
    }
    const int krow = j * 128 + r;
    if constexpr (kGT) {  // fp32 partials (dK_g scaled), every row of the tile
      const int Ngp = gt.ngt * 128;
#pragma unroll
      for (int which = hg; which < 2; which += EWG) {
        float* out = gt.part + which * gt.part_stride +
                     ((int64_t(blockIdx.z) * gridDim.y + u) * Ngp + krow) * int64_t(D);
        const float z = which ? 1.f : scale;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t rr[32];
          if (cnt > 0) {
            tc::ld_32x32b_x32(tmem + lane_base + (which ? C::kColDV : C::kColDK) + c * 32, rr);
            tc::wait_ld();
          }
#pragma unroll
          for (int e = 0; e < 8; ++e)
            *reinterpret_cast<float4*>(out + c * 32 + 4 * e) =
                cnt > 0 ? make_float4(__uint_as_float(rr[4 * e]) * z,
                                      __uint_as_float(rr[4 * e + 1]) * z,
                                      __uint_as_float(rr[4 * e + 2]) * z,
                                      __uint_as_float(rr[4 * e + 3]) * z)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    } else
#pragma unroll
    for (int which = hg; which < 2; which += EWG) {
      __nv_bfloat16* out = (which ? dV : dK) + (u * N + krow) * int64_t(D);
      const float z = which ? 1.f : scale;
      if (cnt == 0) {
        if (krow < N)
          for (int c = 0; c < D; c += 8) *reinterpret_cast<uint4*>(out + c) = make_uint4(0, 0, 0, 0);
        continue;
      }
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + (which ? C::kColDV : C::kColDK) + c * 32, rr);
        tc::wait_ld();
        if (krow < N) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(rr[8 * e + 0]) * z, __uint_as_float(rr[8 * e + 1]) * z);
            v.y = pack_bf16(__uint_as_float(rr[8 * e + 2]) * z, __uint_as_float(rr[8 * e + 3]) * z);
            v.z = pack_bf16(__uint_as_float(rr[8 * e + 4]) * z, __uint_as_float(rr[8 * e + 5]) * z);
            v.w = pack_bf16(__uint_as_float(rr[8 * e + 6]) * z, __uint_as_float(rr[8 * e + 7]) * z);
            *reinterpret_cast<uint4*>(out + c * 32 + e * 8) = v;
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kWMma) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int D>
cudaError_t launch_dkdv_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                          const float* lse, const void* dout, const float* Dv,
                          const int32_t* q_idx, const int32_t* q_cnt, void* dk, void* dv,
                          cudaStream_t stream, const GtProblem* g, float* part, int splits) {
  CUtensorMap mq, mdo, mk, mv;
  const int64_t krows = g ? g->Ng : p.N;
  if (!make_tile_map(&mq, q, p.BH, p.N, D) || !make_tile_map(&mdo, dout, p.BH, p.N, D) ||
      !make_tile_map(&mk, g ? g->kg : k, p.BH, krows, D) ||
      !make_tile_map(&mv, g ? g->vg : v, p.BH, krows, D))
    return cudaErrorNotSupported;
  constexpr int smem = KCfg<D>::kSmem;
  BwdGtArgs ga{};
  if (g) {
    ga.Ng = g->Ng;
    ga.ngt = (g->Ng + 127) / 128;
    ga.bfull2 = logf(float(g->window)) * kLog2e;
    ga.blast2 = logf(float(p.N - (g->Ng - 1) * g->window)) * kLog2e;
    ga.qps = (p.Nb + splits - 1) / splits;
    ga.part = part;
    ga.part_stride = int64_t(splits) * p.BH * ga.ngt * 128 * D;
  }
  constexpr int EWG = D == 64 ? BLADE_BWD_EWG64 : 1;
  auto kern = g ? bwd_dkdv_tc_kernel<D, true, EWG> : bwd_dkdv_tc_kernel<D, false, EWG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(g ? ga.ngt : p.Nb), unsigned(p.BH), unsigned(g ? splits : 1));
  kern<<<grid, bwd_threads<EWG>(), smem, stream>>>(
      mq, mdo, mk, mv, ga, p.N, p.Nb, p.scale, lse, Dv, q_idx, q_cnt,
      reinterpret_cast<__nv_bfloat16*>(dk), reinterpret_cast<__nv_bfloat16*>(dv));
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_dq_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                        const float* lse, const void* dout, const float* Dv,
                        const int32_t* kv_idx, const int32_t* kv_cnt, void* dq,
                        cudaStream_t stream, const GtProblem* g) {
  CUtensorMap mq, mdo, mk, mv, mkg, mvg;
  if (!make_tile_map(&mq, q, p.BH, p.N, D) || !make_tile_map(&mdo, dout, p.BH, p.N, D) ||
      !make_tile_map(&mk, k, p.BH, p.N, D) || !make_tile_map(&mv, v, p.BH, p.N, D))
    return cudaErrorNotSupported;
  BwdGtArgs ga{};
  if (g) {
    if (!make_tile_map(&mkg, g->kg, p.BH, g->Ng, D) || !make_tile_map(&mvg, g->vg, p.BH, g->Ng, D))
      return cudaErrorNotSupported;
    ga.Ng = g->Ng;
    ga.ngt = (g->Ng + 127) / 128;
    ga.bfull2 = logf(float(g->window)) * kLog2e;
    ga.blast2 = logf(float(p.N - (g->Ng - 1) * g->window)) * kLog2e;
  } else {
    mkg = mk;
    mvg = mv;
  }
  constexpr int smem = BCfg<D>::kSmem;
  constexpr int EWG = D == 64 ? BLADE_BWD_EWG64 : 1;
  auto kern = g ? bwd_dq_tc_kernel<D, true, EWG> : bwd_dq_tc_kernel<D, false, EWG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(p.Nb), unsigned(p.BH));
  kern<<<grid, bwd_threads<EWG>(), smem, stream>>>(mq, mdo, mk, mv, mkg, mvg, ga, p.N, p.Nb, p.scale, lse,
                                          Dv, kv_idx, kv_cnt,
                                          reinterpret_cast<__nv_bfloat16*>(dq));
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_bwd_dkdv_tc(const AttnProblem& p, const void* q, const void* k, const void* v,
                               const float* lse, const void* dout, const float* Dv,
                               const int32_t* q_idx, const int32_t* q_cnt, void* dk, void* dv,
                               cudaStream_t stream, const GtProblem* gt, float* part,
                               int splits) {
  if (p.d == 64)
    return launch_dkdv_d<64>(p, q, k, v, lse, dout, Dv, q_idx, q_cnt, dk, dv, stream, gt, part,
                             splits);
  if (p.d == 128)
    return launch_dkdv_d<128>(p, q, k, v, lse, dout, Dv, q_idx, q_cnt, dk, dv, stream, gt, part,
                              splits);
  return cudaErrorNotSupported;
}

cudaError_t launch_bwd_dq_tc(const AttnProblem& p, const void* q, const void* k, const void* v,
                             const float* lse, const void* dout, const float* Dv,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* dq,
                             cudaStream_t stream, const GtProblem* gt) {
  if (p.d == 64)
    return launch_dq_d<64>(p, q, k, v, lse, dout, Dv, kv_idx, kv_cnt, dq, stream, gt);
  if (p.d == 128)
    return launch_dq_d<128>(p, q, k, v, lse, dout, Dv, kv_idx, kv_cnt, dq, stream, gt);
  return cudaErrorNotSupported;
}

}  // namespace blade
