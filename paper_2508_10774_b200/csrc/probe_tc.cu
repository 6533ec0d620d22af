// probe_tc.cu — K-mask.2 on the 5th-gen tensor cores: the sampled attention
// prober of PAPER.md Alg. 1 l.4-5 in the streaming form of Alg. 3
// (GetMaxPooledAttnMap).
//
// CTA = 128 sampled query rows (M = 128) of one unit, streaming every
// 128-key tile of that unit's sampled keys K_s:
//   warps 0..4H-1  row statistics; H warpgroups split each 128-key tile
//              into 128/H-column groups, thread = sampled query row = TMEM lane:
//              running max M and sum l of e^{s - M} over all sampled keys
//              (l.12-15), and the per-(row, key-block) max R (l.15) kept in
//              TMEM beside the S buffers; at the end
//              P_imp[i, j] = max over the k rows of block i of e^{R - M} / l
//              (l.17-19) with a 16/32-lane shuffle max.
//   warp  4H   tcgen05.mma issuer (S = Q_s K_s^T, double-buffered in TMEM)
//   warp  4H+1 TMA producer (Q_s tile once, K_s tiles through a smem ring)
// H = 4 (16 softmax warps, four per SM sub-partition): the per-tile chain
// (TMEM load, block maxima, exponentials, tree sum) is latency-bound, and
// twice the warps of H = 2 hide twice the latency.
// TMEM: S0 [0,128) S1 [128,256) R [256, 256 + N_b)  (N_b <= 256).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"
#include "select.cuh"
#include "tma_host.h"

namespace blade {
namespace {

template <int D>
struct PCfg {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kPanels = D / 64;
  static constexpr int kPanel = 128 * 128;
  static constexpr int kRing = D == 128 ? 4 : 8;
  static constexpr int kOffRing = kTile;
  static constexpr int kOffBar = kOffRing + kRing * kTile;
  static constexpr int kNumBar = 1 + 2 * kRing + 4;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  static constexpr int kSmem = kOffMisc + 16 + 8 * 16 * 4 + 4 * 128 * 4 + 4 * 128 * 8 + 1024;
};

#ifndef BLADE_PROBE_GROUPS
#define BLADE_PROBE_GROUPS 4
#endif
constexpr int kH = BLADE_PROBE_GROUPS;      // column groups (softmax warpgroups)
constexpr int kEW = 4 * kH;                 // softmax warps
constexpr int kWarpMma = kEW, kWarpTma = kEW + 1;
constexpr int kPThreads = 32 * (kEW + 2);
// Selecting in the probe's epilogue runs select.cuh's large unrolled sort once
// per warp per CTA from a cold instruction cache, after the CTA's tensor work;
// the separate select kernel (mask_kernels.cu) keeps it warm across rows.
#ifndef BLADE_PROBE_FUSED_SELECT
#define BLADE_PROBE_FUSED_SELECT 0
#endif

template <int D, int KK>
__global__ void __launch_bounds__(kPThreads, 1)
    probe_tc_kernel(const __grid_constant__ CUtensorMap tmQs, const __grid_constant__ CUtensorMap tmKs,
                    int N, int Nb, int b, float scale_log2, float* __restrict__ pimp,
                    const ProbeSelect sel) {
  using C = PCfg<D>;
  constexpr int G = 128 / KK;  // key blocks per 128-key tile
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem;
  char* sRing = smem + C::kOffRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_full = bars + 1;
  uint64_t* bar_empty = bars + 1 + C::kRing;
  uint64_t* bar_s = bars + 1 + 2 * C::kRing;   // [2] S buffer written
  uint64_t* bar_f = bar_s + 2;                  // [2] S buffer read out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  uint32_t* keep_bits = tmem_slot + 4;  // [8 warps][16]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t u = blockIdx.y;
  const int row0 = blockIdx.x * 128;
  const int NK = Nb * KK;
  const int ntiles = (NK + 127) / 128;
  const int k_last = min(KK, N - (Nb - 1) * b);
  const int first_invalid = (Nb - 1) * KK + k_last;  // sampled columns >= this are padding

  if (warp == kWarpTma && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRing; ++s) {
      tc::mbar_init(bar_full + s, 1);
      tc::mbar_init(bar_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(bar_s + t, 1);
      tc::mbar_init(bar_f + t, kEW);
    }
    tc::fence_barrier_init();
  }
  if (warp == kWarpMma) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpTma) {
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmQs);
      tc::tma_prefetch_desc(&tmKs);
      tc::mbar_arrive_expect_tx(bar_q, C::kTile);
      for (int p = 0; p < C::kPanels; ++p)
        tc::tma_load_3d(sQ + p * C::kPanel, &tmQs, bar_q, p * 64, row0, int(u));
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % C::kRing;
        tc::mbar_wait(bar_empty + s, ((t / C::kRing) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(bar_full + s, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(sRing + s * C::kTile + p * C::kPanel, &tmKs, bar_full + s, p * 64,
                          t * 128, int(u));
      }
    }
  } else if (warp == kWarpMma) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      const uint32_t qa = smem_u32(sQ), rb = smem_u32(sRing);
      tc::mbar_wait(bar_q, 0);
      tc::fence_after_sync();
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % C::kRing, bsel = t & 1;
        tc::mbar_wait(bar_full + s, (t / C::kRing) & 1);
        if (t >= 2) tc::mbar_wait(bar_f + bsel, ((t >> 1) - 1) & 1);
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
    }
  } else if (warp < kEW) {
    // kH warpgroups split each 128-key tile: group h owns columns [CW h, CW (h+1))
    // (key blocks [h*GH, (h+1)*GH) of the tile) with its own running (M, l)
    constexpr int CW = 128 / kH;
    constexpr int GH = G / kH;
    static_assert(GH >= 1, "a column group must hold whole key blocks");
    const int h = warp >> 2, quad = warp & 3;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    // l is kept in fp64 across tiles and each tile's CW terms are summed as a
    // tree: the sequential fp32 sum over N_k terms would dominate the probe's
    // error budget (DESIGN.md §Tie band)
    float m_run = -INFINITY;
    double l_run = 0.0;
    for (int t = 0; t < ntiles; ++t) {
      const int bsel = t & 1;
      tc::mbar_wait(bar_s + bsel, (t >> 1) & 1);
      tc::fence_after_sync();
      float s[CW];
      {
        const uint32_t ta = tmem + lane_base + bsel * 128 + h * CW;
#pragma unroll
        for (int q = 0; q < CW / 32; ++q) {
          uint32_t r0[32];
          tc::ld_32x32b_x32(ta + q * 32, r0);
          tc::wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) s[q * 32 + e] = __uint_as_float(r0[e]);
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_f + bsel);  // S buffer may be overwritten now
      const int col0 = t * 128 + h * CW;
      if (col0 + CW > first_invalid) {
#pragma unroll
        for (int c = 0; c < CW; ++c)
          if (col0 + c >= first_invalid) s[c] = -INFINITY;
      }
      // R: per key-block max of the raw logits (Alg. 3 l.12/l.15); M and R stay
      // unscaled so every exponent is formed as (s - M) * scale once
      uint32_t rv[GH];
      float tmax = -INFINITY;
#pragma unroll
      for (int g = 0; g < GH; ++g) {
        float gm = s[g * KK];
#pragma unroll
        for (int c = 1; c < KK; ++c) gm = fmaxf(gm, s[g * KK + c]);
        tmax = fmaxf(tmax, gm);
        rv[g] = __float_as_uint(gm);
      }
      const uint32_t rcol = tmem + lane_base + 256 + t * G + h * GH;
      if constexpr (GH == 4) {
        tc::st_32x32b_x4(rcol, reinterpret_cast<uint32_t(&)[4]>(rv));
      } else if constexpr (GH == 2) {
        tc::st_32x32b_x2(rcol, reinterpret_cast<uint32_t(&)[2]>(rv));
      } else {
        tc::st_32x32b_x1(rcol, reinterpret_cast<uint32_t(&)[1]>(rv));
      }
      // online row max / sum over this half (l.13-15)
      const float m_new = fmaxf(m_run, tmax);
      if (m_new != -INFINITY) {  // a half tile of padding only leaves (M, l) untouched
        // packed fp32x2 arithmetic: the same roundings as the scalar
        // (s - M) * scale and tree sum, half the FMA-pipe issue slots
        const float2 nm2 = make_float2(-m_new, -m_new), sc2 = make_float2(scale_log2, scale_log2);
#pragma unroll
        for (int c = 0; c < CW; c += 2) {
          const float2 x = mul2(add2(make_float2(s[c], s[c + 1]), nm2), sc2);
          s[c] = ex2(x.x);
          s[c + 1] = ex2(x.y);
        }
#pragma unroll
        for (int w = CW / 2; w >= 2; w >>= 1)
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
    // merge the groups' (M, l) per row (the l.14 recurrence, once)
    float* smm = reinterpret_cast<float*>(keep_bits + 8 * 16);        // [kH][128] m
    double* sml = reinterpret_cast<double*>(smm + 4 * 128);             // [kH][128] l
    const int r = quad * 32 + lane;
    smm[h * 128 + r] = m_run;
    sml[h * 128 + r] = l_run;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kEW * 32) : "memory");
    float M = -INFINITY;
#pragma unroll
    for (int g = 0; g < kH; ++g) M = fmaxf(M, smm[g * 128 + r]);
    double L = 0.0;
#pragma unroll
    for (int g = 0; g < kH; ++g) {
      const float mg = smm[g * 128 + r];
      if (mg != -INFINITY) L += sml[g * 128 + r] * double(ex2((mg - M) * scale_log2));
    }
    // pooling (l.17-19): rows of query block i are KK consecutive lanes; the
    // groups take interleaved 32-column chunks of R
    const int gr = row0 + r;
    const int ib = gr / KK;
    const bool row_ok = gr < NK && (gr % KK) < min(KK, N - ib * b);
    const float inv_l = float(1.0 / L);
    for (int j0 = h * 32; j0 < Nb; j0 += 32 * kH) {
      uint32_t rr[32];
      tc::ld_32x32b_x32(tmem + lane_base + 256 + j0, rr);
      tc::wait_ld();
      float pv[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        float v = row_ok ? ex2((__uint_as_float(rr[e]) - M) * scale_log2) * inv_l : 0.f;
#pragma unroll
        for (int o = 1; o < KK; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        pv[e] = v;
      }
      if ((lane % KK) == 0 && ib < Nb) {
        float* dst = pimp + (u * Nb + ib) * int64_t(Nb) + j0;
        const int nj = min(32, Nb - j0);
        if (nj == 32 && (Nb % 4) == 0) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) = make_float4(pv[e], pv[e + 1], pv[e + 2], pv[e + 3]);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e < nj) dst[e] = pv[e];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  // K-mask.3 fused: the CTA holds complete P_imp rows of its 128 / KK query
  // blocks; one warp selects each (Alg. 1 l.7-10, select.cuh)
  if (BLADE_PROBE_FUSED_SELECT) {
    const int ib = row0 / KK + warp;
    if (warp < 128 / KK && ib < Nb) {
      const int64_t row = u * Nb + ib;
      const bool flag = select_row(pimp + row * Nb, Nb, sel.tau, sel.lo, sel.hi, sel.guard, true,
                                   sel.mask ? sel.mask + row * Nb : nullptr,
                                   sel.kv_idx + row * Nb, sel.kv_cnt + row, keep_bits + warp * 16);
      if (flag && lane == 0) {
        const int slot = atomicAdd(&sel.counters[0], 1);
        sel.flags[slot] = int32_t(row);
        sel.done[slot] = 0;
        if (sel.neg_flagged) sel.kv_cnt[row] = -1 - sel.kv_cnt[row];
      }
    }
  }
  if (warp == kWarpMma) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int D, int KK>
cudaError_t launch_dk(int64_t BH, int N, int Nb, int b, float scale, const void* qs,
                      const void* ks, float* pimp, const ProbeSelect& sel, cudaStream_t stream) {
  CUtensorMap mq, mk;
  const int64_t NK = int64_t(Nb) * KK;
  if (!make_tile_map(&mq, qs, BH, NK, D) || !make_tile_map(&mk, ks, BH, NK, D))
    return cudaErrorNotSupported;
  constexpr int smem = PCfg<D>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(probe_tc_kernel<D, KK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned((NK + 127) / 128), unsigned(BH));
  probe_tc_kernel<D, KK><<<grid, kPThreads, smem, stream>>>(mq, mk, N, Nb, b, scale * kLog2e,
                                                            pimp, sel);
  return cudaGetLastError();
}

}  // namespace

bool probe_tc_selects() { return BLADE_PROBE_FUSED_SELECT != 0; }

bool probe_tc_supported(int d, int kk, int Nb) {
  return (d == 64 || d == 128) && (kk == 16 || kk == 32) && Nb <= 256;
}

cudaError_t launch_probe_tc(int64_t BH, int N, int Nb, int b, int kk, int d, float scale,
                            const void* qs, const void* ks, float* pimp, const ProbeSelect* sel,
                            cudaStream_t stream) {
  if (d == 128 && kk == 16) return launch_dk<128, 16>(BH, N, Nb, b, scale, qs, ks, pimp, *sel, stream);
  if (d == 128 && kk == 32) return launch_dk<128, 32>(BH, N, Nb, b, scale, qs, ks, pimp, *sel, stream);
  if (d == 64 && kk == 16) return launch_dk<64, 16>(BH, N, Nb, b, scale, qs, ks, pimp, *sel, stream);
  if (d == 64 && kk == 32) return launch_dk<64, 32>(BH, N, Nb, b, scale, qs, ks, pimp, *sel, stream);
  return cudaErrorNotSupported;
}

}  // namespace blade
