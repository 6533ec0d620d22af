// attn_tc3.cu — block-sparse attention forward for sm_100a with THREE S
// buffers in TMEM (P:135 global tokens as extra tiles).
//
// CTA = one query block (128 rows) of one unit, walking its kept-block list.
// With two S buffers (attn_tc.cu) S(n+1) can only be issued after P V(n-1)
// has read P(n-1) out of the buffer S(n+1) reuses, so on a Wan layer the
// softmax of tile n+1 waits ~350 cycles for S(n+1) after finishing tile n
// (traced: 1444-cycle softmax, 1790-cycle period).  Three buffers keep S two
// tiles ahead of the softmax:
//   MMA order  S(0) S(1) S(2) | P V(0) S(3) | P V(1) S(4) | ...
// S(n+3) reuses buffer n % 3 after P V(n) has read P(n) (one thread's MMAs
// execute in order).  TMEM: S_b [128 b, 128 b + 128) for b < 3, O [384,
// 384 + d).  Q stays in shared memory (S = Q K^T is an SS MMA); K and V
// stream through separate TMA rings in consumption order.
// Warp roles: 0-3 softmax (thread = query row = TMEM lane), 4 MMA issuer +
// TMEM allocator, 5 TMA (Q, K), 6 TMA (V).
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
#ifdef BLADE_WITH_BASELINES  // comparison baseline, not in the product build
namespace {

using attn::DefaultScale;
using attn::ex2_poly2;
using attn::GtArgs;

template <int D>
struct Cfg3 {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kPanels = D / 64;
  static constexpr int kPanel = 128 * 128;
  static constexpr int kNB = 3;  // S buffers
  static constexpr int kRingK = D == 128 ? 3 : 6;
  static constexpr int kRingV = D == 128 ? 3 : 6;
  static constexpr int kOffQ = 0;
  static constexpr int kOffRingK = kTile;
  static constexpr int kOffRingV = kOffRingK + kRingK * kTile;
  static constexpr int kOffBar = kOffRingV + kRingV * kTile;
  static constexpr int kNumBar = 1 + 2 * kRingK + 2 * kRingV + 3 * kNB;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  static constexpr int kSmem = kOffMisc + 16 + 1024;
  static constexpr uint32_t kColO = 128 * kNB;
};

constexpr int kThreads3 = 224;
constexpr float kRescaleThreshold3 = 8.0f;  // log2 units
#ifndef BLADE_ATTN3_EMU_MASK
#define BLADE_ATTN3_EMU_MASK 0x11  // which of every 8 exponential pairs run on the FMA pipe
#endif
constexpr uint32_t kEmuMask3 = BLADE_ATTN3_EMU_MASK;

template <int D, bool kDefaultScale, bool kGT>
__global__ void __launch_bounds__(kThreads3, 1)
    attn_tc3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV,
                    const __grid_constant__ CUtensorMap tmKg,
                    const __grid_constant__ CUtensorMap tmVg, const GtArgs gt, int N, int Nb,
                    float scale_log2_rt, const int32_t* __restrict__ kv_idx,
                    const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ O,
                    float* __restrict__ LSE) {
  using C = Cfg3<D>;
  constexpr int NB = C::kNB;
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
  uint64_t* bar_s = bar_vempty + C::kRingV;  // [NB] S buffer computed
  uint64_t* bar_p = bar_s + NB;              // [NB] P written (4 warp arrivals)
  // [NB] P V of an item using buffer b done.  Per buffer, so that a wait for
  // P V(n-1) cannot alias with P V(n-3) (three P Vs may be in flight).
  uint64_t* bar_pv = bar_p + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = blockIdx.x;
  const int64_t u = blockIdx.y;
  const int cnt_fine = kv_cnt[u * Nb + i];
  const int cnt = cnt_fine + (kGT ? (gt.Ng + 127) / 128 : 0);
  const int32_t* list = kv_idx + (u * Nb + i) * Nb;

  if (warp == 5 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRingK; ++s) {
      tc::mbar_init(bar_kfull + s, 1);
      tc::mbar_init(bar_kempty + s, 1);
    }
    for (int s = 0; s < C::kRingV; ++s) {
      tc::mbar_init(bar_vfull + s, 1);
      tc::mbar_init(bar_vempty + s, 1);
    }
    for (int b = 0; b < NB; ++b) {
      tc::mbar_init(bar_s + b, 1);
      tc::mbar_init(bar_p + b, 4);
      tc::mbar_init(bar_pv + b, 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 4) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 5 || warp == 6) {
    // ===================== TMA producers =====================
    if (lane == 0) {
      const bool isK = warp == 5;
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
      const int R = isK ? C::kRingK : C::kRingV;
      char* ring = isK ? sRingK : sRingV;
      uint64_t* full = isK ? bar_kfull : bar_vfull;
      uint64_t* empty = isK ? bar_kempty : bar_vempty;
      const CUtensorMap* m = isK ? &tmK : &tmV;
      const CUtensorMap* mg = isK ? &tmKg : &tmVg;
      int jn = cnt_fine > 0 ? __ldg(list) : 0;  // block id, loaded one item ahead
      for (int n = 0; n < cnt; ++n) {
        const int jb = jn;
        if (n + 1 < cnt_fine) jn = __ldg(list + n + 1);
        const int s = n % R;
        tc::mbar_wait(empty + s, ((n / R) & 1) ^ 1);
        const bool fine = !kGT || n < cnt_fine;
        const CUtensorMap* mm = fine ? m : mg;
        const int row0 = fine ? jb * 128 : (n - cnt_fine) * 128;
        tc::mbar_arrive_expect_tx(full + s, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(ring + s * C::kTile + p * C::kPanel, mm, full + s, p * 64, row0, int(u));
      }
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0 && cnt > 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, D, 0, 1);
      const uint32_t qa = smem_u32(sQ), kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
      tc::mbar_wait(bar_q, 0);
      tc::fence_after_sync();
      auto issue_S = [&](int n) {  // S(n) into buffer n % NB
        const int s = n % C::kRingK, b = n % NB;
        tc::mbar_wait(bar_kfull + s, (n / C::kRingK) & 1);
        tc::fence_after_sync();
        const uint32_t kb = kbase + s * C::kTile;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          tc::mma_ss(tmem + b * 128, tc::sw128_desc(qa + off, 16, 1024),
                     tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
        }
        tc::commit(bar_s + b);
        tc::commit(bar_kempty + s);
      };
      for (int n = 0; n < NB && n < cnt; ++n) issue_S(n);
      for (int n = 0; n < cnt; ++n) {
        const int s = n % C::kRingV, b = n % NB;
        tc::mbar_wait(bar_vfull + s, (n / C::kRingV) & 1);
        tc::mbar_wait(bar_p + b, (n / NB) & 1);
        tc::fence_after_sync();
        const uint32_t vb = vbase + s * C::kTile;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc::mma_ts(tmem + C::kColO, tmem + b * 128 + 64 + ks * 8,
                     tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO,
                     (n > 0 || ks > 0) ? 1 : 0);
        tc::commit(bar_pv + b);
        tc::commit(bar_vempty + s);
        if (n + NB < cnt) issue_S(n + NB);
      }
      tc::mbar_wait(bar_pv + (cnt - 1) % NB, ((cnt - 1) / NB) & 1);
    }
  } else if (warp < 4) {
    // ===================== softmax =====================
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    const uint32_t tO = tmem + lane_base + C::kColO;
    const int r = warp * 32 + lane;
    float m_used = -INFINITY, l_sum = 0.f;
    int jn = cnt_fine > 0 ? __ldg(list) : 0;
    for (int n = 0; n < cnt; ++n) {
      const int b = n % NB;
      const int jb = jn;
      if (n + 1 < cnt_fine) jn = __ldg(list + n + 1);
      const uint32_t tS = tmem + lane_base + b * 128;
      tc::mbar_wait(bar_s + b, (n / NB) & 1);
      tc::fence_after_sync();
#ifdef BLADE_ATTN3_SKIP_SOFTMAX  // timing experiment only
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p + b);
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
      // warp-uniform (tcgen05.ld/st are .sync.aligned); always true for n = 0
      if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold3)) {
        const float m_new = fmaxf(m_used, mxs);
        if (n > 0) {
          const float f = ex2(m_used - m_new);
          l_sum *= f;
          // P V(n-1) (and, by commit order, every earlier P V) has written O
          tc::mbar_wait(bar_pv + (n - 1) % NB, ((n - 1) / NB) & 1);
          tc::fence_after_sync();
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
          if ((kEmuMask3 >> (e & 7)) & 1) {
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
      if (lane == 0) tc::mbar_arrive(bar_p + b);
    }
    // epilogue: O / l -> bf16, LSE
    if (cnt > 0) {
      tc::mbar_wait(bar_pv + (cnt - 1) % NB, ((cnt - 1) / NB) & 1);
      tc::fence_after_sync();
    }
    const int row = i * 128 + r;
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
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 4) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int D>
cudaError_t launch3_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                      const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                      const GtProblem* g, cudaStream_t stream) {
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
  constexpr int smem = Cfg3<D>::kSmem;
  const bool dflt = p.scale == (D == 128 ? 0.088388346f : 0.125f);
  auto kern = g ? (dflt ? attn_tc3_kernel<D, true, true> : attn_tc3_kernel<D, false, true>)
                : (dflt ? attn_tc3_kernel<D, true, false> : attn_tc3_kernel<D, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(p.Nb), unsigned(p.BH));
  kern<<<grid, kThreads3, smem, stream>>>(mq, mk, mv, mkg, mvg, ga, p.N, p.Nb, p.scale * kLog2e,
                                          kv_idx, kv_cnt, reinterpret_cast<__nv_bfloat16*>(o),
                                          lse);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_tc3(const AttnProblem& p, const void* q, const void* k, const void* v,
                            const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                            cudaStream_t stream, const GtProblem* gt) {
  if (p.d == 64) return launch3_d<64>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream);
  if (p.d == 128) return launch3_d<128>(p, q, k, v, kv_idx, kv_cnt, o, lse, gt, stream);
  return cudaErrorNotSupported;
}

#else
cudaError_t launch_attn_tc3(const AttnProblem&, const void*, const void*, const void*,
                            const int32_t*, const int32_t*, void*, float*, cudaStream_t,
                            const GtProblem*) {
  return cudaErrorNotSupported;
}
#endif  // BLADE_WITH_BASELINES

}  // namespace blade
