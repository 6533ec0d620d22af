// attn_tc2s.cu — block-sparse attention forward for head dim 64 (PAPER.md
// P:133, ASA_GT global tokens P:135): two query blocks per CTA as in
// attn_tc2.cu, with each block's softmax split over two column halves.
//
// Why: at d = 64 a 128 x 128 tile is 2.5x more exponential work than tensor
// work (MUFU: 16 ex2 / clk / SM), and with one softmax warp per SMSP and
// block the exponential phases of the two blocks barely overlap (trace:
// ~1800 cycles per tile against a 1024-cycle MUFU floor).  Here eight warps
// serve a block: warps (t, h, q) own rows 32 q .. 32 q + 31 and key columns
// [64 h, 64 h + 64) of every tile.  Each column half keeps its own running
// max and sum and accumulates into its OWN O (O_{t,h}, 64 TMEM columns):
// the P V of keys [0, 64) goes to O_{t,0}, that of keys [64, 128) to O_{t,1}
// (the same eight K = 16 MMAs as before, four per half), so the halves never
// exchange a max.  The epilogue merges them once per row:
//   m = max(m_0, m_1), l = sum_h l_h 2^(m_h - m), O = sum_h O_h 2^(m_h - m) / l.
// Four softmax warps per SMSP keep the MUFU fed while the others load,
// reduce and store.
//
// Warp roles (640 threads):
//   warps 0-15  softmax: t = warp / 8 (block), h = (warp / 4) % 2 (half)
//   warp  16    tcgen05.mma issuer + TMEM allocator
//   warp  17    TMA producer: Q_A, Q_B, then K tiles in consumption order
//   warp  18    TMA producer: V tiles in consumption order
//   warp  19    idle
// TMEM (512 columns): S_A [0,128) S_B [128,256), O_{t,h} at 256 + 128 t + 64 h.
// P_{t,h} (bf16, 64 keys) overwrites the lower 32 columns of its own S half
// (chunk by chunk, after that chunk's scores are in registers).
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

constexpr int kD = 64;
constexpr int kTileS = 128 * kD * 2;  // one Q / K / V tile (16 KB)
constexpr int kPanelS = 128 * 128;
constexpr int kRingKS = 6, kRingVS = 5;  // 227 KB: Q 32 + K 96 + V 80 + 2 KB (m, l) exchange
constexpr int kOffQS = 0;
constexpr int kOffRingKS = 2 * kTileS;
constexpr int kOffRingVS = kOffRingKS + kRingKS * kTileS;
constexpr int kOffBarS = kOffRingVS + kRingVS * kTileS;
constexpr int kNumBarS = 1 + 2 * kRingKS + 2 * kRingVS + 3 * 2;  // q, k, v rings, s / p / pv
constexpr int kOffMiscS = kOffBarS + kNumBarS * 8;                // tmem slot (16 B)
constexpr int kOffMLS = kOffMiscS + 16;                           // [2 blocks][128] (m_1, l_1)
constexpr int kSmemS = kOffMLS + 2 * 128 * 8 + 1024;
static_assert(kSmemS <= 227 * 1024, "dynamic shared memory per CTA");
constexpr int kThreadsS = 640;
constexpr float kRescaleThresholdS = 8.0f;  // log2 units
#ifndef BLADE_ATTN2S_EMU_MASK
#define BLADE_ATTN2S_EMU_MASK 0x01  // which of every 8 exponential pairs run on the FMA pipe
#endif
constexpr uint32_t kEmuMaskS = BLADE_ATTN2S_EMU_MASK;

template <bool kDefaultScale, bool kGT>
__global__ void __launch_bounds__(kThreadsS, 1)
    attn_tc2s_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmKg,
                     const __grid_constant__ CUtensorMap tmVg, const GtArgs gt, int N, int Nb,
                     float scale_log2_rt, const int32_t* __restrict__ kv_idx,
                     const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ O,
                     float* __restrict__ LSE, int pdl, const int32_t* __restrict__ order) {
  const float scale_log2 = kDefaultScale ? DefaultScale<kD>::kScaleLog2 : scale_log2_rt;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem + kOffQS;
  char* sRingK = smem + kOffRingKS;
  char* sRingV = smem + kOffRingVS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBarS);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_kempty = bar_kfull + kRingKS;
  uint64_t* bar_vfull = bar_kempty + kRingKS;
  uint64_t* bar_vempty = bar_vfull + kRingVS;
  uint64_t* bar_s = bar_vempty + kRingVS;  // [2] S of block t computed
  uint64_t* bar_p = bar_s + 2;             // [2] P of block t written (8 warp arrivals)
  uint64_t* bar_pv = bar_p + 2;            // [2] last P V of block t done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffMiscS);
  float2* sML = reinterpret_cast<float2*>(smem + kOffMLS);  // [t][row] (m_1, l_1)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t item = order ? int64_t(__ldg(order + blockIdx.y * int64_t(gridDim.x) + blockIdx.x))
                             : blockIdx.y * int64_t(gridDim.x) + blockIdx.x;
  const int64_t u = item / gridDim.x;
  const int i0 = 2 * int(item % gridDim.x);  // block A; block B = i0 + 1 (if < Nb)
  const int nblk = (i0 + 1 < Nb) ? 2 : 1;
  const int ngt = kGT ? (gt.Ng + 127) / 128 : 0;
  int cf0 = kv_cnt[u * Nb + i0];
  int cf1 = nblk == 2 ? kv_cnt[u * Nb + i0 + 1] : 0;
  // a CTA that waited reads its lists through L2 (ld.global.cg): K-mask.4
  // rewrote them while this grid ran (see attn_tc2.cu)
  const bool waited = pdl && (cf0 < 0 || cf1 < 0);
  auto ld_list = [waited](const int32_t* p) { return waited ? __ldcg(p) : __ldg(p); };
  if (waited) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    cf0 = __ldcg(kv_cnt + u * Nb + i0);
    cf1 = nblk == 2 ? __ldcg(kv_cnt + u * Nb + i0 + 1) : 0;
  }
  const int cnt0 = cf0 + ngt, cnt1 = nblk == 2 ? cf1 + ngt : 0;
  const int32_t* list0 = kv_idx + (u * Nb + i0) * Nb;
  const int32_t* list1 = list0 + Nb;

  if (warp == 17 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < kRingKS; ++s) {
      tc::mbar_init(bar_kfull + s, 1);
      tc::mbar_init(bar_kempty + s, 1);
    }
    for (int s = 0; s < kRingVS; ++s) {
      tc::mbar_init(bar_vfull + s, 1);
      tc::mbar_init(bar_vempty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(bar_s + t, 1);
      tc::mbar_init(bar_p + t, 8);
      tc::mbar_init(bar_pv + t, 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 16) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  // registers: 16 softmax warps x 104 + 4 x 40 <= the 640 x 96 allocated at launch
  if (warp >= 16) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 17 || warp == 18) {
      // ===================== TMA producers (17: Q and K, 18: V) =====
      if (lane == 0) {
        const bool isK = warp == 17;
        if (isK) {
          tc::tma_prefetch_desc(&tmQ);
          tc::tma_prefetch_desc(&tmK);
          if (kGT) tc::tma_prefetch_desc(&tmKg);
          tc::mbar_arrive_expect_tx(bar_q, nblk * kTileS);
          for (int t = 0; t < nblk; ++t)
            tc::tma_load_3d(sQ + t * kTileS, &tmQ, bar_q, 0, (i0 + t) * 128, int(u));
        } else {
          tc::tma_prefetch_desc(&tmV);
          if (kGT) tc::tma_prefetch_desc(&tmVg);
        }
        const int R = isK ? kRingKS : kRingVS;
        char* ring = isK ? sRingK : sRingV;
        uint64_t* full = isK ? bar_kfull : bar_vfull;
        uint64_t* empty = isK ? bar_kempty : bar_vempty;
        const CUtensorMap* m = isK ? &tmK : &tmV;
        const CUtensorMap* mg = isK ? &tmKg : &tmVg;
        int g = 0;
        int pre0 = cf0 > 0 ? ld_list(list0) : 0, pre1 = cf1 > 0 ? ld_list(list1) : 0;
        const int mx = cnt0 > cnt1 ? cnt0 : cnt1;
        for (int k = 0; k < mx; ++k) {
          for (int t = 0; t < 2; ++t) {  // consumption order A0 B0 A1 B1 ...
            if (k >= (t ? cnt1 : cnt0)) continue;
            const int cf = t ? cf1 : cf0;
            const bool fine = !kGT || k < cf;
            const int jb = t ? pre1 : pre0;
            if (k + 1 < cf) {
              if (t) pre1 = ld_list(list1 + k + 1);
              else pre0 = ld_list(list0 + k + 1);
            }
            const int s = g % R;
            tc::mbar_wait(empty + s, ((g / R) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(full + s, kTileS);
            tc::tma_load_3d(ring + s * kTileS, fine ? m : mg, full + s, 0,
                            fine ? jb * 128 : (k - cf) * 128, int(u));
            ++g;
          }
        }
      }
    } else if (warp == 16) {
      // ===================== MMA issuer =====================
      if (BLADE_ISSUER(lane)) {
        constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idO = tc::idesc_bf16(128, kD, 0, 1);
        const uint32_t qbase = smem_u32(sQ), kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
        int gk = 0, gv = 0;
        tc::mbar_wait(bar_q, 0);
        tc::fence_after_sync();
        auto issue_S = [&](int t) {  // S_t = Q_t K^T of block t's next item
          const int s = gk % kRingKS;
          tc::mbar_wait(bar_kfull + s, (gk / kRingKS) & 1);
          tc::fence_after_sync();
          const uint32_t kb = kbase + s * kTileS, qb = qbase + t * kTileS;
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks)
            BLADE_MMA_SS(tmem + t * 128, tc::sw128_desc(qb + ks * 32, 16, 1024),
                       tc::sw128_desc(kb + ks * 32, 16, 1024), idS, ks > 0);
          BLADE_COMMIT(bar_s + t);
          BLADE_COMMIT(bar_kempty + s);
          ++gk;
        };
        auto issue_PV = [&](int t, int k) {  // O_{t,h} += P_{t,h} V[64 h, 64 h + 64)
          const int s = gv % kRingVS;
          tc::mbar_wait(bar_vfull + s, (gv / kRingVS) & 1);
          tc::mbar_wait(bar_p + t, k & 1);
          tc::fence_after_sync();
          const uint32_t vb = vbase + s * kTileS;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int h = ks >> 2;
            BLADE_MMA_TS(tmem + 256 + t * 128 + h * 64, tmem + t * 128 + h * 64 + (ks & 3) * 8,
                       tc::sw128_desc(vb + ks * 2048, kPanelS, 1024), idO,
                       (k > 0 || (ks & 3) > 0) ? 1 : 0);
          }
          // only the last P V is awaited (the epilogue); S(k+1) is issued
          // after P V(k), and one thread's tcgen05 ops complete in order
          if (k + 1 == (t ? cnt1 : cnt0)) BLADE_COMMIT(bar_pv + t);
          BLADE_COMMIT(bar_vempty + s);
          ++gv;
        };
        if (cnt0 > 0) issue_S(0);
        if (cnt1 > 0) issue_S(1);
        const int m = cnt0 > cnt1 ? cnt0 : cnt1;
        for (int k = 0; k < m; ++k) {
          if (k < cnt0) {
            issue_PV(0, k);
            if (k + 1 < cnt0) issue_S(0);
          }
          if (k < cnt1) {
            issue_PV(1, k);
            if (k + 1 < cnt1) issue_S(1);
          }
        }
        if (cnt0 > 0) tc::mbar_wait(bar_pv + 0, 0);
        if (cnt1 > 0) tc::mbar_wait(bar_pv + 1, 0);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;\n" ::: "memory");
    // ===================== softmax of block t, column half h =====================
    const int t = warp >> 3, h = (warp >> 2) & 1, qw = warp & 3;
    const int cnt = t ? cnt1 : cnt0;
    const int cnt_fine = t ? cf1 : cf0;
    const int32_t* list = t ? list1 : list0;
    const uint32_t lane_base = uint32_t(qw * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128 + h * 64;         // this half of S_t
    const uint32_t tO = tmem + lane_base + 256 + t * 128 + h * 64;   // O_{t,h}
    const int r = qw * 32 + lane;
    float m_used = -INFINITY, l_sum = 0.f;
    int jn = cnt_fine > 0 ? ld_list(list) : 0;
    const float2 sl2 = make_float2(scale_log2, scale_log2);
    for (int n = 0; n < cnt; ++n) {
      const int jb = jn;
      if (n + 1 < cnt_fine) jn = ld_list(list + n + 1);
      tc::mbar_wait(bar_s + t, n & 1);
      tc::fence_after_sync();
      const bool fine = !kGT || n < cnt_fine;
      const int valid = (fine ? N - jb * 128 : gt.Ng - (n - cnt_fine) * 128) - 64 * h;
      const int last = kGT && !fine ? gt.Ng - 1 - (n - cnt_fine) * 128 - 64 * h : -1;
      // 32 scores of chunk c (keys [32 c, 32 c + 32) of this half), masked /
      // biased; read twice (max pass, exponential pass) to keep 32 live floats
      auto load_chunk = [&](int c, float (&x)[32]) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tS + c * 32, rr);
        tc::wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(rr[e]);
        if (valid < 32 * c + 32) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (32 * c + e >= valid) x[e] = -INFINITY;
        }
        if (kGT && !fine) {  // + ln(n_w) on the pooled region, raw-score units
#pragma unroll
          for (int e = 0; e < 32; ++e) x[e] += 32 * c + e == last ? gt.bias_last : gt.bias_full;
        }
      };
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float x[32];
        load_chunk(c, x);
        float t4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float a = fmaxf(x[g], x[g + 4]);
#pragma unroll
          for (int e = g + 8; e < 32; e += 8) a = fmaxf(a, fmaxf(x[e], x[e + 4]));
          t4[g] = a;
        }
        mx = fmaxf(mx, fmaxf(fmaxf(t4[0], t4[1]), fmaxf(t4[2], t4[3])));
      }
      const float mxs = mx * scale_log2;
      // warp-uniform (tcgen05.ld/st are .sync.aligned).  O_{t,h} is current:
      // S_t(n) was issued after P V_t(n-1) and has completed.  A half whose
      // columns were all padding so far keeps m_used = -inf (its P is 0).
      if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThresholdS)) {
        const float m_new = fmaxf(m_used, mxs);
        if (n > 0) {
          const float f = ex2(m_used - m_new);
          l_sum *= f;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
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
      const float mneg = m_used == -INFINITY ? 0.f : -m_used;
      const float2 nm = make_float2(mneg, mneg);
      // P of chunk c goes to columns [16 c, 16 c + 16) of this half: chunk 0's
      // scores are in registers by then, chunk 1's columns are untouched
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float x[32];
        load_chunk(c, x);
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 xx = fma2(make_float2(x[2 * e], x[2 * e + 1]), sl2, nm);
          float2 pp;
          if ((kEmuMaskS >> (e & 7)) & 1) {
            pp = ex2_poly2(xx);
          } else {
            pp.x = ex2(xx.x);
            pp.y = ex2(xx.y);
          }
          acc4[e & 3] = add2(acc4[e & 3], pp);
          pk[e] = pack_bf16(pp.x, pp.y);
        }
        tc::st_32x32b_x16(tS + c * 16, pk);
      }
      const float2 acc = add2(add2(acc4[0], acc4[1]), add2(acc4[2], acc4[3]));
      l_sum += acc.x + acc.y;
      tc::wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar_p + t);
    }
    if (cnt > 0) {
      // epilogue: merge the two halves' (m, l) and O, then O / l -> bf16, LSE
      if (h == 1) sML[t * 128 + r] = make_float2(m_used, l_sum);
      asm volatile("bar.sync %0, 256;\n" ::"r"(2 + t) : "memory");  // the block's 8 warps
      if (h == 0) {
        const float2 o1 = sML[t * 128 + r];
        const float m = fmaxf(m_used, o1.x);
        const float f0 = ex2(m_used - m);
        const float f1 = o1.x == -INFINITY ? 0.f : ex2(o1.x - m);
        const float l = l_sum * f0 + o1.y * f1;
        const float inv = 1.f / l;
        const float g0 = f0 * inv, g1 = f1 * inv;
        tc::mbar_wait(bar_pv + t, 0);
        tc::fence_after_sync();
        const int row = (i0 + t) * 128 + r;
        __nv_bfloat16* orow = O + (u * N + row) * int64_t(kD);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t a[16], b[16];
          tc::ld_32x32b_x16(tO + c * 16, a);
          tc::ld_32x32b_x16(tO + 64 + c * 16, b);
          tc::wait_ld();
          if (row < N) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float v[8];
#pragma unroll
              for (int x = 0; x < 8; ++x)
                v[x] = __uint_as_float(a[8 * e + x]) * g0 + __uint_as_float(b[8 * e + x]) * g1;
              uint4 w;
              w.x = pack_bf16(v[0], v[1]);
              w.y = pack_bf16(v[2], v[3]);
              w.z = pack_bf16(v[4], v[5]);
              w.w = pack_bf16(v[6], v[7]);
              *reinterpret_cast<uint4*>(orow + c * 16 + e * 8) = w;
            }
          }
        }
        if (row < N && LSE) LSE[u * N + row] = (m + log2f(l)) * 0.69314718055994531f;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 16) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

}  // namespace

cudaError_t launch_attn_tc2s(const AttnProblem& p, const void* q, const void* k, const void* v,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                             cudaStream_t stream, const GtProblem* g, bool pdl,
                             const int32_t* order) {
  if (p.d != kD) return cudaErrorNotSupported;
  CUtensorMap mq, mk, mv, mkg, mvg;
  if (!make_tile_map(&mq, q, p.BH, p.N, kD) || !make_tile_map(&mk, k, p.BH, p.N, kD) ||
      !make_tile_map(&mv, v, p.BH, p.N, kD))
    return cudaErrorNotSupported;
  GtArgs ga{0, 0.f, 0.f};
  if (g) {
    if (!make_tile_map(&mkg, g->kg, p.BH, g->Ng, kD) ||
        !make_tile_map(&mvg, g->vg, p.BH, g->Ng, kD))
      return cudaErrorNotSupported;
    ga.Ng = g->Ng;
    ga.bias_full = logf(float(g->window)) / p.scale;
    ga.bias_last = logf(float(p.N - (g->Ng - 1) * g->window)) / p.scale;
  } else {
    mkg = mk;
    mvg = mv;
  }
  const bool dflt = p.scale == 0.125f;
  auto kern = g ? (dflt ? attn_tc2s_kernel<true, true> : attn_tc2s_kernel<false, true>)
                : (dflt ? attn_tc2s_kernel<true, false> : attn_tc2s_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemS);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned((p.Nb + 1) / 2), unsigned(p.BH));
  cfg.blockDim = dim3(kThreadsS);
  cfg.dynamicSmemBytes = kSmemS;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;  // programmatic dependent launch behind the refine kernel
  e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mkg, mvg, ga, p.N, p.Nb, p.scale * kLog2e,
                         kv_idx, kv_cnt, reinterpret_cast<__nv_bfloat16*>(o), lse, pdl ? 1 : 0,
                         order);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace blade
