// attn_tc1s.cu — block-sparse attention forward for head dim 128 (PAPER.md
// P:133, ASA_GT global tokens P:135): one query block per CTA, S double-
// buffered in TMEM, the softmax split over two column halves with one O
// accumulator each.
//
// Why: in the pair kernel (attn_tc2.cu) a block's softmax is one warp per
// SMSP walking a 128-column row (trace: ~1650 cycles per tile, 128 MUFU
// ops at 8 cycles each plus its max / pack / store chain), and S(n+1) of a
// block cannot start before its P(n) is consumed, so each block's period is
// softmax + P V + S + latencies.  Here:
//  * eight softmax warps: warp (h, q) owns rows 32 q .. 32 q + 31 and key
//    columns [64 h, 64 h + 64) of every tile, with its own running max and
//    sum and its own accumulator O_h (P V of keys [64 h, 64 h + 64) goes to
//    O_h: the same eight K = 16 MMAs, four per half).  Two warps per SMSP
//    share the MUFU, each with half the chain; the halves never exchange a
//    max; the epilogue merges m = max(m_0, m_1), l = sum_h l_h 2^(m_h - m),
//    O = sum_h O_h 2^(m_h - m) / l once per row;
//  * S double-buffered: S(n+1) is computed while the softmax works on S(n),
//    and S(n+2) (into buffer n & 1) is issued right after P V(n) (the tensor
//    pipe executes one thread's MMAs in order, so P(n) has been read).
//
// Warp roles (384 threads):
//   warps 0-7   softmax: h = warp / 4 (column half), q = warp % 4 (lanes)
//   warp  8     tcgen05.mma issuer + TMEM allocator
//   warp  9     TMA producer: Q, then K tiles
//   warp  10    TMA producer: V tiles
//   warp  11    idle
// TMEM (512 columns): S_b at 128 b (b = 0, 1), O_h at 256 + 128 h.  P_{b,h}
// (bf16, 64 keys) overwrites columns [64 h, 64 h + 32) of S_b, chunk by chunk
// after that chunk's scores are in registers.
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

constexpr int kD1 = 128;
constexpr int kTile1 = 128 * kD1 * 2;  // one Q / K / V tile (32 KB)
constexpr int kPanel1 = 128 * 128;     // one 128-byte SW128 panel (64 of d)
constexpr int kRingK1 = 3, kRingV1 = 3;
constexpr int kOffQ1 = 0;
constexpr int kOffRingK1 = kTile1;
constexpr int kOffRingV1 = kOffRingK1 + kRingK1 * kTile1;
constexpr int kOffBar1 = kOffRingV1 + kRingV1 * kTile1;
// bar_q, k / v rings, bar_s[2], bar_p[2], bar_pv
constexpr int kNumBar1 = 1 + 2 * kRingK1 + 2 * kRingV1 + 5;
constexpr int kOffMisc1 = kOffBar1 + kNumBar1 * 8;  // tmem slot (16 B)
constexpr int kOffML1 = kOffMisc1 + 16;             // [128] (m_1, l_1)
constexpr int kSmem1 = kOffML1 + 128 * 8 + 1024;
static_assert(kSmem1 <= 227 * 1024, "dynamic shared memory per CTA");
constexpr int kThreads1 = 384;
constexpr float kRescaleThreshold1 = 8.0f;  // log2 units
#ifndef BLADE_ATTN1S_EMU_MASK
#define BLADE_ATTN1S_EMU_MASK 0x00  // which of every 8 exponential pairs run on the FMA pipe
#endif
constexpr uint32_t kEmuMask1 = BLADE_ATTN1S_EMU_MASK;

template <bool kDefaultScale, bool kGT>
__global__ void __launch_bounds__(kThreads1, 1)
    attn_tc1s_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmKg,
                     const __grid_constant__ CUtensorMap tmVg, const GtArgs gt, int N, int Nb,
                     float scale_log2_rt, const int32_t* __restrict__ kv_idx,
                     const int32_t* __restrict__ kv_cnt, __nv_bfloat16* __restrict__ O,
                     float* __restrict__ LSE, int pdl, const int32_t* __restrict__ order) {
  const float scale_log2 = kDefaultScale ? DefaultScale<kD1>::kScaleLog2 : scale_log2_rt;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem + kOffQ1;
  char* sRingK = smem + kOffRingK1;
  char* sRingV = smem + kOffRingV1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar1);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_kempty = bar_kfull + kRingK1;
  uint64_t* bar_vfull = bar_kempty + kRingK1;
  uint64_t* bar_vempty = bar_vfull + kRingV1;
  uint64_t* bar_s = bar_vempty + kRingV1;  // [2] S buffer b computed
  uint64_t* bar_p = bar_s + 2;             // [2] P of buffer b written (8 warp arrivals)
  uint64_t* bar_pv = bar_p + 2;            // every P V done (one phase per tile)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffMisc1);
  float2* sML = reinterpret_cast<float2*>(smem + kOffML1);  // [row] (m_1, l_1)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t item = order ? int64_t(__ldg(order + blockIdx.y * int64_t(gridDim.x) + blockIdx.x))
                             : blockIdx.y * int64_t(gridDim.x) + blockIdx.x;
  const int64_t u = item / gridDim.x;
  const int i0 = int(item % gridDim.x);  // the query block
  const int ngt = kGT ? (gt.Ng + 127) / 128 : 0;
  int cf = kv_cnt[u * Nb + i0];
  // a CTA that waited reads its list through L2 (ld.global.cg): K-mask.4
  // rewrote it while this grid ran (see attn_tc2.cu)
  const bool waited = pdl && cf < 0;
  auto ld_list = [waited](const int32_t* p) { return waited ? __ldcg(p) : __ldg(p); };
  if (waited) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    cf = __ldcg(kv_cnt + u * Nb + i0);
  }
  const int cnt = cf + ngt;
  const int32_t* list = kv_idx + (u * Nb + i0) * Nb;

  if (warp == 9 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < kRingK1; ++s) {
      tc::mbar_init(bar_kfull + s, 1);
      tc::mbar_init(bar_kempty + s, 1);
    }
    for (int s = 0; s < kRingV1; ++s) {
      tc::mbar_init(bar_vfull + s, 1);
      tc::mbar_init(bar_vempty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(bar_s + b, 1);
      tc::mbar_init(bar_p + b, 8);
    }
    tc::mbar_init(bar_pv, 1);
    tc::fence_barrier_init();
  }
  if (warp == 8) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 8) {
    if (warp == 9 || warp == 10) {
      // ===================== TMA producers (9: Q and K, 10: V) =====
      if (lane == 0) {
        const bool isK = warp == 9;
        if (isK) {
          tc::tma_prefetch_desc(&tmQ);
          tc::tma_prefetch_desc(&tmK);
          if (kGT) tc::tma_prefetch_desc(&tmKg);
          tc::mbar_arrive_expect_tx(bar_q, kTile1);
          for (int p = 0; p < 2; ++p)
            tc::tma_load_3d(sQ + p * kPanel1, &tmQ, bar_q, p * 64, i0 * 128, int(u));
        } else {
          tc::tma_prefetch_desc(&tmV);
          if (kGT) tc::tma_prefetch_desc(&tmVg);
        }
        const int R = isK ? kRingK1 : kRingV1;
        char* ring = isK ? sRingK : sRingV;
        uint64_t* full = isK ? bar_kfull : bar_vfull;
        uint64_t* empty = isK ? bar_kempty : bar_vempty;
        const CUtensorMap* m = isK ? &tmK : &tmV;
        const CUtensorMap* mg = isK ? &tmKg : &tmVg;
        int pre = cf > 0 ? ld_list(list) : 0;
        for (int k = 0; k < cnt; ++k) {
          const bool fine = !kGT || k < cf;
          const int jb = pre;
          if (k + 1 < cf) pre = ld_list(list + k + 1);
          const int s = k % R;
          tc::mbar_wait(empty + s, ((k / R) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(full + s, kTile1);
          for (int p = 0; p < 2; ++p)
            tc::tma_load_3d(ring + s * kTile1 + p * kPanel1, fine ? m : mg, full + s, p * 64,
                            fine ? jb * 128 : (k - cf) * 128, int(u));
        }
      }
    } else if (warp == 8) {
      // ===================== MMA issuer =====================
      if (BLADE_ISSUER(lane)) {
        constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idO = tc::idesc_bf16(128, kD1, 0, 1);
        const uint32_t qbase = smem_u32(sQ), kbase = smem_u32(sRingK), vbase = smem_u32(sRingV);
        tc::mbar_wait(bar_q, 0);
        tc::fence_after_sync();
        auto issue_S = [&](int k) {  // S(k) into buffer k & 1
          const int s = k % kRingK1;
          tc::mbar_wait(bar_kfull + s, (k / kRingK1) & 1);
          tc::fence_after_sync();
          const uint32_t kb = kbase + s * kTile1;
#pragma unroll
          for (int ks = 0; ks < kD1 / 16; ++ks) {
            const uint32_t off = (ks >> 2) * kPanel1 + (ks & 3) * 32;
            BLADE_MMA_SS(tmem + (k & 1) * 128, tc::sw128_desc(qbase + off, 16, 1024),
                       tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
          }
          BLADE_COMMIT(bar_s + (k & 1));
          BLADE_COMMIT(bar_kempty + s);
        };
        if (cnt > 0) issue_S(0);
        if (cnt > 1) issue_S(1);
        for (int k = 0; k < cnt; ++k) {
          const int s = k % kRingV1, b = k & 1;
          tc::mbar_wait(bar_vfull + s, (k / kRingV1) & 1);
          tc::mbar_wait(bar_p + b, (k >> 1) & 1);
          tc::fence_after_sync();
          const uint32_t vb = vbase + s * kTile1;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {  // O_h += P_{b,h} V[64 h, 64 h + 64)
            const int h = ks >> 2;
            BLADE_MMA_TS(tmem + 256 + h * 128, tmem + b * 128 + h * 64 + (ks & 3) * 8,
                       tc::sw128_desc(vb + ks * 2048, kPanel1, 1024), idO,
                       (k > 0 || (ks & 3) > 0) ? 1 : 0);
          }
          BLADE_COMMIT(bar_pv);
          BLADE_COMMIT(bar_vempty + s);
          if (k + 2 < cnt) issue_S(k + 2);  // buffer b: after P V(k) has read P(k)
        }
        if (cnt > 0) tc::mbar_wait(bar_pv, (cnt - 1) & 1);
      }
    }
  } else {
    // ===================== softmax, column half h =====================
    const int h = warp >> 2, qw = warp & 3;
    const uint32_t lane_base = uint32_t(qw * 32) << 16;
    const uint32_t tO = tmem + lane_base + 256 + h * 128;  // O_h
    const int r = qw * 32 + lane;
    float m_used = -INFINITY, l_sum = 0.f;
    int jn = cf > 0 ? ld_list(list) : 0;
    const float2 sl2 = make_float2(scale_log2, scale_log2);
    for (int n = 0; n < cnt; ++n) {
      const int jb = jn;
      if (n + 1 < cf) jn = ld_list(list + n + 1);
      const int b = n & 1;
      const uint32_t tS = tmem + lane_base + b * 128 + h * 64;  // this half of S_b
      tc::mbar_wait(bar_s + b, (n >> 1) & 1);
      tc::fence_after_sync();
      const bool fine = !kGT || n < cf;
      const int valid = (fine ? N - jb * 128 : gt.Ng - (n - cf) * 128) - 64 * h;
      const int last = kGT && !fine ? gt.Ng - 1 - (n - cf) * 128 - 64 * h : -1;
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
      // warp-uniform (tcgen05.ld/st are .sync.aligned).  A half whose columns
      // were all padding so far keeps m_used = -inf (its P is 0).
      if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold1)) {
        const float m_new = fmaxf(m_used, mxs);
        if (n > 0) {  // O_h must be current: P V(n-1) done
          tc::mbar_wait(bar_pv, (n - 1) & 1);
          tc::fence_after_sync();
          const float f = ex2(m_used - m_new);
          l_sum *= f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
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
          if ((kEmuMask1 >> (e & 7)) & 1) {
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
      if (lane == 0) tc::mbar_arrive(bar_p + b);
    }
    if (cnt > 0) {
      // epilogue: merge the two halves' (m, l) and O, then O / l -> bf16, LSE
      if (h == 1) sML[r] = make_float2(m_used, l_sum);
      asm volatile("bar.sync 1, 256;\n" ::: "memory");  // the 8 softmax warps
      if (h == 0) {
        const float2 o1 = sML[r];
        const float m = fmaxf(m_used, o1.x);
        const float f0 = ex2(m_used - m);
        const float f1 = o1.x == -INFINITY ? 0.f : ex2(o1.x - m);
        const float l = l_sum * f0 + o1.y * f1;
        const float inv = 1.f / l;
        const float g0 = f0 * inv, g1 = f1 * inv;
        tc::mbar_wait(bar_pv, (cnt - 1) & 1);
        tc::fence_after_sync();
        const int row = i0 * 128 + r;
        __nv_bfloat16* orow = O + (u * N + row) * int64_t(kD1);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t a[16], bb[16];
          tc::ld_32x32b_x16(tO + c * 16, a);
          tc::ld_32x32b_x16(tO + 128 + c * 16, bb);
          tc::wait_ld();
          if (row < N) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float v[8];
#pragma unroll
              for (int x = 0; x < 8; ++x)
                v[x] = __uint_as_float(a[8 * e + x]) * g0 + __uint_as_float(bb[8 * e + x]) * g1;
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
  if (warp == 8) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

}  // namespace

cudaError_t launch_attn_tc1s(const AttnProblem& p, const void* q, const void* k, const void* v,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                             cudaStream_t stream, const GtProblem* g, bool pdl,
                             const int32_t* order) {
  if (p.d != kD1) return cudaErrorNotSupported;
  CUtensorMap mq, mk, mv, mkg, mvg;
  if (!make_tile_map(&mq, q, p.BH, p.N, kD1) || !make_tile_map(&mk, k, p.BH, p.N, kD1) ||
      !make_tile_map(&mv, v, p.BH, p.N, kD1))
    return cudaErrorNotSupported;
  GtArgs ga{0, 0.f, 0.f};
  if (g) {
    if (!make_tile_map(&mkg, g->kg, p.BH, g->Ng, kD1) ||
        !make_tile_map(&mvg, g->vg, p.BH, g->Ng, kD1))
      return cudaErrorNotSupported;
    ga.Ng = g->Ng;
    ga.bias_full = logf(float(g->window)) / p.scale;
    ga.bias_last = logf(float(p.N - (g->Ng - 1) * g->window)) / p.scale;
  } else {
    mkg = mk;
    mvg = mv;
  }
  const bool dflt = p.scale == 0.088388346f;
  auto kern = g ? (dflt ? attn_tc1s_kernel<true, true> : attn_tc1s_kernel<false, true>)
                : (dflt ? attn_tc1s_kernel<true, false> : attn_tc1s_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(p.Nb), unsigned(p.BH));
  cfg.blockDim = dim3(kThreads1);
  cfg.dynamicSmemBytes = kSmem1;
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
