// probe2.cu — K-mask.2, the sampled attention prober of PAPER.md Alg. 1 l.3-5
// in the streaming form of Alg. 3 (GetMaxPooledAttnMap,
// P:633-662), on the 5th-gen tensor cores, reading the sampled rows straight
// from Q and K.
//
// The sampled rows come from the gathered copies Q_s / K_s (K-mask.1) by
// tiled TMA.  Loading them straight from Q and K with the sm_100 TMA
// gather4 mode (four 128-byte rows per instruction, one per sampled slot)
// was built and measured 2.5x slower on the Wan layer (273 vs 109 us: the
// TMA unit sustained ~1.5 TB/s of 128-byte row requests, ~100 cycles per
// gather4 per SM), so the 25 MB gathered copy stays.
//
// CTA = 128 sampled query rows (M = 128) of one unit, streaming every
// 128-key tile of that unit's sampled keys:
//   warps 0..15  row statistics.  Warps 0-7 take the even tiles, 8-15 the odd
//                ones (S is double-buffered in TMEM, one buffer per parity),
//                so the two halves are a tile apart and their exponential
//                phases interleave with the other half's load / max phases
//                on the same SM sub-partition.  Within a half, warp
//                (h, quad) owns columns [64 h, 64 h + 64) of its tiles for
//                rows 32 quad .. 32 quad + 31 (thread = sampled query row =
//                TMEM lane): running max M and sum l of e^{s - M} (l.12-15),
//                the per-(row, key-block) max R (l.15) stored in TMEM.
//                At the end the four partial (M, l) of a row are merged
//                (l.14) and P_imp[i, j] = max over the k rows of block i of
//                e^{R - M} / l (l.17-19) is formed as
//                2^(max_s ((R_sj - M_s) c - log2 l_s)): the max over the
//                block's rows is taken before the (single) exponential.
//   warp 16      tcgen05.mma issuer (S = Q_s K_s^T, M=N=128, K = d)
//   warp 17      TMA producer (the Q_s tile once, K_s tiles through a ring)
// TMEM: S0 [0,128) S1 [128,256) R [256, 256 + R columns).
// Exponentials: ex2.approx on MUFU, and for the pairs selected by
// BLADE_PROBE_EMU (mask over 8 pairs) a degree-5 minimax polynomial on the
// FMA pipe with the same accuracy (|rel err| < 2.4e-7 in fp32).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"
#include "tma_host.h"

namespace blade {
namespace {

template <int D>
struct P2Cfg {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kPanels = D / 64;
  static constexpr int kPanel = 128 * 128;
  static constexpr int kRing = D == 128 ? 4 : 8;
  static constexpr int kOffRing = kTile;
  static constexpr int kOffBar = kOffRing + kRing * kTile;
  static constexpr int kNumBar = 1 + 2 * kRing + 4;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  // misc: tmem slot (16 B), M partials [4][128] f32, l partials [4][128] f64
  static constexpr int kSmem = kOffMisc + 16 + 4 * 128 * 4 + 4 * 128 * 8 + 1024;
};

constexpr int kSW = 16;                 // softmax warps
constexpr int kWarpMma2 = kSW, kWarpTma2 = kSW + 1;
constexpr int kP2Threads = 32 * (kSW + 2);

#ifndef BLADE_PROBE_EMU
// which of every 8 exponential pairs run on the FMA pipe: pair 1 (keep-ratio
// mask, L2 flushed: Wan 0.165 vs 0.169 ms, Cog 0.179 vs 0.187 ms; 0x01 0.167 /
// 0.182, 0x10, 0x11, 0x22 0.167-0.169 / 0.183)
#define BLADE_PROBE_EMU 0x02
#endif
constexpr uint32_t kEmu = BLADE_PROBE_EMU;

// 2^x for a pair on the FMA pipe: x = n + f, n = rint(x) (1.5 * 2^23 trick),
// f in [-1/2, 1/2], 2^f by a degree-5 relative-minimax polynomial, n added to
// the exponent field.  x is clamped at -125 (2^-125 ~ 2.4e-38: a term that
// small cannot move a sum whose largest term is 1).
BLADE_DEVINL float2 ex2_poly5x2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = add2(x, make_float2(12582912.f, 12582912.f));
  const float2 n = add2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = fma2(n, make_float2(-1.f, -1.f), x);
  float2 p = fma2(f, make_float2(1.3276472454890609e-3f, 1.3276472454890609e-3f),
                  make_float2(9.675540961325169e-3f, 9.675540961325169e-3f));
  p = fma2(p, f, make_float2(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = fma2(p, f, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = fma2(p, f, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = fma2(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

BLADE_DEVINL float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;\n" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <int D, int KK>
__global__ void __launch_bounds__(kP2Threads, 1)
    probe2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  int N, int Nb, int b, float scale_log2, float* __restrict__ pimp) {
  using C = P2Cfg<D>;
  constexpr int G = KK <= 64 ? 128 / KK : 1;  // key blocks per 128-key tile
  constexpr int CPB = KK == 128 ? 2 : 1;      // R columns per key block (k = b: one per half)
  constexpr int CPT = G * CPB;                // R columns per tile
  constexpr int CPH = CPT / 2;                // R columns per warp column half
  constexpr int KH = KK <= 64 ? KK : 64;      // keys per R value
  constexpr int TPP = 256 / CPT;              // tiles per R pass (256 TMEM columns)
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem;
  char* sRing = smem + C::kOffRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_full = bars + 1;
  uint64_t* bar_empty = bars + 1 + C::kRing;
  uint64_t* bar_s = bars + 1 + 2 * C::kRing;  // [2] S buffer (= sequence parity) written
  uint64_t* bar_f = bar_s + 2;                 // [2] S buffer read out (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  float* smm = reinterpret_cast<float*>(smem + C::kOffMisc + 16);  // [4][128]
  double* sml = reinterpret_cast<double*>(smm + 4 * 128);           // [4][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t u = blockIdx.y;
  const int row0 = blockIdx.x * 128;
  const int NK = Nb * KK;
  const int ntiles = (NK + 127) / 128;
  const int k_last = min(KK, N - (Nb - 1) * b);
  const int first_invalid = (Nb - 1) * KK + k_last;  // sampled columns >= this are padding
  // The tile sequence: pass 0 streams every tile (row statistics, and R of
  // tiles [0, TPP)); R needs N_b CPB TMEM columns, so when that exceeds 256
  // (N_b > 256, or k = b with N_b > 128) passes p >= 1 stream tiles
  // [p TPP, (p+1) TPP) again for their R only (no exponentials), each pass
  // pooled before the next overwrites the R columns.
  const int npass = (ntiles + TPP - 1) / TPP;
  const int nseq = ntiles + (ntiles > TPP ? ntiles - TPP : 0);
  auto seq_tile = [&](int T) { return T < ntiles ? T : T - ntiles + TPP; };

  if (warp == kWarpTma2 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRing; ++s) {
      tc::mbar_init(bar_full + s, 1);
      tc::mbar_init(bar_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(bar_s + t, 1);
      tc::mbar_init(bar_f + t, kSW / 2);
    }
    tc::fence_barrier_init();
  }
  if (warp == kWarpMma2) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  // K-mask.3 (select_kernel, a programmatic dependent) may be scheduled now;
  // it waits for this grid's completion before reading P_imp
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  if (warp == kWarpTma2) {
    // ===================== producer: tiled TMA loads of Q_s / K_s =====
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmQ);
      tc::tma_prefetch_desc(&tmK);
      // a programmatic dependent of K-mask.1: Q_s / K_s complete past this
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      tc::mbar_arrive_expect_tx(bar_q, C::kTile);
      for (int p = 0; p < C::kPanels; ++p)
        tc::tma_load_3d(sQ + p * C::kPanel, &tmQ, bar_q, p * 64, row0, int(u));
      for (int T = 0; T < nseq; ++T) {
        const int s = T % C::kRing, t = seq_tile(T);
        tc::mbar_wait(bar_empty + s, ((T / C::kRing) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(bar_full + s, C::kTile);
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(sRing + s * C::kTile + p * C::kPanel, &tmK, bar_full + s, p * 64,
                          t * 128, int(u));
      }
    }
  } else if (warp == kWarpMma2) {
    // ===================== MMA issuer =====================
    if (BLADE_ISSUER(lane)) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      const uint32_t qa = smem_u32(sQ), rb = smem_u32(sRing);
      tc::mbar_wait(bar_q, 0);
      tc::fence_after_sync();
      for (int T = 0; T < nseq; ++T) {
        const int s = T % C::kRing, bsel = T & 1;
        tc::mbar_wait(bar_full + s, (T / C::kRing) & 1);
        if (T >= 2) tc::mbar_wait(bar_f + bsel, ((T >> 1) - 1) & 1);
        tc::fence_after_sync();
        const uint32_t kb = rb + s * C::kTile;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          BLADE_MMA_SS(tmem + bsel * 128, tc::sw128_desc(qa + off, 16, 1024),
                     tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
        }
        BLADE_COMMIT(bar_s + bsel);
        BLADE_COMMIT(bar_empty + s);
      }
    }
  } else {
    // ===================== row statistics =====================
    const int par = warp >> 3, h = (warp >> 2) & 1, quad = warp & 3;
    const int grp = warp >> 2;  // (par, h): which of the four partial states
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    const int r = quad * 32 + lane;
    const int gr = row0 + r;
    const int ib = gr / KK;
    const bool row_ok = gr < NK && (gr % KK) < min(KK, N - ib * b);
    float m_run = -INFINITY;
    double l_run = 0.0;
    float M = 0.f, lg = 0.f;
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    for (int pass = 0; pass < npass; ++pass) {
      const int Ta = pass == 0 ? 0 : ntiles + (pass - 1) * TPP;
      const int Tb = pass == 0 ? ntiles : ntiles + min(ntiles, (pass + 1) * TPP) - TPP;
      for (int T = Ta + ((Ta & 1) != par ? 1 : 0); T < Tb; T += 2) {
        const int t = seq_tile(T);
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
        // R: per key-block max of the raw logits (Alg. 3 l.12/l.15); with
        // k = b one value per half block, the halves combined when pooling
        uint32_t rv[CPH];
        float tmax = -INFINITY;
#pragma unroll
        for (int g = 0; g < CPH; ++g) {
          float gm = fmax3(s[g * KH], s[g * KH + 1], s[g * KH + 2]);
#pragma unroll
          for (int c = 3; c + 1 < KH; c += 2) gm = fmax3(gm, s[g * KH + c], s[g * KH + c + 1]);
          if ((KH & 1) == 0) gm = fmaxf(gm, s[g * KH + KH - 1]);
          tmax = fmaxf(tmax, gm);
          rv[g] = __float_as_uint(gm);
        }
        if (t >= pass * TPP && t < (pass + 1) * TPP) {  // R of this pass's tiles
          const uint32_t rcol = tmem + lane_base + 256 + (t - pass * TPP) * CPT + h * CPH;
          if constexpr (CPH == 4) {
            tc::st_32x32b_x4(rcol, reinterpret_cast<uint32_t(&)[4]>(rv));
          } else if constexpr (CPH == 2) {
            tc::st_32x32b_x2(rcol, reinterpret_cast<uint32_t(&)[2]>(rv));
          } else {
            tc::st_32x32b_x1(rcol, reinterpret_cast<uint32_t(&)[1]>(rv));
          }
        }
        if (pass > 0) continue;  // the row statistics are complete after pass 0
        // online row max / sum over this half tile (l.13-15)
        const float m_new = fmaxf(m_run, tmax);
        if (m_new != -INFINITY) {  // a half tile of padding only leaves (M, l) untouched
          const float2 nm2 = make_float2(-m_new, -m_new);
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 x = mul2(add2(make_float2(s[c], s[c + 1]), nm2), sc2);
            if ((kEmu >> ((c >> 1) & 7)) & 1) {
              const float2 y = ex2_poly5x2(x);
              s[c] = y.x;
              s[c + 1] = y.y;
            } else {
              s[c] = ex2(x.x);
              s[c + 1] = ex2(x.y);
            }
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
      if (pass == 0) smm[grp * 128 + r] = m_run, sml[grp * 128 + r] = l_run;
      tc::fence_before_sync();  // R columns written by every statistics warp, read below
      asm volatile("bar.sync 1, %0;\n" ::"n"(kSW * 32) : "memory");
      tc::fence_after_sync();
      if (pass == 0) {  // merge the four partial (M, l) of each row (l.14, once)
        M = -INFINITY;
#pragma unroll
        for (int g = 0; g < 4; ++g) M = fmaxf(M, smm[g * 128 + r]);
        double L = 0.0;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const float mg = smm[g * 128 + r];
          if (mg != -INFINITY) L += sml[g * 128 + r] * double(ex2((mg - M) * scale_log2));
        }
        lg = float(log2(L));
      }
      // pooling (l.17-19): v_sj = (R_sj - M_s) c - log2 l_s, P_imp = 2^(max_s v_sj);
      // rows of query block i are KK consecutive lanes (k > 32: spread over
      // warps, combined by atomicMax on the pre-zeroed output); the four
      // groups take interleaved 32-column chunks of this pass's R
      const int pc = min(256, Nb * CPB - pass * 256);  // R columns of this pass
      for (int c0 = grp * 32; c0 < pc; c0 += 128) {
        uint32_t rr[32];
        tc::ld_32x32b_x32(tmem + lane_base + 256 + c0, rr);
        tc::wait_ld();
        constexpr int NE = 32 / CPB;  // blocks per chunk
        const int j0 = (pass * 256 + c0) / CPB;
        float pv[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const float rmax = CPB == 2 ? fmaxf(__uint_as_float(rr[2 * e]), __uint_as_float(rr[2 * e + 1]))
                                      : __uint_as_float(rr[e]);
          float v = row_ok ? (rmax - M) * scale_log2 - lg : -INFINITY;
#pragma unroll
          for (int o = 1; o < KK && o < 32; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
          pv[e] = v;
        }
        const int nj = min(NE, Nb - j0);
        if (KK > 32) {  // a block spans several warps: max over them (pimp pre-zeroed)
          if (lane == 0 && ib < Nb) {
            float* dst = pimp + (u * Nb + ib) * int64_t(Nb) + j0;
            for (int e = 0; e < nj; ++e)
              atomicMax(reinterpret_cast<int*>(dst + e), __float_as_int(ex2(pv[e])));
          }
        } else if ((lane % KK) == 0 && ib < Nb) {
          float* dst = pimp + (u * Nb + ib) * int64_t(Nb) + j0;
          if (nj == 32 && (Nb % 4) == 0) {
#pragma unroll
            for (int e = 0; e < NE; e += 4)
              *reinterpret_cast<float4*>(dst + e) =
                  make_float4(ex2(pv[e]), ex2(pv[e + 1]), ex2(pv[e + 2]), ex2(pv[e + 3]));
          } else {
#pragma unroll
            for (int e = 0; e < NE; ++e)
              if (e < nj) dst[e] = ex2(pv[e]);
          }
        }
      }
      if (pass + 1 < npass) {  // R reads of this pass done before the next pass writes R
        tc::fence_before_sync();
        asm volatile("bar.sync 1, %0;\n" ::"n"(kSW * 32) : "memory");
        tc::fence_after_sync();
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kWarpMma2) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int D, int KK>
cudaError_t launch_p2(int64_t BH, int N, int Nb, int b, float scale, const void* qs,
                      const void* ks, float* pimp, cudaStream_t stream) {
  CUtensorMap mq, mk;
  const int64_t NK = int64_t(Nb) * KK;
  if (!make_tile_map(&mq, qs, BH, NK, D) || !make_tile_map(&mk, ks, BH, NK, D))
    return cudaErrorNotSupported;
  constexpr int smem = P2Cfg<D>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(probe2_kernel<D, KK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (KK > 32) {  // pooled by atomicMax over two warps (non-negative floats)
    e = cudaMemsetAsync(pimp, 0, size_t(BH) * Nb * Nb * 4, stream);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(unsigned((NK + 127) / 128), unsigned(BH));
  // programmatic dependent launch behind K-mask.1 (sample_gather_kernel): the
  // prologue (barriers, TMEM, descriptor prefetch) overlaps its tail
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kP2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, probe2_kernel<D, KK>, mq, mk, N, Nb, b,
                         scale * 1.4426950408889634f, pimp);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

bool probe2_supported(int d, int kk, int Nb, int64_t, int) {
  // R lives in TMEM columns [256, 512), in passes of 256 columns
  return (d == 64 || d == 128) && (kk == 16 || kk == 32 || kk == 64 || kk == 128) && Nb <= 512;
}

cudaError_t launch_probe2(int64_t BH, int N, int Nb, int b, int kk, int d, float scale,
                          const void* qs, const void* ks, float* pimp, cudaStream_t stream) {
  if (d == 128 && kk == 16) return launch_p2<128, 16>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 128 && kk == 32) return launch_p2<128, 32>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 128 && kk == 64) return launch_p2<128, 64>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 64 && kk == 16) return launch_p2<64, 16>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 64 && kk == 32) return launch_p2<64, 32>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 64 && kk == 64) return launch_p2<64, 64>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 128 && kk == 128) return launch_p2<128, 128>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  if (d == 64 && kk == 128) return launch_p2<64, 128>(BH, N, Nb, b, scale, qs, ks, pimp, stream);
  return cudaErrorNotSupported;
}

}  // namespace blade
