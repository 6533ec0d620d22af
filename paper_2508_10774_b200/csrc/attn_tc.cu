// attn_tc.cu — block-sparse attention forward for sm_100a on the 5th-gen
// tensor cores (tcgen05 + TMEM + TMA).  PAPER.md P:133 (Step 2.2 (1),
// "Standard ASA ... integrated with a block-sparse attention kernel").
//
// CTA = two query blocks (i0 = 2p, i1 = 2p+1) of one unit: two 128-row Q
// tiles whose kept-block lists are walked as one ascending UNION, so a key
// block kept by both tiles is loaded once (adjacent blocks of a locality-
// ordered video sequence keep mostly the same key blocks).  Warp roles:
//   warps 0-3  softmax, tile 0 (thread = query row = TMEM lane)
//   warps 4-7  softmax, tile 1
//   warp  8    tcgen05.mma issuer (one thread) + TMEM allocator
//   warp  9    TMA producer (one thread): Q tiles once, then K_j, V_j per
//              union block into a ring of 128-key smem slots
//   warps 10-11 idle (complete the third warpgroup for setmaxnreg)
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+d) O1 [256+d, ..).
// P_t (bf16) overwrites the upper half of S_t and is the A operand of the
// P V MMA straight from TMEM.  MMA issue order per union block n:
//   PV_t(n) then S_t(n+1) for each tile t kept there (FA4-style ping-pong
//   between the two tiles' softmax warpgroups).  O is rescaled lazily, only
//   when a row max grows by more than 2^8.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"
#include "tma_host.h"

namespace blade {
namespace {

template <int D>
struct Cfg {
  static constexpr int kTile = 128 * D * 2;          // Q tile / K slot / V slot bytes
  static constexpr int kPanels = D / 64;             // 128-byte SW128 panels along d
  static constexpr int kPanel = 128 * 128;           // 128 rows x 128 B
  static constexpr int kRing = D == 128 ? 4 : 8;     // K/V slots
  static constexpr int kOffRing = 2 * kTile;
  static constexpr int kOffBar = kOffRing + kRing * kTile;
  static constexpr int kNumBar = 1 + 2 * kRing + 6;
  static constexpr int kOffMisc = kOffBar + kNumBar * 8;
  static constexpr int kSmem = kOffMisc + 16 + 3 * 16 * 4 + 1024;  // + align slack
  static __device__ __forceinline__ uint32_t col_s(int t) { return uint32_t(t) * 128u; }
  static __device__ __forceinline__ uint32_t col_o(int t) { return 256u + uint32_t(t) * D; }
};

constexpr int kThreads = 384;  // 3 warpgroups; warps 10-11 idle
constexpr float kRescaleThreshold = 8.0f;  // log2 units

BLADE_DEVINL int next_block(const uint32_t* bm, int from, int nwords) {
  int w = from >> 5;
  if (w >= nwords) return -1;
  uint32_t bits = bm[w] & (~0u << (from & 31));
  while (true) {
    if (bits) return (w << 5) + __ffs(bits) - 1;
    if (++w >= nwords) return -1;
    bits = bm[w];
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, int N, int Nb, float scale_log2,
                   const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
                   __nv_bfloat16* __restrict__ O, float* __restrict__ LSE,
                   volatile int* dbg) {
  using C = Cfg<D>;
  const bool dbg_on = dbg != nullptr && blockIdx.x == 0 && blockIdx.y == 0;
#define TC_DBG(i, v) \
  do {               \
    if (dbg_on) dbg[i] = (v); \
  } while (0)
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  char* sQ = smem;
  char* sRing = smem + C::kOffRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_full = bars + 1;
  uint64_t* bar_empty = bars + 1 + C::kRing;
  uint64_t* bar_s = bars + 1 + 2 * C::kRing;     // [2]
  uint64_t* bar_p = bar_s + 2;                    // [2]
  uint64_t* bar_o = bar_p + 2;                    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  uint32_t* bm = tmem_slot + 4;                   // [2][16] kept-block bitmaps + [16] union
  int* last_blk = reinterpret_cast<int*>(tmem_slot + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t u = blockIdx.y;
  const int i0 = blockIdx.x * 2;
  const int ntile = (i0 + 1 < Nb) ? 2 : 1;
  const int nwords = (Nb + 31) >> 5;

  // ---- setup: kept-block bitmaps, barriers, TMEM ------------------------------
  if (tid < 32) bm[tid] = 0;
  __syncthreads();
  for (int t = 0; t < ntile; ++t) {
    const int64_t row = u * Nb + i0 + t;
    const int cnt = kv_cnt[row];
    const int32_t* lst = kv_idx + row * Nb;
    for (int e = tid; e < cnt; e += kThreads) {
      const int j = lst[e];
      atomicOr(&bm[t * 16 + (j >> 5)], 1u << (j & 31));
    }
  }
  if (warp == 9 && lane == 0) {
    tc::mbar_init(bar_q, 1);
    for (int s = 0; s < C::kRing; ++s) {
      tc::mbar_init(bar_full + s, 1);
      tc::mbar_init(bar_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(bar_s + t, 1);
      tc::mbar_init(bar_p + t, 128);
      tc::mbar_init(bar_o + t, 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 8) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) TC_DBG(10, int(tmem));
  if (tid < 16) bm[32 + tid] = bm[tid] | bm[16 + tid];
  if (tid < 2) {
    int lb = -1;
    for (int w = nwords - 1; w >= 0 && lb < 0; --w)
      if (bm[tid * 16 + w]) lb = (w << 5) + 31 - __clz(bm[tid * 16 + w]);
    last_blk[tid] = lb;
  }
  __syncthreads();

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::);
  if (warp == 9) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmQ);
      tc::tma_prefetch_desc(&tmK);
      tc::tma_prefetch_desc(&tmV);
      tc::mbar_arrive_expect_tx(bar_q, ntile * C::kTile);
      for (int t = 0; t < ntile; ++t)
        for (int p = 0; p < C::kPanels; ++p)
          tc::tma_load_3d(sQ + t * C::kTile + p * C::kPanel, &tmQ, bar_q, p * 64, (i0 + t) * 128,
                          int(u));
      uint32_t L = 0;
      uint32_t* un = bm + 32;
      for (int j = next_block(un, 0, nwords); j >= 0; j = next_block(un, j + 1, nwords)) {
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++L) {
          const int s = L % C::kRing;
          TC_DBG(0, 2 * int(L));
          tc::mbar_wait(bar_empty + s, ((L / C::kRing) & 1) ^ 1);
          TC_DBG(0, 2 * int(L) + 1);
          tc::mbar_arrive_expect_tx(bar_full + s, C::kTile);
          for (int p = 0; p < C::kPanels; ++p)
            tc::tma_load_3d(sRing + s * C::kTile + p * C::kPanel, kv ? &tmV : &tmK, bar_full + s,
                            p * 64, j * 128, int(u));
        }
      }
    }
  } else if (warp == 8) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, D, 0, 1);
      const uint32_t qbase = smem_u32(sQ), rbase = smem_u32(sRing);
      const uint32_t* un = bm + 32;
      auto in_tile = [&](int t, int j) -> bool { return (bm[t * 16 + (j >> 5)] >> (j & 31)) & 1u; };
      auto issue_S = [&](int t, uint32_t slot) {
        const uint32_t qa = qbase + t * C::kTile, kb = rbase + slot * C::kTile;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * C::kPanel + (ks & 3) * 32;
          tc::mma_ss(tmem + C::col_s(t), tc::sw128_desc(qa + off, 16, 1024),
                     tc::sw128_desc(kb + off, 16, 1024), idS, ks > 0);
        }
        tc::commit(bar_s + t);
      };
      auto issue_PV = [&](int t, uint32_t slot, bool acc) {
        const uint32_t vb = rbase + slot * C::kTile;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc::mma_ts(tmem + C::col_o(t), tmem + C::col_s(t) + 64 + ks * 8,
                     tc::sw128_desc(vb + ks * 2048, C::kPanel, 1024), idO, (acc || ks > 0) ? 1 : 0);
      };
      auto wait_full = [&](uint32_t L) {
        tc::mbar_wait(bar_full + L % C::kRing, (L / C::kRing) & 1);
        tc::fence_after_sync();
      };
      TC_DBG(1, 1);
      tc::mbar_wait(bar_q, 0);
      TC_DBG(1, 2);
      tc::fence_after_sync();
      uint32_t pcnt[2] = {0, 0};
      bool first[2] = {true, true};
      int j = next_block(un, 0, nwords);
      uint32_t n = 0;  // union index of j; K(n) is load 2n, V(n) load 2n+1
      // prologue: S of the first union block
      wait_full(0);
      for (int t = 0; t < ntile; ++t)
        if (in_tile(t, j)) issue_S(t, 0);
      tc::commit(bar_empty + 0);
      while (j >= 0) {
        const int jn = next_block(un, j + 1, nwords);
        const uint32_t LK1 = 2 * (n + 1), LV = 2 * n + 1;
        bool kready = false;
        // tiles that skip j but keep jn: start their next S as early as possible
        for (int t = 0; t < ntile; ++t) {
          if (jn >= 0 && !in_tile(t, j) && in_tile(t, jn)) {
            if (!kready) { wait_full(LK1); kready = true; }
            issue_S(t, LK1 % C::kRing);
          }
        }
        TC_DBG(1, 100 + 10 * int(n));
        wait_full(LV);
        TC_DBG(1, 101 + 10 * int(n));
        for (int t = 0; t < ntile; ++t) {
          if (!in_tile(t, j)) continue;
          TC_DBG(1, 102 + t + 10 * int(n));
          tc::mbar_wait(bar_p + t, pcnt[t] & 1);
          TC_DBG(1, 104 + t + 10 * int(n));
          ++pcnt[t];
          tc::fence_after_sync();
          issue_PV(t, LV % C::kRing, !first[t]);
          first[t] = false;
          if (j == last_blk[t]) tc::commit(bar_o + t);
          if (jn >= 0 && in_tile(t, jn)) {
            if (!kready) { wait_full(LK1); kready = true; }
            issue_S(t, LK1 % C::kRing);
          }
        }
        tc::commit(bar_empty + LV % C::kRing);
        if (jn >= 0) tc::commit(bar_empty + LK1 % C::kRing);
        j = jn;
        ++n;
      }
      // drain: the last commits must land before the CTA's smem is released
      const uint32_t LV = 2 * (n - 1) + 1;
      TC_DBG(1, 5000);
      tc::mbar_wait(bar_empty + LV % C::kRing, (LV / C::kRing) & 1);
      TC_DBG(1, 5001);
    }
  }
  } else {
    // ===================== softmax warpgroups =====================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::);
    const int t = warp >> 2, quad = warp & 3;
    if (t < ntile) {
      const uint32_t lane_base = uint32_t(quad * 32) << 16;
      const uint32_t tS = tmem + lane_base + C::col_s(t);
      const uint32_t tO = tmem + lane_base + C::col_o(t);
      const uint32_t* mybm = bm + t * 16;
      float m_used = -INFINITY, l_sum = 0.f;
      uint32_t cnt = 0;
      for (int j = next_block(mybm, 0, nwords); j >= 0; j = next_block(mybm, j + 1, nwords), ++cnt) {
        if (lane == 0) TC_DBG(2 + warp, 10 * int(cnt) + 1);
        tc::mbar_wait(bar_s + t, cnt & 1);
        if (lane == 0) TC_DBG(2 + warp, 10 * int(cnt) + 2);
        tc::fence_after_sync();
        float s[128];
        {
          uint32_t r0[32], r1[32], r2[32], r3[32];
          tc::ld_32x32b_x32(tS + 0, r0);
          tc::ld_32x32b_x32(tS + 32, r1);
          tc::ld_32x32b_x32(tS + 64, r2);
          tc::ld_32x32b_x32(tS + 96, r3);
          tc::wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            s[e] = __uint_as_float(r0[e]);
            s[32 + e] = __uint_as_float(r1[e]);
            s[64 + e] = __uint_as_float(r2[e]);
            s[96 + e] = __uint_as_float(r3[e]);
          }
        }
        const int valid = N - j * 128;
        if (valid < 128) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= valid) s[c] = -INFINITY;
        }
        float mx = s[0];
#pragma unroll
        for (int c = 1; c < 128; ++c) mx = fmaxf(mx, s[c]);
        const float mxs = mx * scale_log2;
        // warp-uniform decision (tcgen05.ld/st below are .sync.aligned); true on the
        // first block since m_used = -inf
        if (__any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold)) {
          const float m_new = fmaxf(m_used, mxs);
          if (cnt > 0) {
            const float f = ex2(m_used - m_new);
            l_sum *= f;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t r[32];
              tc::ld_32x32b_x32(tO + c * 32, r);
              tc::wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * f);
              tc::st_32x32b_x32(tO + c * 32, r);
            }
          }
          m_used = m_new;
        }
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float p0 = ex2(fmaf(s[c * 32 + 2 * e], scale_log2, -m_used));
            const float p1 = ex2(fmaf(s[c * 32 + 2 * e + 1], scale_log2, -m_used));
            acc += p0 + p1;
            pk[e] = pack_bf16(p0, p1);
          }
          tc::st_32x32b_x16(tS + 64 + c * 16, pk);
        }
        l_sum += acc;
        tc::wait_st();
        tc::fence_before_sync();
        tc::mbar_arrive(bar_p + t);
        if (lane == 0) TC_DBG(2 + warp, 10 * int(cnt) + 3);
      }
      // epilogue: O / l -> bf16, LSE
      if (lane == 0) TC_DBG(2 + warp, 9000);
      tc::mbar_wait(bar_o + t, 0);
      if (lane == 0) TC_DBG(2 + warp, 9001);
      tc::fence_after_sync();
      const int row = (i0 + t) * 128 + quad * 32 + lane;
      const float inv = 1.f / l_sum;
      __nv_bfloat16* orow = O + (u * N + row) * int64_t(D);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tc::ld_32x32b_x32(tO + c * 32, r);
        tc::wait_ld();
        if (row < N) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(r[8 * e + 0]) * inv, __uint_as_float(r[8 * e + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(r[8 * e + 2]) * inv, __uint_as_float(r[8 * e + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(r[8 * e + 4]) * inv, __uint_as_float(r[8 * e + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(r[8 * e + 6]) * inv, __uint_as_float(r[8 * e + 7]) * inv);
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
  if (tid == 0) TC_DBG(11, 777);
#undef TC_DBG
}

template <int D>
cudaError_t launch_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                     const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                     cudaStream_t stream) {
  CUtensorMap mq, mk, mv;
  if (!make_tile_map(&mq, q, p.BH, p.N, D) || !make_tile_map(&mk, k, p.BH, p.N, D) ||
      !make_tile_map(&mv, v, p.BH, p.N, D))
    return cudaErrorNotSupported;
  constexpr int smem = Cfg<D>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned((p.Nb + 1) / 2), unsigned(p.BH));
  // BLADE_TC_DEBUG=1: CTA (0,0) writes role progress to mapped host memory and
  // the launcher waits up to 5 s, dumping the progress and exiting on a hang.
  static int* dbg_host = nullptr;
  int* dbg_dev = nullptr;
  const char* env = getenv("BLADE_TC_DEBUG");
  if (env && env[0] == '1') {
    if (!dbg_host) cudaHostAlloc(&dbg_host, 64 * sizeof(int), cudaHostAllocMapped);
    memset(dbg_host, 0xff, 64 * sizeof(int));
    cudaHostGetDevicePointer(&dbg_dev, dbg_host, 0);
  }
  attn_tc_kernel<D><<<grid, kThreads, smem, stream>>>(
      mq, mk, mv, p.N, p.Nb, p.scale * kLog2e, kv_idx, kv_cnt,
      reinterpret_cast<__nv_bfloat16*>(o), lse, dbg_dev);
  e = cudaGetLastError();
  if (dbg_dev && e == cudaSuccess) {
    for (int it = 0; it < 500 && cudaStreamQuery(stream) == cudaErrorNotReady; ++it) usleep(10000);
    if (cudaStreamQuery(stream) == cudaErrorNotReady) {
      fprintf(stderr, "attn_tc HANG: load=%d mma=%d softmax=[%d %d %d %d | %d %d %d %d] tmem=%d end=%d\n",
              dbg_host[0], dbg_host[1], dbg_host[2], dbg_host[3], dbg_host[4], dbg_host[5],
              dbg_host[6], dbg_host[7], dbg_host[8], dbg_host[9], dbg_host[10], dbg_host[11]);
      fflush(stderr);
      _exit(3);
    }
  }
  return e;
}

}  // namespace

size_t attn_tc_workspace(const AttnProblem&) { return 256; }

cudaError_t launch_attn_tc(const AttnProblem& p, const void* q, const void* k, const void* v,
                           const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                           char*, size_t, cudaStream_t stream) {
  if (p.d == 64) return launch_d<64>(p, q, k, v, kv_idx, kv_cnt, o, lse, stream);
  if (p.d == 128) return launch_d<128>(p, q, k, v, kv_idx, kv_cnt, o, lse, stream);
  return cudaErrorNotSupported;
}

}  // namespace blade
