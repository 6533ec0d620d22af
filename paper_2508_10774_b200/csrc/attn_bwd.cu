// attn_bwd.cu — block-sparse attention backward (F3; PAPER.md P:158-161:
// sparsity-aware distillation trains the student through the ASA mechanism,
// so the gradient flows through the masked attention of P:133).  Reading
// R-23: the mask (kv lists) is a constant of the backward.
//
// For query row r and its kept keys T(r), with P_rt = exp(scale q_r.k_t - LSE_r):
//   D_r   = dO_r . O_r                                   (bsa_bwd_dot_kernel)
//   dV_t  = sum_r P_rt dO_r
//   dK_t  = scale sum_r P_rt (dO_r . v_t - D_r) q_r      (bsa_bwd_dkdv_kernel)
//   dQ_r  = scale sum_t P_rt (dO_r . v_t - D_r) k_t      (bsa_bwd_dq_kernel)
// dK/dV walk, per key block, the TRANSPOSED lists (query blocks that keep
// it; bsa_bwd_transpose_kernel), dQ walks the forward lists, so every output
// row is written by exactly one CTA (no atomics, deterministic).
//
// The dK/dV and dQ products run in the tcgen05 kernels of attn_bwd_tc.cu;
// the mma.sync kernels below (FlashAttention-2 structure: CTA = 64 rows, 4
// warps x 16 rows, 64-row tiles of the other operand double-buffered with
// cp.async) are the legacy-tensor-path baseline, compiled only into
// -DBLADE_WITH_BASELINES builds (selectable there with
// -DBLADE_BWD_{DKDV,DQ}_MMA_SYNC; 12.3 ms vs 3.9 ms on the Wan layer); the
// product build returns UNSUPPORTED where a TMA tensor map cannot be built.
// P and dS are rounded to bf16 for their MMAs in both.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/blade_asa.h"
#include "common.cuh"
#include "internal.h"

namespace blade {
namespace {

constexpr int BW_ROWS = 64;   // rows owned by a CTA
constexpr int BW_TILE = 64;   // rows of the streamed operand per step
constexpr int BW_THREADS = 128;
constexpr int kMaxNbBwd = 512;

// ---- D_r = dO_r . O_r --------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) bsa_bwd_dot_kernel(const __nv_bfloat16* __restrict__ O,
                                                         const __nv_bfloat16* __restrict__ dO,
                                                         int64_t rows, float* __restrict__ Dv) {
  constexpr int G = D / 8;  // lanes per row, one 16-byte vector each
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t row = t / G;
  const int c = int(t % G);
  float acc = 0.f;
  if (row < rows) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(O + row * D) + c);
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(dO + row * D) + c);
    const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 fa = __bfloat1622float2(ha[e]), fb = __bfloat1622float2(hb[e]);
      acc = fmaf(fa.x, fb.x, acc);
      acc = fmaf(fa.y, fb.y, acc);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (row < rows && c == 0) Dv[row] = acc;
}

// ---- transposed lists: q_idx[u, j, :] = query blocks i with j in kv_idx[u, i] -
// CTA = (unit, 32 key blocks j0..j0+31): scans the unit's lists, sets bit i of
// j's row in a [32][N_b/32] smem bitmap, then one thread per j emits its
// query blocks in ascending order.
__global__ void __launch_bounds__(256) bsa_bwd_transpose_kernel(const int32_t* __restrict__ kv_idx,
                                                               const int32_t* __restrict__ kv_cnt,
                                                               int Nb, int32_t* __restrict__ q_idx,
                                                               int32_t* __restrict__ q_cnt) {
  __shared__ uint32_t bm[32][kMaxNbBwd / 32];  // [key block j - j0][query word]
  const int64_t u = blockIdx.y;
  const int j0 = blockIdx.x * 32;
  const int nw = (Nb + 31) / 32;
  for (int e = threadIdx.x; e < 32 * nw; e += blockDim.x) bm[e / nw][e % nw] = 0u;
  __syncthreads();
  __shared__ int scnt[kMaxNbBwd];
  const int32_t* li = kv_idx + u * Nb * Nb;
  for (int i = threadIdx.x; i < Nb; i += blockDim.x) scnt[i] = __ldg(kv_cnt + u * Nb + i);
  __syncthreads();
  // 8 independent loads in flight per thread (the scan is latency-bound)
  const int total = Nb * Nb;
  for (int base = threadIdx.x; base < total; base += 8 * blockDim.x) {
    int val[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = base + q * blockDim.x;
      val[q] = e < total ? __ldg(li + e) : -1;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = base + q * blockDim.x;
      if (e < total) {
        const int i = e / Nb, k = e % Nb;
        const int j = val[q] - j0;
        if (k < scnt[i] && j >= 0 && j < 32) atomicOr(&bm[j][i >> 5], 1u << (i & 31));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 32 && j0 + int(threadIdx.x) < Nb) {
    const int j = j0 + threadIdx.x;
    int32_t* out = q_idx + (u * Nb + j) * Nb;
    int n = 0;
    for (int w = 0; w < nw; ++w) {
      uint32_t bits = bm[threadIdx.x][w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        out[n++] = w * 32 + b;
      }
    }
    q_cnt[u * Nb + j] = n;
  }
}

// 64 rows x D bf16 tile, rows past N zero-filled (cp.async, 16-byte chunks)
template <int D>
BLADE_DEVINL void load_tile(uint32_t dst, const __nv_bfloat16* base, int row0, int N, int tid) {
  constexpr int CH = D / 8;
  for (int e = tid; e < BW_TILE * CH; e += BW_THREADS) {
    const int r = e / CH, c = e % CH;
    const int gr = row0 + r;
    cp_async16(dst + swz<D>(r, c), base + int64_t(min(gr, N - 1)) * D + c * 8, gr < N ? 16 : 0);
  }
}

// A fragments (16 rows x 16 cols per k-step) of the warp's 16 rows of a tile
template <int D>
BLADE_DEVINL void load_a_rows(uint32_t tile, int row0, int lane, uint32_t (&a)[D / 16][4]) {
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int r = row0 + (lane & 7) + 8 * ((lane >> 3) & 1);
    const int c = ks * 2 + (lane >> 4);
    ldsm_x4(tile + swz<D>(r, c), a[ks][0], a[ks][1], a[ks][2], a[ks][3]);
  }
}

// acc[8][4] (16 rows x 64 cols) = A(16 x D) * Bt^T where Bt is a 64 x D tile
// in smem (cols of the result = rows of Bt)
template <int D>
BLADE_DEVINL void mma_rows_x_tileT(const uint32_t (&a)[D / 16][4], uint32_t bt, int lane,
                                   float (&acc)[8][4]) {
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b0, b1, b2, b3;
      const int r = np * 16 + (lane & 7) + 8 * (lane >> 4);
      const int c = ks * 2 + ((lane >> 3) & 1);
      ldsm_x4(bt + swz<D>(r, c), b0, b1, b2, b3);
      mma_bf16(acc[2 * np], a[ks], b0, b1);
      mma_bf16(acc[2 * np + 1], a[ks], b2, b3);
    }
  }
}

// out[D/8][4] (16 rows x D) += P(16 x 64, fp32 fragments, rounded to bf16) * T
// where T is a 64 x D tile in smem (rows = the contracted index)
template <int D>
BLADE_DEVINL void mma_p_x_tile(const float (&p)[8][4], uint32_t tile, int lane,
                               float (&out)[D / 8][4]) {
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {
    uint32_t pa[4];
    pa[0] = pack_bf16(p[2 * kt][0], p[2 * kt][1]);
    pa[1] = pack_bf16(p[2 * kt][2], p[2 * kt][3]);
    pa[2] = pack_bf16(p[2 * kt + 1][0], p[2 * kt + 1][1]);
    pa[3] = pack_bf16(p[2 * kt + 1][2], p[2 * kt + 1][3]);
#pragma unroll
    for (int dp = 0; dp < D / 16; ++dp) {
      uint32_t b0, b1, b2, b3;
      const int r = kt * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
      const int c = dp * 2 + (lane >> 4);
      ldsm_x4_t(tile + swz<D>(r, c), b0, b1, b2, b3);
      mma_bf16(out[2 * dp], pa, b0, b1);
      mma_bf16(out[2 * dp + 1], pa, b2, b3);
    }
  }
}

template <int D>
BLADE_DEVINL void store_rows(__nv_bfloat16* base, int row0_global, int N, int lane,
                             const float (&acc)[D / 8][4], float mul) {
  const int g = lane >> 2, qd = lane & 3;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = row0_global + g + 8 * h;
    if (r < N) {
      __nv_bfloat16* row = base + int64_t(r) * D;
#pragma unroll
      for (int n = 0; n < D / 8; ++n)
        *reinterpret_cast<uint32_t*>(row + n * 8 + qd * 2) =
            pack_bf16(acc[n][2 * h] * mul, acc[n][2 * h + 1] * mul);
    }
  }
}

// ---- dK, dV: CTA = 64 keys (half of key block j), walks the query blocks
//      that keep j, 64 queries at a time --------------------------------------
template <int D>
__global__ void __launch_bounds__(BW_THREADS) bsa_bwd_dkdv_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
    const __nv_bfloat16* __restrict__ V, const __nv_bfloat16* __restrict__ dO,
    const float* __restrict__ LSE, const float* __restrict__ Dv, int N, int Nb, float scale,
    const int32_t* __restrict__ q_idx, const int32_t* __restrict__ q_cnt,
    __nv_bfloat16* __restrict__ dK, __nv_bfloat16* __restrict__ dV) {
  extern __shared__ __align__(128) char smem[];
  constexpr int TB = BW_TILE * D * 2;
  char* sK = smem;
  char* sV = sK + TB;
  char* sQ = sV + TB;        // [2]
  char* sdO = sQ + 2 * TB;   // [2]
  float* sL = reinterpret_cast<float*>(sdO + 2 * TB);  // [2][64] LSE * log2 e
  float* sD = sL + 2 * BW_TILE;                         // [2][64] D_r
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = blockIdx.x >> 1;
  const int key0 = j * 128 + (blockIdx.x & 1) * BW_ROWS;
  const int64_t u = blockIdx.y;
  const int64_t base = u * int64_t(N) * D;
  if (key0 >= N) return;
  const int nq = q_cnt[u * Nb + j];
  const int32_t* qlist = q_idx + (u * Nb + j) * Nb;
  const int ntiles = 2 * nq;  // 64-query tiles
  const float sl2 = scale * kLog2e;

  load_tile<D>(smem_u32(sK), K + base, key0, N, tid);
  load_tile<D>(smem_u32(sV), V + base, key0, N, tid);
  auto load_q = [&](int t, int st) {
    const int q0 = qlist[t >> 1] * 128 + (t & 1) * BW_TILE;
    load_tile<D>(smem_u32(sQ + st * TB), Q + base, q0, N, tid);
    load_tile<D>(smem_u32(sdO + st * TB), dO + base, q0, N, tid);
    if (tid < BW_TILE) {
      const int r = q0 + tid;
      sL[st * BW_TILE + tid] = r < N ? LSE[u * N + r] * kLog2e : INFINITY;  // P = 0 past N
      sD[st * BW_TILE + tid] = r < N ? Dv[u * N + r] : 0.f;
    }
  };
  if (ntiles > 0) load_q(0, 0);
  cp_async_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;
  const int qd = lane & 3;

  for (int t = 0; t < ntiles; ++t) {
    const int st = t & 1;
    if (t + 1 < ntiles) load_q(t + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t q_t = smem_u32(sQ + st * TB), do_t = smem_u32(sdO + st * TB);
    const float* L = sL + st * BW_TILE;
    const float* Dd = sD + st * BW_TILE;
    // P^T (16 keys x 64 queries) = exp2(scale log2e K Q^T - LSE log2e)
    float p[8][4];
    {
      uint32_t ka[D / 16][4];
      load_a_rows<D>(smem_u32(sK), warp * 16, lane, ka);
      mma_rows_x_tileT<D>(ka, q_t, lane, p);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float l0 = L[n * 8 + qd * 2], l1 = L[n * 8 + qd * 2 + 1];
      p[n][0] = ex2(fmaf(p[n][0], sl2, -l0));
      p[n][1] = ex2(fmaf(p[n][1], sl2, -l1));
      p[n][2] = ex2(fmaf(p[n][2], sl2, -l0));
      p[n][3] = ex2(fmaf(p[n][3], sl2, -l1));
    }
    // dV += P^T dO
    mma_p_x_tile<D>(p, do_t, lane, dv);
    // dP^T = V dO^T; dS^T = P^T (dP^T - D)
    float ds[8][4];
    {
      uint32_t va[D / 16][4];
      load_a_rows<D>(smem_u32(sV), warp * 16, lane, va);
      mma_rows_x_tileT<D>(va, do_t, lane, ds);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float d0 = Dd[n * 8 + qd * 2], d1 = Dd[n * 8 + qd * 2 + 1];
      ds[n][0] = p[n][0] * (ds[n][0] - d0);
      ds[n][1] = p[n][1] * (ds[n][1] - d1);
      ds[n][2] = p[n][2] * (ds[n][2] - d0);
      ds[n][3] = p[n][3] * (ds[n][3] - d1);
    }
    // dK += dS^T Q  (scaled at the end)
    mma_p_x_tile<D>(ds, q_t, lane, dk);
    __syncthreads();
  }
  store_rows<D>(dK + base, key0 + warp * 16, N, lane, dk, scale);
  store_rows<D>(dV + base, key0 + warp * 16, N, lane, dv, 1.f);
}

// ---- dQ: CTA = 64 queries (half of query block i), walks i's kept blocks,
//      64 keys at a time ------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(BW_THREADS) bsa_bwd_dq_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
    const __nv_bfloat16* __restrict__ V, const __nv_bfloat16* __restrict__ dO,
    const float* __restrict__ LSE, const float* __restrict__ Dv, int N, int Nb, float scale,
    const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
    __nv_bfloat16* __restrict__ dQ) {
  extern __shared__ __align__(128) char smem[];
  constexpr int TB = BW_TILE * D * 2;
  char* sQ = smem;
  char* sdO = sQ + TB;
  char* sK = sdO + TB;       // [2]
  char* sV = sK + 2 * TB;    // [2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = blockIdx.x >> 1;
  const int q0 = i * 128 + (blockIdx.x & 1) * BW_ROWS;
  const int64_t u = blockIdx.y;
  const int64_t base = u * int64_t(N) * D;
  if (q0 >= N) return;
  const int cnt = kv_cnt[u * Nb + i];
  const int32_t* list = kv_idx + (u * Nb + i) * Nb;
  const int ntiles = 2 * cnt;
  const float sl2 = scale * kLog2e;

  load_tile<D>(smem_u32(sQ), Q + base, q0, N, tid);
  load_tile<D>(smem_u32(sdO), dO + base, q0, N, tid);
  auto load_kv = [&](int t, int st) {
    const int k0 = list[t >> 1] * 128 + (t & 1) * BW_TILE;
    load_tile<D>(smem_u32(sK + st * TB), K + base, k0, N, tid);
    load_tile<D>(smem_u32(sV + st * TB), V + base, k0, N, tid);
  };
  if (ntiles > 0) load_kv(0, 0);
  cp_async_commit();

  const int g = lane >> 2, qd = lane & 3;
  float lse2[2], dr[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = q0 + warp * 16 + g + 8 * h;
    lse2[h] = r < N ? LSE[u * N + r] * kLog2e : 0.f;
    dr[h] = r < N ? Dv[u * N + r] : 0.f;
  }
  float dq[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) dq[n][0] = dq[n][1] = dq[n][2] = dq[n][3] = 0.f;
  uint32_t qa[D / 16][4], doa[D / 16][4];

  for (int t = 0; t < ntiles; ++t) {
    const int st = t & 1;
    if (t + 1 < ntiles) load_kv(t + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
      load_a_rows<D>(smem_u32(sQ), warp * 16, lane, qa);
      load_a_rows<D>(smem_u32(sdO), warp * 16, lane, doa);
    }
    const uint32_t k_t = smem_u32(sK + st * TB), v_t = smem_u32(sV + st * TB);
    const int k0 = list[t >> 1] * 128 + (t & 1) * BW_TILE;
    float p[8][4], ds[8][4];
    mma_rows_x_tileT<D>(qa, k_t, lane, p);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = k0 + n * 8 + qd * 2 + (e & 1) < N;
        p[n][e] = ok ? ex2(fmaf(p[n][e], sl2, -lse2[e >> 1])) : 0.f;
      }
    }
    mma_rows_x_tileT<D>(doa, v_t, lane, ds);
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) ds[n][e] = p[n][e] * (ds[n][e] - dr[e >> 1]);
    mma_p_x_tile<D>(ds, k_t, lane, dq);
    __syncthreads();
  }
  store_rows<D>(dQ + base, q0 + warp * 16, N, lane, dq, scale);
}

// ---- ASA_GT backward (F1 + F3; oracle
//      sparse_attention_gt_backward_unit).  With the forward's LSE taken over
//      the kept keys AND the global tokens, P_rt = exp(s_rt - LSE_r) and D_r =
//      dO_r . O_r already make the plain kernels above exact for the kept
//      keys; the global tokens add, per window w (bias b_w = ln n_w):
//        dVg_w = sum_r P_rw dO_r,  dKg_w = scale sum_r dS_rw q_r  (every query)
//        dQ_r += scale sum_w dS_rw kg_w
//      and MeanPool_n passes dKg_w / n_w, dVg_w / n_w to each token of w
//      (the bf16 rounding of the pooled rows is the identity, R-24). ---------

BLADE_DEVINL float gt_bias_log2(int w, int Ng, int N, int window) {
  if (w >= Ng) return -INFINITY;  // padding rows / cols of the last 64-tile
  return __logf(float(min(window, N - w * window))) * kLog2e;
}

// CTA = (64 global tokens g0.., head u, query-tile split s): dKg, dVg partial
// sums over the split's 64-query tiles, fp32 to part[{0,1}][s][u][Ngp][D].
template <int D>
__global__ void __launch_bounds__(BW_THREADS) gt_bwd_dkdv_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Kg,
    const __nv_bfloat16* __restrict__ Vg, const __nv_bfloat16* __restrict__ dO,
    const float* __restrict__ LSE, const float* __restrict__ Dv, int N, int Ng, int window,
    float scale, int tiles_per_split, int64_t part_stride, float* __restrict__ part) {
  extern __shared__ __align__(128) char smem[];
  constexpr int TB = BW_TILE * D * 2;
  char* sK = smem;
  char* sV = sK + TB;
  char* sQ = sV + TB;        // [2]
  char* sdO = sQ + 2 * TB;   // [2]
  float* sL = reinterpret_cast<float*>(sdO + 2 * TB);
  float* sD = sL + 2 * BW_TILE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g0 = blockIdx.x * BW_ROWS;
  const int64_t u = blockIdx.y;
  const int s = blockIdx.z;
  const int Ngp = gridDim.x * BW_ROWS;
  const int nqt = (N + BW_TILE - 1) / BW_TILE;
  const int t0 = s * tiles_per_split, t1 = min(nqt, t0 + tiles_per_split);
  const int64_t base = u * int64_t(N) * D;
  const int64_t gbase = u * int64_t(Ng) * D;
  const float sl2 = scale * kLog2e;

  load_tile<D>(smem_u32(sK), Kg + gbase, g0, Ng, tid);
  load_tile<D>(smem_u32(sV), Vg + gbase, g0, Ng, tid);
  auto load_q = [&](int t, int st) {
    const int q0 = t * BW_TILE;
    load_tile<D>(smem_u32(sQ + st * TB), Q + base, q0, N, tid);
    load_tile<D>(smem_u32(sdO + st * TB), dO + base, q0, N, tid);
    if (tid < BW_TILE) {
      const int r = q0 + tid;
      sL[st * BW_TILE + tid] = r < N ? LSE[u * N + r] * kLog2e : INFINITY;
      sD[st * BW_TILE + tid] = r < N ? Dv[u * N + r] : 0.f;
    }
  };
  if (t0 < t1) load_q(t0, 0);
  cp_async_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;
  const int g = lane >> 2, qd = lane & 3;
  const float b0 = gt_bias_log2(g0 + warp * 16 + g, Ng, N, window);
  const float b1 = gt_bias_log2(g0 + warp * 16 + g + 8, Ng, N, window);

  for (int t = t0; t < t1; ++t) {
    const int st = (t - t0) & 1;
    if (t + 1 < t1) load_q(t + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t q_t = smem_u32(sQ + st * TB), do_t = smem_u32(sdO + st * TB);
    const float* L = sL + st * BW_TILE;
    const float* Dd = sD + st * BW_TILE;
    float p[8][4];
    {
      uint32_t ka[D / 16][4];
      load_a_rows<D>(smem_u32(sK), warp * 16, lane, ka);
      mma_rows_x_tileT<D>(ka, q_t, lane, p);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float l0 = L[n * 8 + qd * 2], l1 = L[n * 8 + qd * 2 + 1];
      p[n][0] = ex2(fmaf(p[n][0], sl2, b0 - l0));
      p[n][1] = ex2(fmaf(p[n][1], sl2, b0 - l1));
      p[n][2] = ex2(fmaf(p[n][2], sl2, b1 - l0));
      p[n][3] = ex2(fmaf(p[n][3], sl2, b1 - l1));
    }
    mma_p_x_tile<D>(p, do_t, lane, dv);
    float ds[8][4];
    {
      uint32_t va[D / 16][4];
      load_a_rows<D>(smem_u32(sV), warp * 16, lane, va);
      mma_rows_x_tileT<D>(va, do_t, lane, ds);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float d0 = Dd[n * 8 + qd * 2], d1 = Dd[n * 8 + qd * 2 + 1];
      ds[n][0] = p[n][0] * (ds[n][0] - d0);
      ds[n][1] = p[n][1] * (ds[n][1] - d1);
      ds[n][2] = p[n][2] * (ds[n][2] - d0);
      ds[n][3] = p[n][3] * (ds[n][3] - d1);
    }
    mma_p_x_tile<D>(ds, q_t, lane, dk);
    __syncthreads();
  }
  float* pk = part + (int64_t(s) * gridDim.y + u) * Ngp * D;
  float* pv = pk + part_stride;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = g0 + warp * 16 + g + 8 * h;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      *reinterpret_cast<float2*>(pk + int64_t(r) * D + n * 8 + qd * 2) =
          make_float2(dk[n][2 * h] * scale, dk[n][2 * h + 1] * scale);
      *reinterpret_cast<float2*>(pv + int64_t(r) * D + n * 8 + qd * 2) =
          make_float2(dv[n][2 * h], dv[n][2 * h + 1]);
    }
  }
}

// dKg/dVg (sum over the splits) / n_w, fp32 [2][BH][Ng][D]
__global__ void gt_bwd_reduce_kernel(const float* __restrict__ part, int64_t part_stride,
                                     int splits, int64_t BH, int Ng, int Ngp, int D, int N,
                                     int window, float* __restrict__ g_out) {
  const int64_t per = BH * Ng * D;
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= 2 * per) return;
  const int which = int(e / per);
  const int64_t r = e % per;
  const int c = int(r % D);
  const int w = int((r / D) % Ng);
  const int64_t u = r / (int64_t(D) * Ng);
  const float* src = part + which * part_stride + (u * Ngp + w) * D + c;
  float acc = 0.f;
  for (int s = 0; s < splits; ++s) acc += src[int64_t(s) * BH * Ngp * D];
  g_out[e] = acc / float(min(window, N - w * window));
}

// dK[t] += dKg[w(t)] / n_w, dV likewise (bf16 read-modify-write, 8 per thread)
__global__ void gt_bwd_unpool_kernel(const float* __restrict__ gsum, int64_t BH, int N, int Ng,
                                     int D, int window, __nv_bfloat16* __restrict__ dK,
                                     __nv_bfloat16* __restrict__ dV) {
  const int64_t per8 = BH * N * D / 8;
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= 2 * per8) return;
  const int which = int(e / per8);
  const int64_t r = (e % per8) * 8;
  const int c = int(r % D);
  const int t = int((r / D) % N);
  const int64_t u = r / (int64_t(D) * N);
  const float* src = gsum + which * BH * Ng * D + (u * Ng + t / window) * D + c;
  __nv_bfloat16* dst = (which ? dV : dK) + r;
  uint4 raw = *reinterpret_cast<const uint4*>(dst);
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
  const float4 a = *reinterpret_cast<const float4*>(src);
  const float4 b = *reinterpret_cast<const float4*>(src + 4);
  const float add[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    h[i] = __floats2bfloat162_rn(f.x + add[2 * i], f.y + add[2 * i + 1]);
  }
  *reinterpret_cast<uint4*>(dst) = raw;
}

// CTA = 64 queries: dQ_r += scale sum_w dS_rw kg_w over all global tokens
template <int D>
__global__ void __launch_bounds__(BW_THREADS) gt_bwd_dq_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Kg,
    const __nv_bfloat16* __restrict__ Vg, const __nv_bfloat16* __restrict__ dO,
    const float* __restrict__ LSE, const float* __restrict__ Dv, int N, int Ng, int window,
    float scale, __nv_bfloat16* __restrict__ dQ) {
  extern __shared__ __align__(128) char smem[];
  constexpr int TB = BW_TILE * D * 2;
  char* sQ = smem;
  char* sdO = sQ + TB;
  char* sK = sdO + TB;       // [2]
  char* sV = sK + 2 * TB;    // [2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = blockIdx.x * BW_ROWS;
  const int64_t u = blockIdx.y;
  const int64_t base = u * int64_t(N) * D;
  const int64_t gbase = u * int64_t(Ng) * D;
  const int ntiles = (Ng + BW_TILE - 1) / BW_TILE;
  const float sl2 = scale * kLog2e;

  load_tile<D>(smem_u32(sQ), Q + base, q0, N, tid);
  load_tile<D>(smem_u32(sdO), dO + base, q0, N, tid);
  auto load_kv = [&](int t, int st) {
    load_tile<D>(smem_u32(sK + st * TB), Kg + gbase, t * BW_TILE, Ng, tid);
    load_tile<D>(smem_u32(sV + st * TB), Vg + gbase, t * BW_TILE, Ng, tid);
  };
  load_kv(0, 0);
  cp_async_commit();

  const int g = lane >> 2, qd = lane & 3;
  float lse2[2], dr[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = q0 + warp * 16 + g + 8 * h;
    lse2[h] = r < N ? LSE[u * N + r] * kLog2e : 0.f;
    dr[h] = r < N ? Dv[u * N + r] : 0.f;
  }
  float dq[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) dq[n][0] = dq[n][1] = dq[n][2] = dq[n][3] = 0.f;
  uint32_t qa[D / 16][4], doa[D / 16][4];

  for (int t = 0; t < ntiles; ++t) {
    const int st = t & 1;
    if (t + 1 < ntiles) load_kv(t + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
      load_a_rows<D>(smem_u32(sQ), warp * 16, lane, qa);
      load_a_rows<D>(smem_u32(sdO), warp * 16, lane, doa);
    }
    const uint32_t k_t = smem_u32(sK + st * TB), v_t = smem_u32(sV + st * TB);
    float p[8][4], ds[8][4];
    mma_rows_x_tileT<D>(qa, k_t, lane, p);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float bw = gt_bias_log2(t * BW_TILE + n * 8 + qd * 2 + (e & 1), Ng, N, window);
        p[n][e] = ex2(fmaf(p[n][e], sl2, bw - lse2[e >> 1]));
      }
    }
    mma_rows_x_tileT<D>(doa, v_t, lane, ds);
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) ds[n][e] = p[n][e] * (ds[n][e] - dr[e >> 1]);
    mma_p_x_tile<D>(ds, k_t, lane, dq);
    __syncthreads();
  }
  // dQ (already holding the kept-key part) += scale * acc
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = q0 + warp * 16 + g + 8 * h;
    if (r < N) {
      __nv_bfloat16* row = dQ + base + int64_t(r) * D;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        __nv_bfloat162* x = reinterpret_cast<__nv_bfloat162*>(row + n * 8 + qd * 2);
        const float2 f = __bfloat1622float2(*x);
        *x = __floats2bfloat162_rn(f.x + dq[n][2 * h] * scale, f.y + dq[n][2 * h + 1] * scale);
      }
    }
  }
}

#ifdef BLADE_WITH_BASELINES
constexpr bool kBaselines = true;
#else
constexpr bool kBaselines = false;
#endif
#if defined(BLADE_WITH_BASELINES) && defined(BLADE_BWD_DKDV_MMA_SYNC)
constexpr bool kForceDkdvMma = true;
#else
constexpr bool kForceDkdvMma = false;
#endif
#if defined(BLADE_WITH_BASELINES) && defined(BLADE_BWD_DQ_MMA_SYNC)
constexpr bool kForceDqMma = true;
#else
constexpr bool kForceDqMma = false;
#endif

template <int D>
cudaError_t launch_bwd_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                         const void* o, const float* lse, const void* dout,
                         const int32_t* kv_idx, const int32_t* kv_cnt, void* dq, void* dk,
                         void* dv, char* ws, cudaStream_t stream, const GtProblem* gp) {
  const BwdWorkspace w = bwd_workspace_layout(p);
  float* Dvec = reinterpret_cast<float*>(ws + w.off_d);
  int32_t* q_idx = reinterpret_cast<int32_t*>(ws + w.off_qidx);
  int32_t* q_cnt = reinterpret_cast<int32_t*>(ws + w.off_qcnt);
  auto B = [](const void* x) { return reinterpret_cast<const __nv_bfloat16*>(x); };
  const int64_t rows = p.BH * p.N;
  bsa_bwd_dot_kernel<D><<<unsigned((rows * (D / 8) + 255) / 256), 256, 0, stream>>>(
      B(o), B(dout), rows, Dvec);
  bsa_bwd_transpose_kernel<<<dim3(unsigned((p.Nb + 31) / 32), unsigned(p.BH)), 256, 0, stream>>>(
      kv_idx, kv_cnt, p.Nb, q_idx, q_cnt);
  constexpr int TB = BW_TILE * D * 2;
  const int smem_kv = 6 * TB + 4 * BW_TILE * 4;
  const int smem_q = 6 * TB;
  dim3 grid(unsigned(2 * p.Nb), unsigned(p.BH));
  cudaError_t e;
  // dK, dV on tcgen05 (attn_bwd_tc.cu); the mma.sync kernels of this file are
  // compiled only into -DBLADE_WITH_BASELINES builds (comparison baseline, or
  // -DBLADE_BWD_DKDV_MMA_SYNC / -DBLADE_BWD_DQ_MMA_SYNC to force them)
  bool dkdv_done = false;
  if constexpr (!kForceDkdvMma) {
    e = launch_bwd_dkdv_tc(p, q, k, v, lse, dout, Dvec, q_idx, q_cnt, dk, dv, stream);
    if (e != cudaSuccess && e != cudaErrorNotSupported) return e;
    dkdv_done = e == cudaSuccess;
  }
  if (!dkdv_done) {
    if constexpr (kBaselines) {
      e = cudaFuncSetAttribute(bsa_bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_kv);
      if (e != cudaSuccess) return e;
      bsa_bwd_dkdv_kernel<D><<<grid, BW_THREADS, smem_kv, stream>>>(
          B(q), B(k), B(v), B(dout), lse, Dvec, p.N, p.Nb, p.scale, q_idx, q_cnt,
          reinterpret_cast<__nv_bfloat16*>(dk), reinterpret_cast<__nv_bfloat16*>(dv));
    } else {
      return cudaErrorNotSupported;
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (gp) {  // dK_g, dV_g partials -> sums / n_w -> spread over the windows
    const GtBwdWorkspace gw = gt_bwd_workspace_layout(p, gp->Ng);
    float* part = reinterpret_cast<float*>(ws + gw.off_part);
    float* gsum = reinterpret_cast<float*>(ws + gw.off_gsum);
    const int64_t part_stride = int64_t(gw.splits) * p.BH * gw.Ngp * D;
    bool done = false;
    if constexpr (!kForceDkdvMma) {
      e = launch_bwd_dkdv_tc(p, q, k, v, lse, dout, Dvec, nullptr, nullptr, nullptr, nullptr,
                             stream, gp, part, gw.splits);
      if (e != cudaSuccess && e != cudaErrorNotSupported) return e;
      done = e == cudaSuccess;
    }
    if (!done) {
      if constexpr (kBaselines) {
        e = cudaFuncSetAttribute(gt_bwd_dkdv_kernel<D>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
        if (e != cudaSuccess) return e;
        const int nqt = (p.N + BW_TILE - 1) / BW_TILE;
        const int tps = (nqt + gw.splits - 1) / gw.splits;
        gt_bwd_dkdv_kernel<D><<<dim3(unsigned(gw.Ngp / BW_ROWS), unsigned(p.BH),
                                     unsigned(gw.splits)),
                                BW_THREADS, smem_kv, stream>>>(
            B(q), B(gp->kg), B(gp->vg), B(dout), lse, Dvec, p.N, gp->Ng, gp->window, p.scale,
            tps, part_stride, part);
      } else {
        return cudaErrorNotSupported;
      }
    }
    const int64_t nred = 2 * p.BH * gp->Ng * D;
    gt_bwd_reduce_kernel<<<unsigned((nred + 255) / 256), 256, 0, stream>>>(
        part, part_stride, gw.splits, p.BH, gp->Ng, gw.Ngp, D, p.N, gp->window, gsum);
    const int64_t nun = 2 * p.BH * p.N * D / 8;
    gt_bwd_unpool_kernel<<<unsigned((nun + 255) / 256), 256, 0, stream>>>(
        gsum, p.BH, p.N, gp->Ng, D, gp->window, reinterpret_cast<__nv_bfloat16*>(dk),
        reinterpret_cast<__nv_bfloat16*>(dv));
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if constexpr (!kForceDqMma) {
    e = launch_bwd_dq_tc(p, q, k, v, lse, dout, Dvec, kv_idx, kv_cnt, dq, stream, gp);
    if (e != cudaErrorNotSupported) return e;
  }
  if constexpr (kBaselines) {
    e = cudaFuncSetAttribute(bsa_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_q);
    if (e != cudaSuccess) return e;
    bsa_bwd_dq_kernel<D><<<grid, BW_THREADS, smem_q, stream>>>(
        B(q), B(k), B(v), B(dout), lse, Dvec, p.N, p.Nb, p.scale, kv_idx, kv_cnt,
        reinterpret_cast<__nv_bfloat16*>(dq));
    if (gp) {  // + the global tokens' share of dQ (read-modify-write)
      e = cudaFuncSetAttribute(gt_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_q);
      if (e != cudaSuccess) return e;
      gt_bwd_dq_kernel<D><<<dim3(unsigned((p.N + BW_ROWS - 1) / BW_ROWS), unsigned(p.BH)),
                            BW_THREADS, smem_q, stream>>>(
          B(q), B(gp->kg), B(gp->vg), B(dout), lse, Dvec, p.N, gp->Ng, gp->window, p.scale,
          reinterpret_cast<__nv_bfloat16*>(dq));
    }
  } else {
    return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd(const AttnProblem& p, const void* q, const void* k, const void* v,
                            const void* o, const float* lse, const void* dout,
                            const int32_t* kv_idx, const int32_t* kv_cnt, void* dq, void* dk,
                            void* dv, char* ws, cudaStream_t stream) {
  if (p.d == 64)
    return launch_bwd_d<64>(p, q, k, v, o, lse, dout, kv_idx, kv_cnt, dq, dk, dv, ws, stream,
                            nullptr);
  if (p.d == 128)
    return launch_bwd_d<128>(p, q, k, v, o, lse, dout, kv_idx, kv_cnt, dq, dk, dv, ws, stream,
                             nullptr);
  return cudaErrorNotSupported;
}

cudaError_t launch_attn_gt_bwd(const AttnProblem& p, const GtProblem& gp, const void* q,
                               const void* k, const void* v, const void* o, const float* lse,
                               const void* dout, const int32_t* kv_idx, const int32_t* kv_cnt,
                               void* dq, void* dk, void* dv, char* ws, cudaStream_t stream) {
  if (p.d == 64)
    return launch_bwd_d<64>(p, q, k, v, o, lse, dout, kv_idx, kv_cnt, dq, dk, dv, ws, stream, &gp);
  if (p.d == 128)
    return launch_bwd_d<128>(p, q, k, v, o, lse, dout, kv_idx, kv_cnt, dq, dk, dv, ws, stream,
                             &gp);
  return cudaErrorNotSupported;
}

}  // namespace blade
