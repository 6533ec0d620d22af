// mask_kernels.cu — ASA mask generation on sm_100a (Alg. 1 l.2-10,
// Alg. 2/3 P:615-662).  Four stages, all enqueued on the caller's stream:
//
//   K-mask.1 sample_gather_kernel  A1-A3: per (unit, block, Q|K) one warp
//            draws the k_i in-block offsets (counter hash, reading R-1),
//            and copies the sampled rows, block-major, into Q_s / K_s.
//   K-mask.2 probe_kernel          A4-A6: per (unit, 64 sampled query rows)
//            S = Q_s K_s^T on tensor cores, streaming row max M / row sum l
//            over all N_k sampled keys, the per-(row, key-block) max R, then
//            P_imp[i, j] = max_{s in block i} e^{R_sj - M_s} / l_s (Alg. 3).
//   K-mask.3 select_kernel         A7-A8: one warp per (unit, q-block) row:
//            fp64 normalisation, bitonic sort (p desc, id asc), warp scan,
//            cut at tau, clamp, compaction to kv_idx / kv_cnt / mask.  Rows
//            whose decision margin is within the guard band of the fp32
//            probe error are queued for K-mask.4.
//   K-mask.4 refine_partial/final  the queued rows' P_imp recomputed in
//            fp64 on CUDA cores from the same sampled rows, then reselected
//            (reading R-14: decisions outside the 1e-6 tie band are exact).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace blade {
namespace {

constexpr int kMaxNb = 512;

// ---------------------------------------------------------------------------
// K-mask.1  sampling + gather
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) sample_gather_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, int64_t BH,
    int N, int Nb, int b, int kk, uint64_t seed, int mode, int share_qk, int64_t unit_offset,
    int32_t* __restrict__ sample_idx, __nv_bfloat16* __restrict__ qs,
    __nv_bfloat16* __restrict__ ks, int* __restrict__ counters) {
  __shared__ int offs[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = int64_t(blockIdx.x) * 8 + warp;
  if (w == 0 && lane == 0) counters[0] = 0;  // refine queue length
  if (w >= BH * Nb * 2) return;
  const int which = int(w & 1);
  const int64_t rest = w >> 1;
  const int i = int(rest % Nb);
  const int64_t u = rest / Nb;
  const int valid = min(b, N - i * b);
  const int ki = min(kk, valid);
  int32_t* sidx = sample_idx ? sample_idx + ((u * 2 + which) * Nb + i) * kk : nullptr;

  if (mode == 2) {
    for (int p = lane; p < ki; p += 32) offs[warp][p] = sidx[p];
  } else if (mode == 1) {
    for (int p = lane; p < ki; p += 32)
      offs[warp][p] = int((int64_t(2 * p + 1) * valid) / (2 * ki));
  } else {
    const int wh = share_qk ? 0 : which;
    const uint64_t key =
        smix(smix(smix(seed, uint64_t(unit_offset + u)), uint64_t(i)), uint64_t(wh));
    uint64_t r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int o = lane + 32 * e;
      r[e] = o < valid ? smix(key, uint64_t(o)) : ~0ull;
    }
    // rank of (r, o) among all valid offsets; keep rank < ki
    int rank[4] = {0, 0, 0, 0};
    for (int e2 = 0; e2 < 4; ++e2) {
      for (int src = 0; src < 32; ++src) {
        const int o2 = src + 32 * e2;
        const uint64_t r2 = __shfl_sync(0xffffffffu, r[e2], src);
        if (o2 >= valid) continue;  // warp-uniform
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int o = lane + 32 * e;
          rank[e] += (r2 < r[e] || (r2 == r[e] && o2 < o)) ? 1 : 0;
        }
      }
    }
    int base = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int o = lane + 32 * e;
      const bool sel = o < valid && rank[e] < ki;
      const unsigned bits = __ballot_sync(0xffffffffu, sel);
      if (sel) offs[warp][base + __popc(bits & ((1u << lane) - 1u))] = o;
      base += __popc(bits);
    }
  }
  __syncwarp();
  if (sidx && mode != 2)
    for (int p = lane; p < kk; p += 32) sidx[p] = p < ki ? offs[warp][p] : -1;

  // gather rows (16-byte vectors); rows p >= ki are zero
  const __nv_bfloat16* src = (which == 0 ? q : k) + (u * N + int64_t(i) * b) * D;
  __nv_bfloat16* dst = (which == 0 ? qs : ks) + (u * int64_t(Nb) * kk + int64_t(i) * kk) * D;
  constexpr int CH = D / 8;  // 16-byte chunks per row
  for (int e = lane; e < kk * CH; e += 32) {
    const int p = e / CH, c = e % CH;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (p < ki) val = *reinterpret_cast<const uint4*>(src + int64_t(offs[warp][p]) * D + c * 8);
    *reinterpret_cast<uint4*>(dst + int64_t(p) * D + c * 8) = val;
  }
}

// ---------------------------------------------------------------------------
// K-mask.2  probe (tensor cores via mma.sync m16n8k16; 4 warps x 16 rows)
// ---------------------------------------------------------------------------
constexpr int PR_ROWS = 64;   // sampled query rows per CTA
constexpr int PR_KEYS = 64;   // sampled keys per pipeline stage

template <int D>
__global__ void __launch_bounds__(128) probe_kernel(const __nv_bfloat16* __restrict__ qs,
                                                     const __nv_bfloat16* __restrict__ ks,
                                                     int N, int Nb, int b, int kk,
                                                     float scale_log2,
                                                     float* __restrict__ pimp) {
  extern __shared__ __align__(128) char smem[];
  char* sQ = smem;                                      // [64][D] bf16 swizzled
  char* sK = sQ + PR_ROWS * D * 2;                      // [2][64][D]
  float* sR = reinterpret_cast<float*>(sK + 2 * PR_KEYS * D * 2);  // [64][Nb]
  float* sM = sR + PR_ROWS * Nb;                        // [64]
  float* sL = sM + PR_ROWS;                             // [64]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t u = blockIdx.y;
  const int NK = Nb * kk;
  const int row0 = blockIdx.x * PR_ROWS;
  const __nv_bfloat16* gQ = qs + u * int64_t(NK) * D;
  const __nv_bfloat16* gK = ks + u * int64_t(NK) * D;
  constexpr int CH = D / 8;

  // Q tile
  for (int e = tid; e < PR_ROWS * CH; e += 128) {
    const int r = e / CH, c = e % CH;
    const int gr = row0 + r;
    cp_async16(smem_u32(sQ) + swz<D>(r, c), gQ + int64_t(min(gr, NK - 1)) * D + c * 8,
               gr < NK ? 16 : 0);
  }
  auto load_k = [&](int t, int stage) {
    char* dstb = sK + stage * PR_KEYS * D * 2;
    for (int e = tid; e < PR_KEYS * CH; e += 128) {
      const int r = e / CH, c = e % CH;
      const int gr = t * PR_KEYS + r;
      cp_async16(smem_u32(dstb) + swz<D>(r, c), gK + int64_t(min(gr, NK - 1)) * D + c * 8,
                 gr < NK ? 16 : 0);
    }
  };
  load_k(0, 0);
  cp_async_commit();
  for (int e = tid; e < PR_ROWS * Nb; e += 128) sR[e] = -INFINITY;

  // per-thread rows: g = lane/4 and g+8 of this warp's 16
  const int g = lane >> 2, qd = lane & 3;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qa[D / 16][4];
  const int ntiles = (NK + PR_KEYS - 1) / PR_KEYS;

  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) load_k(t + 1, (t + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int ks_ = 0; ks_ < D / 16; ++ks_) {
        const int r = warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int c = ks_ * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ) + swz<D>(r, c), qa[ks_][0], qa[ks_][1], qa[ks_][2], qa[ks_][3]);
      }
    }
    const uint32_t kb = smem_u32(sK + (t & 1) * PR_KEYS * D * 2);
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int ks_ = 0; ks_ < D / 16; ++ks_) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of n8 tiles (16 keys)
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + 8 * (lane >> 4);
        const int c = ks_ * 2 + ((lane >> 3) & 1);
        ldsm_x4(kb + swz<D>(r, c), b0, b1, b2, b3);
        mma_bf16(s[2 * np], qa[ks_], b0, b1);
        mma_bf16(s[2 * np + 1], qa[ks_], b2, b3);
      }
    }
    // scale into the log2 domain, mask invalid sampled keys
    float tmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = t * PR_KEYS + n * 8 + qd * 2 + h;
        const int jb = col / kk, rr = col - jb * kk;
        const bool ok = col < NK && rr < min(kk, min(b, N - jb * b));
        s[n][h] = ok ? s[n][h] * scale_log2 : -INFINITY;
        s[n][2 + h] = ok ? s[n][2 + h] * scale_log2 : -INFINITY;
        tmax[0] = fmaxf(tmax[0], s[n][h]);
        tmax[1] = fmaxf(tmax[1], s[n][2 + h]);
      }
    }
    // R: max over each 16-key group, folded into key block j = col / kk
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        float gm = fmaxf(fmaxf(s[2 * gi][2 * hr], s[2 * gi][2 * hr + 1]),
                         fmaxf(s[2 * gi + 1][2 * hr], s[2 * gi + 1][2 * hr + 1]));
        gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, 1));
        gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, 2));
        const int col0 = t * PR_KEYS + gi * 16;
        if (qd == 0 && col0 < NK) {
          float* rp = sR + (warp * 16 + g + 8 * hr) * Nb + col0 / kk;
          *rp = fmaxf(*rp, gm);
        }
      }
    }
    // online row max / sum (Alg. 3 l.12-15)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float tm = tmax[hr];
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 2));
      const float m_new = fmaxf(m_run[hr], tm);
      float acc = 0.f;
      if (m_new != -INFINITY) {
#pragma unroll
        for (int n = 0; n < 8; ++n) acc += ex2(s[n][2 * hr] - m_new) + ex2(s[n][2 * hr + 1] - m_new);
        l_run[hr] = l_run[hr] * ex2(m_run[hr] - m_new) + acc;
      }
      m_run[hr] = m_new;
    }
    __syncthreads();  // stage (t&1) is refilled by the next iteration's prefetch
  }
  // final row stats
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    float l = l_run[hr];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (qd == 0) {
      sM[warp * 16 + g + 8 * hr] = m_run[hr];
      sL[warp * 16 + g + 8 * hr] = l;
    }
  }
  __syncthreads();
  // max-pool over the k_i valid sampled rows of each query block (Alg. 3 l.17-19)
  const int rows_here = min(PR_ROWS, NK - row0);
  const int qb0 = row0 / kk;
  const int qb1 = (row0 + rows_here - 1) / kk;
  for (int e = tid; e < (qb1 - qb0 + 1) * Nb; e += 128) {
    const int ib = qb0 + e / Nb, j = e % Nb;
    const int ki = min(kk, min(b, N - ib * b));
    const int r_lo = max(ib * kk, row0), r_hi = min(ib * kk + ki, row0 + rows_here);
    float best = 0.f;
    for (int r = r_lo; r < r_hi; ++r) {
      const int rl = r - row0;
      best = fmaxf(best, ex2(sR[rl * Nb + j] - sM[rl]) / sL[rl]);
    }
    float* dst = pimp + (u * Nb + ib) * int64_t(Nb) + j;
    if (kk <= PR_ROWS)
      *dst = best;
    else
      atomicMax(reinterpret_cast<int*>(dst), __float_as_int(best));  // positive floats
  }
}

// ---------------------------------------------------------------------------
// K-mask.3 / K-mask.4 shared selection (one warp, fp64; Alg. 1 l.7-10)
// ---------------------------------------------------------------------------
struct SelScratch {
  double val[kMaxNb];
  int id[kMaxNb];
  uint8_t keep[kMaxNb];
};

BLADE_DEVINL bool sel_before(double va, int ia, double vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

// val[0:Nb) holds the raw P_imp row in fp64.  Writes the row's outputs and
// returns true when the decision margin is inside the guard band.
__device__ bool select_row_warp(SelScratch& sc, int Nb, double tau, int lo, int hi,
                                double guard, bool want_flag, uint8_t* mask_row,
                                int32_t* kv_idx_row, int32_t* kv_cnt_out) {
  const int lane = threadIdx.x & 31;
  int P2 = 32;
  while (P2 < Nb) P2 <<= 1;
  // l.7 normalise (Z summed lane-strided, then a fixed xor tree)
  double z = 0.0;
  for (int j = lane; j < Nb; j += 32) z += sc.val[j];
#pragma unroll
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  for (int j = lane; j < P2; j += 32) {
    sc.val[j] = j < Nb ? sc.val[j] / z : -1.0;
    sc.id[j] = j;
  }
  __syncwarp();
  // l.8 bitonic sort: p-hat descending, ties by ascending block id (R-7)
  for (int kb = 2; kb <= P2; kb <<= 1) {
    for (int jb = kb >> 1; jb > 0; jb >>= 1) {
      for (int x = lane; x < P2; x += 32) {
        const int y = x ^ jb;
        if (y > x) {
          const double vx = sc.val[x], vy = sc.val[y];
          const int ix = sc.id[x], iy = sc.id[y];
          const bool up = (x & kb) == 0;
          const bool swap = up ? sel_before(vy, iy, vx, ix) : sel_before(vx, ix, vy, iy);
          if (swap) {
            sc.val[x] = vy; sc.val[y] = vx;
            sc.id[x] = iy;  sc.id[y] = ix;
          }
        }
      }
      __syncwarp();
    }
  }
  // l.9 cumulative sums C_r (r = 1..Nb): per-lane segments + warp scan
  const int seg = P2 / 32;
  const int r0 = lane * seg;
  double part = 0.0;
  for (int r = r0; r < r0 + seg && r < Nb; ++r) part += sc.val[r];
  double incl = part;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  double run = incl - part;  // exclusive prefix
  int first = Nb + 1;
  for (int r = r0; r < r0 + seg && r < Nb; ++r) {
    run += sc.val[r];
    if (run >= tau && first > Nb) first = r + 1;
    sc.val[r] = run;  // reuse val as C_r (sorted p recoverable as differences)
  }
  // keep the sorted p-hat beside C: recompute from differences when needed
#pragma unroll
  for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  __syncwarp();
  const int m0 = first <= Nb ? first : Nb;
  const int m = min(max(m0, lo), hi);

  bool flag = false;
  if (want_flag && lane == 0) {
    auto C = [&](int r) { return r <= 0 ? 0.0 : sc.val[r - 1]; };
    auto clampi = [&](int x) { return min(max(x, lo), hi); };
    const double band = guard * tau;
    const bool cut_matters = clampi(m0 - 1) != m || clampi(m0 + 1) != m;
    if (cut_matters && (fabs(C(m0) - tau) <= band || (m0 >= 2 && fabs(C(m0 - 1) - tau) <= band)))
      flag = true;
    if (m < Nb) {
      const double pm = C(m) - C(m - 1), pn = C(m + 1) - C(m);
      if (pm - pn <= guard * pm) flag = true;
    }
  }
  flag = __shfl_sync(0xffffffffu, flag ? 1 : 0, 0) != 0;
  // l.10 mask row + compaction (kept ids ascending)
  for (int j = lane; j < Nb; j += 32) sc.keep[j] = 0;
  __syncwarp();
  for (int r = lane; r < m; r += 32) sc.keep[sc.id[r]] = 1;
  __syncwarp();
  int base = 0;
  for (int j0 = 0; j0 < Nb; j0 += 32) {
    const int j = j0 + lane;
    const bool kp = j < Nb && sc.keep[j];
    const unsigned bits = __ballot_sync(0xffffffffu, kp);
    if (kp) kv_idx_row[base + __popc(bits & ((1u << lane) - 1u))] = j;
    if (mask_row && j < Nb) mask_row[j] = kp ? 1 : 0;
    base += __popc(bits);
  }
  for (int r = m + lane; r < Nb; r += 32) kv_idx_row[r] = -1;
  if (lane == 0) *kv_cnt_out = m;
  __syncwarp();
  return flag;
}

constexpr int SEL_WARPS = 4;

__global__ void __launch_bounds__(SEL_WARPS * 32) select_kernel(
    const float* __restrict__ pimp, int64_t rows, int Nb, double tau, int lo, int hi,
    double guard, uint8_t* __restrict__ mask, int32_t* __restrict__ kv_idx,
    int32_t* __restrict__ kv_cnt, int* __restrict__ counters, int32_t* __restrict__ flags) {
  extern __shared__ __align__(128) char smem[];
  SelScratch& sc = reinterpret_cast<SelScratch*>(smem)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * SEL_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float* src = pimp + row * Nb;
  for (int j = lane; j < Nb; j += 32) sc.val[j] = double(src[j]);
  __syncwarp();
  const bool flag = select_row_warp(sc, Nb, tau, lo, hi, guard, true,
                                    mask ? mask + row * Nb : nullptr, kv_idx + row * Nb,
                                    kv_cnt + row);
  if (flag && lane == 0) {
    const int slot = atomicAdd(&counters[0], 1);
    flags[slot] = int32_t(row);
  }
}

// ---------------------------------------------------------------------------
// K-mask.4a  fp64 partial probe of queued rows: one CTA per (queued row,
// chunk of 256 sampled keys).  Thread t owns one sampled key; logits for 16
// query rows at a time are exact-product fp64 dot products.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) refine_partial_kernel(
    const __nv_bfloat16* __restrict__ qs, const __nv_bfloat16* __restrict__ ks, int N,
    int Nb, int b, int kk, double scale, int nchunks, const int* __restrict__ counters,
    const int32_t* __restrict__ flags, double* __restrict__ r64, double* __restrict__ mpart,
    double* __restrict__ lpart) {
  __shared__ double sq[16][D];
  __shared__ double sRg[16][16];   // [16-key group][s] group max
  __shared__ double sMc[16];
  __shared__ double sLw[8][16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nflag = counters[0];
  const int NK = Nb * kk;
  const int G = kk < 16 ? kk : 16;  // keys per reduction group (kk >= 16 here)
  for (int item = blockIdx.x; item < nflag * nchunks; item += gridDim.x) {
    const int f = item / nchunks, c = item % nchunks;
    const int64_t row = flags[f];
    const int64_t u = row / Nb;
    const int i = int(row % Nb);
    const int ki = min(kk, min(b, N - i * b));
    const int key = c * 256 + tid;
    const int jb = key / kk, rr = key - jb * kk;
    const bool kvalid = key < NK && rr < min(kk, min(b, N - jb * b));
    const __nv_bfloat16* kp = ks + (u * NK + min(key, NK - 1)) * int64_t(D);
    for (int sg = 0; sg < kk; sg += 16) {
      __syncthreads();
      for (int e = tid; e < 16 * D; e += 256) {
        const int s = e / D, dd = e % D;
        sq[s][dd] = double(__bfloat162float(qs[(u * NK + int64_t(i) * kk + sg + s) * D + dd]));
      }
      __syncthreads();
      double L[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) L[s] = 0.0;
      for (int d0 = 0; d0 < D; d0 += 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(kp + d0);
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
        double kv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) kv[e] = double(__bfloat162float(h[e]));
#pragma unroll
        for (int s = 0; s < 16; ++s)
#pragma unroll
          for (int e = 0; e < 8; ++e) L[s] = fma(sq[s][d0 + e], kv[e], L[s]);
      }
#pragma unroll
      for (int s = 0; s < 16; ++s) L[s] = kvalid ? L[s] * scale : -INFINITY;
      // R: max over each group of 16 consecutive keys (a key block for k=16)
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        double v = L[s];
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((lane & 15) == 0) sRg[tid >> 4][s] = v;
      }
      __syncthreads();
      // combine groups into key blocks, store R, and the chunk max per s
      const int gpb = kk / G;  // groups per key block
      const int nblk = 256 / kk;
      if (tid < 16 * nblk) {
        const int s = tid & 15, bl = tid >> 4;
        double v = -INFINITY;
        for (int gg = 0; gg < gpb; ++gg) v = fmax(v, sRg[bl * gpb + gg][s]);
        const int j = c * nblk + bl;
        if (j < Nb && sg + s < ki) r64[(int64_t(f) * kk + sg + s) * Nb + j] = v;
      }
      if (tid < 16) {
        double v = -INFINITY;
        for (int gg = 0; gg < 16; ++gg) v = fmax(v, sRg[gg][tid]);
        sMc[tid] = v;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        double e = (L[s] == -INFINITY) ? 0.0 : exp(L[s] - sMc[s]);
#pragma unroll
        for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) sLw[warp][s] = e;
      }
      __syncthreads();
      if (tid < 16 && sg + tid < ki) {
        double l = 0.0;
        for (int ww = 0; ww < 8; ++ww) l += sLw[ww][tid];
        const int64_t o = (int64_t(f) * nchunks + c) * kk + sg + tid;
        mpart[o] = sMc[tid];
        lpart[o] = l;
      }
    }
  }
}

// K-mask.4b  combine the partials of each queued row into its fp64 P_imp row
// (Alg. 3 l.14, l.17-19) and reselect it.  One CTA per queued row: threads
// own query rows for the combine, key blocks for the max-pool, then warp 0
// reruns the selection on the fp64 row.
constexpr int RF_THREADS = 256;

__global__ void __launch_bounds__(RF_THREADS) refine_final_kernel(
    int Nb, int N, int b, int kk, int nchunks, double tau, int lo, int hi,
    const int* __restrict__ counters, const int32_t* __restrict__ flags,
    const double* __restrict__ r64, const double* __restrict__ mpart,
    const double* __restrict__ lpart, float* __restrict__ pimp, uint8_t* __restrict__ mask,
    int32_t* __restrict__ kv_idx, int32_t* __restrict__ kv_cnt, int32_t* n_refined) {
  extern __shared__ __align__(128) char smem[];
  SelScratch& sc = *reinterpret_cast<SelScratch*>(smem);
  double* sMs = reinterpret_cast<double*>(smem + sizeof(SelScratch));
  double* sLs = sMs + 128;
  const int tid = threadIdx.x;
  const int nflag = counters[0];
  if (blockIdx.x == 0 && tid == 0 && n_refined) *n_refined = nflag;
  for (int f = blockIdx.x; f < nflag; f += gridDim.x) {
    const int64_t row = flags[f];
    const int i = int(row % Nb);
    const int ki = min(kk, min(b, N - i * b));
    __syncthreads();
    if (tid < ki) {
      double M = -INFINITY;
      for (int c = 0; c < nchunks; ++c) M = fmax(M, mpart[(int64_t(f) * nchunks + c) * kk + tid]);
      double l = 0.0;
      for (int c = 0; c < nchunks; ++c) {
        const int64_t o = (int64_t(f) * nchunks + c) * kk + tid;
        if (mpart[o] != -INFINITY) l += lpart[o] * exp(mpart[o] - M);
      }
      sMs[tid] = M;
      sLs[tid] = l;
    }
    __syncthreads();
    for (int j = tid; j < Nb; j += RF_THREADS) {
      double best = 0.0;
      for (int s = 0; s < ki; ++s)
        best = fmax(best, exp(r64[(int64_t(f) * kk + s) * Nb + j] - sMs[s]) / sLs[s]);
      sc.val[j] = best;
      if (pimp) pimp[row * Nb + j] = float(best);
    }
    __syncthreads();
    if (tid < 32)
      select_row_warp(sc, Nb, tau, lo, hi, 0.0, false, mask ? mask + row * Nb : nullptr,
                      kv_idx + row * Nb, kv_cnt + row);
  }
}

template <int D>
cudaError_t launch_mask_d(const MaskProblem& p, const void* q, const void* k, uint8_t* mask,
                          int32_t* kv_idx, int32_t* kv_cnt, float* p_imp_out,
                          int32_t* sample_idx, int32_t* n_refined, char* ws,
                          cudaStream_t stream) {
  const MaskWorkspace w = mask_workspace_layout(p);
  auto* qs = reinterpret_cast<__nv_bfloat16*>(ws + w.off_qs);
  auto* ks = reinterpret_cast<__nv_bfloat16*>(ws + w.off_ks);
  float* pimp = p_imp_out ? p_imp_out : reinterpret_cast<float*>(ws + w.off_pimp);
  int* counters = reinterpret_cast<int*>(ws + w.off_counters);
  int32_t* flags = reinterpret_cast<int32_t*>(ws + w.off_flags);
  double* r64 = reinterpret_cast<double*>(ws + w.off_r64);
  double* mpart = reinterpret_cast<double*>(ws + w.off_mpart);
  double* lpart = reinterpret_cast<double*>(ws + w.off_lpart);
  const int64_t rows = p.BH * p.Nb;

  {  // K-mask.1
    const int64_t warps = p.BH * p.Nb * 2;
    sample_gather_kernel<D><<<unsigned((warps + 7) / 8), 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
        p.BH, p.N, p.Nb, p.b, p.kk, p.seed, p.mode, p.share_qk, p.unit_offset, sample_idx, qs,
        ks, counters);
  }
  if (probe_tc_supported(D, p.kk, p.Nb)) {  // K-mask.2 on tcgen05 (k in {16, 32}, N_b <= 256)
    cudaError_t e = launch_probe_tc(p.BH, p.N, p.Nb, p.b, p.kk, D, p.scale, qs, ks, pimp, stream);
    if (e != cudaSuccess) return e;
  } else {
  if (p.kk > PR_ROWS) {
    cudaError_t e = cudaMemsetAsync(pimp, 0, size_t(rows) * p.Nb * 4, stream);
    if (e != cudaSuccess) return e;
  }
  {  // K-mask.2 (mma.sync fallback for other k / longer sequences)
    const size_t smem = size_t(PR_ROWS) * D * 2 + 2 * PR_KEYS * D * 2 +
                        size_t(PR_ROWS) * p.Nb * 4 + 2 * PR_ROWS * 4;
    cudaError_t e = cudaFuncSetAttribute(probe_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned((p.Nb * p.kk + PR_ROWS - 1) / PR_ROWS), unsigned(p.BH));
    probe_kernel<D><<<grid, 128, smem, stream>>>(qs, ks, p.N, p.Nb, p.b, p.kk,
                                                 p.scale * kLog2e, pimp);
  }
  }
  const size_t sel_smem = SEL_WARPS * sizeof(SelScratch);
  {  // K-mask.3
    cudaError_t e = cudaFuncSetAttribute(select_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sel_smem));
    if (e != cudaSuccess) return e;
    select_kernel<<<unsigned((rows + SEL_WARPS - 1) / SEL_WARPS), SEL_WARPS * 32, sel_smem,
                    stream>>>(pimp, rows, p.Nb, p.tau, p.lo, p.hi, p.guard, mask, kv_idx, kv_cnt,
                              counters, flags);
  }
  {  // K-mask.4 (persistent grids; the queue length is read on the device)
    refine_partial_kernel<D><<<148 * 4, 256, 0, stream>>>(
        qs, ks, p.N, p.Nb, p.b, p.kk, double(p.scale), w.nchunks, counters, flags, r64, mpart,
        lpart);
    const size_t fsmem = sizeof(SelScratch) + 256 * sizeof(double);
    refine_final_kernel<<<148, RF_THREADS, fsmem, stream>>>(
        p.Nb, p.N, p.b, p.kk, w.nchunks, p.tau, p.lo, p.hi, counters, flags, r64, mpart, lpart,
        p_imp_out, mask, kv_idx, kv_cnt, n_refined);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mask(const MaskProblem& p, const void* q, const void* k, uint8_t* mask,
                        int32_t* kv_idx, int32_t* kv_cnt, float* p_imp_out,
                        int32_t* sample_idx, int32_t* n_refined, char* ws,
                        cudaStream_t stream) {
  if (p.d == 64)
    return launch_mask_d<64>(p, q, k, mask, kv_idx, kv_cnt, p_imp_out, sample_idx, n_refined,
                             ws, stream);
  if (p.d == 128)
    return launch_mask_d<128>(p, q, k, mask, kv_idx, kv_cnt, p_imp_out, sample_idx, n_refined,
                              ws, stream);
  return cudaErrorInvalidValue;
}

}  // namespace blade
