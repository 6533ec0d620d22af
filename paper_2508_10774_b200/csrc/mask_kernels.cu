// mask_kernels.cu — ASA mask generation on sm_100a (Alg. 1 l.2-10,
// Alg. 2/3 P:615-662).  Four stages, all enqueued on the caller's stream:
//
//   K-mask.1 sample_gather_kernel  A1-A3: per (unit, block, Q|K) one warp
//            draws the k_i in-block offsets (counter hash, reading R-1),
//            and copies the sampled rows, block-major, into Q_s / K_s.
//   K-mask.2 probe2_kernel (probe2.cu) A4-A6: per (unit, 128 sampled query
//            rows) S = Q_s K_s^T on the tcgen05 tensor cores, streaming row
//            max M / row sum l over all N_k sampled keys, the per-(row,
//            key-block) max R in TMEM, then P_imp[i, j] = max_{s in block i}
//            e^{R_sj - M_s} / l_s (Alg. 3).
//   K-mask.3 selection (select.cuh)    A7-A8: one warp per (unit, q-block)
//            row: fp64 normalisation, register bitonic sort (p desc, id
//            asc), warp scan, cut at tau, clamp, compaction to kv_idx /
//            kv_cnt / mask (select_kernel).  Rows whose
//            decision margin is inside the guard band of the fp32 probe
//            error are queued for K-mask.4.
//   K-mask.4 refine_kernel         the queued rows' P_imp recomputed in fp64
//            on CUDA cores from the same sampled rows, then reselected
//            (reading R-14: decisions outside the 1e-6 tie band are exact).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdio.h>

#include "common.cuh"
#include "internal.h"
#include "select.cuh"

namespace blade {
namespace {

constexpr int kMaxNb = 512;

// Ascending bitonic sort of P = 32 E (hash, offset) pairs across a warp, E
// per lane at positions x = E lane + e (distances < E in registers, larger
// ones by shuffles); ties of the hash broken by the offset (reading R-1).
template <int E>
BLADE_DEVINL void bitonic_pairs(uint64_t (&r)[E], int (&o)[E], int lane) {
  auto less = [](uint64_t ra, int oa, uint64_t rb, int ob) {
    return ra < rb || (ra == rb && oa < ob);
  };
#pragma unroll
  for (int kb = 2; kb <= 32 * E; kb <<= 1) {
#pragma unroll
    for (int jb = kb >> 1; jb > 0; jb >>= 1) {
      if (jb < E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int pe = e ^ jb;
          if (pe > e) {
            const bool up = ((lane * E + e) & kb) == 0;
            const bool sw = up ? less(r[pe], o[pe], r[e], o[e]) : less(r[e], o[e], r[pe], o[pe]);
            if (sw) {
              const uint64_t tr = r[e]; r[e] = r[pe]; r[pe] = tr;
              const int to = o[e]; o[e] = o[pe]; o[pe] = to;
            }
          }
        }
      } else {
        const int lm = jb / E;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t orr = __shfl_xor_sync(0xffffffffu, r[e], lm);
          const int oo = __shfl_xor_sync(0xffffffffu, o[e], lm);
          const bool up = ((lane * E + e) & kb) == 0;
          const bool mine_first = less(r[e], o[e], orr, oo);
          if (mine_first != (lower == up)) {
            r[e] = orr;
            o[e] = oo;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K-mask.1  sampling + gather
// ---------------------------------------------------------------------------
// One warp per (unit, block, Q|K).  Every shuffle runs in warp-converged
// code (no data-dependent branch around a collective: the compiler would wrap
// each in a WARPSYNC / ENDCOLLECTIVE sequence); whole warps past the end only
// skip their memory accesses.
//
// kSmallK (k <= 16): only offsets whose hash lies below a threshold T can be
// among the k_i smallest when at least k_i hashes do; with T / 2^64 = 40 /
// valid about 40 candidates survive, sorted 2 per lane instead of all 128.
// Exact: the k_i smallest (hash, offset) pairs of all offsets are the k_i
// smallest of the candidates whenever there are >= k_i of them.  Otherwise
// (fewer than k_i, or more than 64 candidates: ~1e-6 per block) lane 0 selects
// serially from all offsets.  Larger k: the full 128-pair sort.
template <int D, bool kSmallK>
__global__ void __launch_bounds__(256) sample_gather_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, int64_t BH,
    int N, int Nb, int b, int kk, uint64_t seed, int mode, int share_qk, int64_t unit_offset,
    int32_t* __restrict__ sample_idx, __nv_bfloat16* __restrict__ qs,
    __nv_bfloat16* __restrict__ ks, int* __restrict__ counters, int* __restrict__ attn_work) {
  __shared__ int offs[8][128];
  __shared__ uint32_t sel_bits[8][4];
  __shared__ uint64_t cand_h[8][64];
  __shared__ int cand_o[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = int64_t(blockIdx.x) * 8 + warp;
  // K-mask.2 (probe2_kernel, a programmatic dependent) may be scheduled now;
  // its producer waits for this grid's completion before reading Q_s / K_s
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (w == 0 && lane == 0) {
    counters[0] = 0;                     // refine queue length
    if (attn_work) attn_work[0] = 0;     // the persistent attention's item counter
  }
  const bool active = w < BH * Nb * 2;
  const int which = int(w & 1);
  const int64_t rest = w >> 1;
  const int i = int(rest % Nb);
  const int64_t u = active ? rest / Nb : 0;
  const int valid = min(b, N - i * b);
  const int ki = min(kk, valid);
  int32_t* sidx = sample_idx && active ? sample_idx + ((u * 2 + which) * Nb + i) * kk : nullptr;

  if (mode == 2) {
    if (active)
      for (int p = lane; p < ki; p += 32) offs[warp][p] = sidx[p];
  } else if (mode == 1) {
    for (int p = lane; p < ki; p += 32)
      offs[warp][p] = int((int64_t(2 * p + 1) * valid) / (2 * ki));
  } else {
    const int wh = share_qk ? 0 : which;
    const uint64_t key =
        smix(smix(smix(seed, uint64_t(unit_offset + u)), uint64_t(i)), uint64_t(wh));
    if (lane < 4) sel_bits[warp][lane] = 0u;
    __syncwarp();
    if constexpr (kSmallK) {
      const uint64_t T = valid <= 40 ? ~0ull
                                     : uint64_t(40.0 / double(valid) * 18446744073709551616.0);
      uint64_t h[4];
      int cnt = 0, pos[4];
      bool c[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int o = lane + 32 * e;
        h[e] = o < valid ? smix(key, uint64_t(o)) : ~0ull;
        c[e] = o < valid && h[e] <= T;
        const uint32_t bal = __ballot_sync(0xffffffffu, c[e]);
        pos[e] = cnt + __popc(bal & ((1u << lane) - 1u));
        cnt += __popc(bal);
      }
      const bool fast = cnt >= ki && cnt <= 64;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c[e] && pos[e] < 64) {
          cand_h[warp][pos[e]] = h[e];
          cand_o[warp][pos[e]] = lane + 32 * e;
        }
      __syncwarp();
      uint64_t r[2];
      int o[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int x = lane * 2 + e;
        r[e] = x < cnt ? cand_h[warp][x] : ~0ull;
        o[e] = x < cnt ? cand_o[warp][x] : 1024 + x;  // pads sort last
      }
      bitonic_pairs<2>(r, o, lane);  // unconditional: converged shuffles
      if (fast) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (lane * 2 + e < ki) atomicOr(&sel_bits[warp][o[e] >> 5], 1u << (o[e] & 31));
      } else if (lane == 0) {  // rare: k_i smallest of all offsets, serially
        uint64_t last_h = 0;
        int last_o = -1;
        for (int n = 0; n < ki; ++n) {
          uint64_t bh = ~0ull;
          int bo = 1 << 30;
          for (int oo = 0; oo < valid; ++oo) {
            const uint64_t hh = smix(key, uint64_t(oo));
            const bool after = hh > last_h || (hh == last_h && oo > last_o);
            if (after && (hh < bh || (hh == bh && oo < bo))) {
              bh = hh;
              bo = oo;
            }
          }
          sel_bits[warp][bo >> 5] |= 1u << (bo & 31);
          last_h = bh;
          last_o = bo;
        }
      }
    } else {
      // bitonic sort of the 128 (hash, offset) pairs, ascending; 4 per lane at
      // positions x = 4*lane + e; invalid offsets carry the maximal hash and
      // their (larger) offset, so they sort after every valid one
      uint64_t r[4];
      int o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o[e] = lane * 4 + e;
        r[e] = o[e] < valid ? smix(key, uint64_t(o[e])) : ~0ull;
      }
      bitonic_pairs<4>(r, o, lane);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (lane * 4 + e < ki) atomicOr(&sel_bits[warp][o[e] >> 5], 1u << (o[e] & 31));
    }
    // the k_i selected offsets, ascending: per 32-offset word, each lane
    // places its offset at the word's running count
    __syncwarp();
    int base = 0;
#pragma unroll
    for (int ww = 0; ww < 4; ++ww) {
      const uint32_t bits = sel_bits[warp][ww];
      if ((bits >> lane) & 1u) offs[warp][base + __popc(bits & ((1u << lane) - 1u))] = ww * 32 + lane;
      base += __popc(bits);
    }
  }
  if (!active) return;
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
// K-mask.3  selection, one warp per (unit, q-block) row.
// ---------------------------------------------------------------------------
constexpr int SEL_WARPS = 4;
// 6 CTAs per SM (<= 85 registers): the Wan layer's 768 CTAs fit one wave
// (at 96 registers, 5 per SM, 1.04 waves)
#ifndef BLADE_SEL_MIN_BLOCKS
#define BLADE_SEL_MIN_BLOCKS 6
#endif

__global__ void __launch_bounds__(SEL_WARPS * 32, BLADE_SEL_MIN_BLOCKS) select_kernel(
    const float* __restrict__ pimp, int64_t rows, int Nb, double tau, int lo, int hi,
    double guard, uint8_t* __restrict__ mask, int32_t* __restrict__ kv_idx,
    int32_t* __restrict__ kv_cnt, int* __restrict__ counters, int32_t* __restrict__ flags,
    int* __restrict__ done, int neg_flagged) {
  __shared__ uint32_t keep_bits[SEL_WARPS][16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * SEL_WARPS + warp;
  // a programmatic dependent of K-mask.2: P_imp (and the zeroed refine queue
  // counter of K-mask.1, complete before K-mask.2 began) visible past this
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (row >= rows) return;
  const bool flag = select_row(pimp + row * Nb, Nb, tau, lo, hi, guard, true,
                               mask ? mask + row * Nb : nullptr, kv_idx + row * Nb, kv_cnt + row,
                               keep_bits[warp]);
  if (flag && lane == 0) {
    const int slot = atomicAdd(&counters[0], 1);
    flags[slot] = int32_t(row);
    done[slot] = 0;
    // fused forward (blade_asa_fwd): mark the row's count provisional (-1 - m)
    // until K-mask.4 writes the final one; attention CTAs of such rows wait
    if (neg_flagged) kv_cnt[row] = -1 - kv_cnt[row];
  }
}

// ---------------------------------------------------------------------------
// K-mask.4  fp64 recomputation of queued rows.  One CTA (128 threads) per
// (queued row, chunk of 128 sampled keys): thread t owns one sampled key and
// forms the exact-product fp64 logits against the row's k_i sampled queries,
// 16 at a time; per chunk it leaves R (per key block), the chunk max M_c and
// l_c = sum exp(L - M_c).  The CTA that finishes a row's last chunk combines
// them (Alg. 3 l.14: M = max M_c, l = sum l_c e^{M_c - M}), forms the fp64
// P_imp row (l.17-19) and reselects it.  The reselection sorts the fp64
// values rounded to fp32 (relative error 6e-8, far inside the 1e-6 tie band).
// ---------------------------------------------------------------------------
constexpr int RF_THREADS = 128;

#ifdef BLADE_RF_TIMING  // timing experiment: globaltimer stamps (ns) of the refine phases
__device__ unsigned long long g_rf[8];  // 0 min start, 1 max end, 2 max item end, 3 sum combine,
                                        // 4 sum select, 5 rows, 6 max item duration
BLADE_DEVINL unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// Alg. 1 l.7-10 for one refined row by a CTA of NT threads, in
// fp64: Z = sum_j P_imp (l.7); a bitonic sort of (p~, id) in shared memory,
// descending with ties by ascending id (l.8, reading R-7); C_m by a block scan
// of the sorted values, m0 = first m with C_m >= tau (N_b if none or tau >= 1,
// reading R-4), m = clamp(m0, lo, hi) (l.9); kept ids compacted ascending
// (l.10).  Summation orders differ from the oracle's sequential sums only by
// fp64 rounding (~1e-16), far inside the 1e-6 tie band.  scratch: >= kMaxNb
// (8 + 4) + NT 8 + 64 bytes of shared memory.
template <int NT>
__device__ void cta_select_f64(const double* p, int Nb, double tau, int lo, int hi,
                               uint8_t* mask_row, int32_t* kv_idx_row, int32_t* kv_cnt_out,
                               char* scratch) {
  double* sv = reinterpret_cast<double*>(scratch);          // [kMaxNb] sort values
  int* si = reinterpret_cast<int*>(sv + kMaxNb);            // [kMaxNb] sort ids
  double* red = reinterpret_cast<double*>(si + kMaxNb);     // [NT]
  uint32_t* bits = reinterpret_cast<uint32_t*>(red + NT);   // [16]
  const int tid = threadIdx.x;
  int P2 = 1;
  while (P2 < Nb) P2 <<= 1;
  double z = 0.0;
  for (int j = tid; j < Nb; j += NT) z += p[j];
  red[tid] = z;
  if (tid < 16) bits[tid] = 0u;
  __syncthreads();
  for (int o = NT / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  const double Z = red[0];
  for (int j = tid; j < P2; j += NT) {
    sv[j] = j < Nb ? p[j] / Z : -1.0;  // pads sort last
    si[j] = j;
  }
  __syncthreads();
  for (int kb = 2; kb <= P2; kb <<= 1) {
    for (int jb = kb >> 1; jb > 0; jb >>= 1) {
      for (int x = tid; x < P2; x += NT) {
        const int y = x ^ jb;
        if (y > x) {
          const double vx = sv[x], vy = sv[y];
          const int ix = si[x], iy = si[y];
          const bool x_first = vx > vy || (vx == vy && ix < iy);
          if (x_first != ((x & kb) == 0)) {
            sv[x] = vy; sv[y] = vx;
            si[x] = iy; si[y] = ix;
          }
        }
      }
      __syncthreads();
    }
  }
  // C_m: thread t owns sorted positions [t PER, (t+1) PER)
  constexpr int PER = kMaxNb / NT;
  double run = 0.0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int x = tid * PER + e;
    run += x < Nb ? sv[x] : 0.0;
  }
  __syncthreads();
  red[tid] = run;
  __syncthreads();
  for (int o = 1; o < NT; o <<= 1) {  // inclusive Hillis-Steele scan of the thread totals
    const double add = tid >= o ? red[tid - o] : 0.0;
    __syncthreads();
    red[tid] += add;
    __syncthreads();
  }
  double c = tid > 0 ? red[tid - 1] : 0.0;
  int first = Nb + 1;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int x = tid * PER + e;
    if (x < Nb) {
      c += sv[x];
      if (c >= tau && first > Nb) first = x + 1;
    }
  }
  __syncthreads();
  int* cnt = reinterpret_cast<int*>(red);
  cnt[tid] = first;
  __syncthreads();
  for (int o = NT / 2; o > 0; o >>= 1) {
    if (tid < o) cnt[tid] = min(cnt[tid], cnt[tid + o]);
    __syncthreads();
  }
  const int m0 = (tau >= 1.0 || cnt[0] > Nb) ? Nb : cnt[0];
  const int m = min(max(m0, lo), hi);
  for (int x = tid; x < m; x += NT) atomicOr(&bits[si[x] >> 5], 1u << (si[x] & 31));
  __syncthreads();
  if (tid < 32) {  // ascending compaction through the bitmap (one warp, converged)
    const int nwords = (Nb + 31) >> 5;
    const uint32_t myw = tid < nwords ? bits[tid] : 0u;
    const int cw = __popc(myw);
    int pre = cw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, o);
      if (tid >= o) pre += y;
    }
    pre -= cw;
    uint32_t wv = myw;
    while (wv) {
      const int bb = __ffs(wv) - 1;
      wv &= wv - 1;
      kv_idx_row[pre++] = tid * 32 + bb;
    }
  }
  for (int x = m + tid; x < Nb; x += NT) kv_idx_row[x] = -1;
  if (mask_row)
    for (int j = tid; j < Nb; j += NT) mask_row[j] = (bits[j >> 5] >> (j & 31)) & 1u;
  if (tid == 0) *kv_cnt_out = m;
}

// K-mask.4 on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64).  One CTA
// (4 warps) per (queued row, chunk of 128 sampled keys), persistent grid.
// The chunk's 128 key rows (bf16) are staged in shared memory once; warp w
// owns keys [32 w, 32 w + 32) of the chunk (four n-tiles of 8) against 16 of
// the block's sampled query rows at a time (two m-tiles of 8).  The d axis is
// permuted so that lane l of a fragment walks d = (l & 3) (D/4) + kappa,
// kappa = 0 .. D/4 - 1: every lane's operands for all D/4 k-steps are one
// contiguous run of its row (four 16-byte loads per row), converted to fp64
// on the fly (exact).  The sum over d is the same dot product as the oracle's
// up to fp64 rounding order.  The accumulators give the chunk's exact-product
// fp64 logits; per chunk the CTA leaves R (per key block), the chunk max M_c
// and l_c = sum exp(L - M_c).  The CTA that finishes a row's last chunk
// combines them (Alg. 3 l.14: M = max M_c, l = sum l_c e^{M_c - M}), forms
// the fp64 P_imp row (l.17-19) and reselects it.  The reselection works on
// the fp64 values (the whole CTA, cta_select_f64).
constexpr int RF_CK = 128;  // sampled keys per work item

BLADE_DEVINL void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// bf16 -> fp64 with integer ops (ALU pipe; the F2F.F64 conversion runs on the
// narrow XU pipe and bound this kernel): exponent rebias 127 -> 1023, the 7
// mantissa bits on top of the 52; exact for every finite normal bf16, zero
// and bf16 subnormals (|x| < 1.2e-38, never in a logit that matters) -> +-0.
BLADE_DEVINL double bf16bits_f64(uint32_t h16) {
  const uint32_t t = h16 & 0x7fffu;
  const uint32_t hi = (t >= 0x80u ? t * 8192u + 0x38000000u : 0u) | ((h16 & 0x8000u) << 16);
  return __hiloint2double(int(hi), 0);
}
BLADE_DEVINL double bf16_lo_f64(uint32_t w) { return bf16bits_f64(w & 0xffffu); }
BLADE_DEVINL double bf16_hi_f64(uint32_t w) { return bf16bits_f64(w >> 16); }

template <int D>
#ifndef BLADE_RF_MINB
#define BLADE_RF_MINB 5  // refine CTAs per SM: tau 0.95 (129 rows) 0.365 ms mask vs 0.452 at 3, 0.386 at 4
#endif
__global__ void __launch_bounds__(RF_THREADS, BLADE_RF_MINB) refine_kernel(
    const __nv_bfloat16* __restrict__ qs, const __nv_bfloat16* __restrict__ ks, int N, int Nb,
    int b, int kk, double scale, int nchunks, double tau, int lo, int hi,
    const int* __restrict__ counters, const int32_t* __restrict__ flags, int* __restrict__ done,
    double* __restrict__ r64, double* __restrict__ mpart, double* __restrict__ lpart,
    float* __restrict__ pimp_out, uint8_t* __restrict__ mask, int32_t* __restrict__ kv_idx,
    int32_t* __restrict__ kv_cnt, int32_t* __restrict__ n_refined) {
  constexpr int RS = D * 2 + 16;   // smem row stride (bytes): conflict-free 16-byte reads
  constexpr int DQ = D / 4;        // k-steps; each lane's contiguous d run
  constexpr int NV = DQ / 8;       // 16-byte vectors per lane and row
  // the staged key rows; the last CTA of a row reuses the space for the
  // combine (P_imp row, sorted row, ranks) once every warp is past the MMA
  __shared__ __align__(16) char sK[RF_CK * RS];
  static_assert(RF_CK * RS >= kMaxNb * 8 + kMaxNb * 12 + RF_THREADS * 8 + 64,
                "combine scratch must fit in sK");
  double* sRow = reinterpret_cast<double*>(sK);    // refined P_imp row, then p~ (l.7)
  __shared__ __align__(16) char sQ[16 * RS];
  __shared__ double sRg[8][16];    // [16-key group][s] group max / combine scratch
  __shared__ double sW[4][16];     // per-warp partials
  __shared__ double sMc[16];
  __shared__ double sMs[128];
  __shared__ int last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g8 = lane >> 2, kl = lane & 3;
  // a programmatically dependent attention launch (blade_asa_fwd) may start
  // now: its CTAs of refined rows wait in griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int nflag = counters[0];
  if (blockIdx.x == 0 && tid == 0 && n_refined) *n_refined = nflag;
  const int NK = Nb * kk;
#ifdef BLADE_RF_TIMING
  const unsigned long long t_cta = gtime();
  if (tid == 0) atomicMin(&g_rf[0], t_cta);
#endif
  for (int item = blockIdx.x; item < nflag * nchunks; item += gridDim.x) {
#ifdef BLADE_RF_TIMING
    const unsigned long long t_item = gtime();
#endif
    const int f = item / nchunks, c = item % nchunks;
    const int64_t row = flags[f];
    const int64_t u = row / Nb;
    const int i = int(row % Nb);
    const int ki = min(kk, min(b, N - i * b));
    __syncthreads();  // the previous item's smem reads are done
    // stage the chunk's key rows (zero past N_k): asynchronous 16-byte copies,
    // all in flight at once
    for (int e = tid; e < RF_CK * (D / 8); e += RF_THREADS) {
      const int t = e / (D / 8), v8 = e % (D / 8);
      const int key = c * RF_CK + t;
      const bool ok = key < NK;
      cp_async16(smem_u32(sK + t * RS + v8 * 16),
                 ks + (u * NK + (ok ? key : 0)) * int64_t(D) + v8 * 8, ok ? 16 : 0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // validity of this lane's keys (2 per n-tile): padded samples of a ragged
    // last block and slots past N_k get -inf
    bool kv[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = c * RF_CK + warp * 32 + nt * 8 + 2 * kl + e;
        const int jb = key / kk, rr = key - jb * kk;
        kv[nt][e] = key < NK && rr < min(kk, min(b, N - jb * b));
      }
    for (int sg = 0; sg < kk; sg += 16) {
      __syncthreads();
      for (int e = tid; e < 16 * (D / 8); e += RF_THREADS) {
        const int s = e / (D / 8), v8 = e % (D / 8);
        cp_async16(smem_u32(sQ + s * RS + v8 * 16),
                   qs + (u * NK + int64_t(i) * kk + sg + s) * D + v8 * 8, 16);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      double acc[2][4][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      // fragments: query row mt 8 + g8, key row 32 warp + 8 nt + g8, each lane
      // walking its d run [kl DQ, kl DQ + DQ) one 16-byte vector at a time
      const char* qrow = sQ + g8 * RS + kl * DQ * 2;
      const char* krow = sK + (warp * 32 + g8) * RS + kl * DQ * 2;
#pragma unroll 1
      for (int v = 0; v < NV; ++v) {
        uint4 qf[2], kf[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
          qf[mt] = *reinterpret_cast<const uint4*>(qrow + mt * 8 * RS + v * 16);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          kf[nt] = *reinterpret_cast<const uint4*>(krow + nt * 8 * RS + v * 16);
#pragma unroll
        for (int w = 0; w < 4; ++w) {  // 32-bit word w of the vector: kappa 8v+2w, +1
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double a[2], bb[4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              const uint32_t x = reinterpret_cast<const uint32_t*>(&qf[mt])[w];
              a[mt] = h ? bf16_hi_f64(x) : bf16_lo_f64(x);
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const uint32_t x = reinterpret_cast<const uint32_t*>(&kf[nt])[w];
              bb[nt] = h ? bf16_hi_f64(x) : bf16_lo_f64(x);
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) dmma_m8n8k4(acc[mt][nt], a[mt], bb[nt]);
          }
        }
      }
      // logits (Alg. 1 l.4: L = Q_s K_s^T * scale), -inf on invalid keys;
      // per-(row, 16-key group) max: groups 2 warp + (nt >> 1)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int gh = 0; gh < 2; ++gh) {
          double v = -INFINITY;
#pragma unroll
          for (int nt = 2 * gh; nt < 2 * gh + 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              acc[mt][nt][e] = kv[nt][e] ? acc[mt][nt][e] * scale : -INFINITY;
              v = fmax(v, acc[mt][nt][e]);
            }
          v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 1));
          v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 2));
          if (kl == 0) sRg[warp * 2 + gh][mt * 8 + g8] = v;
        }
      }
      __syncthreads();
      const int gpb = kk / 16;        // 16-key groups per key block
      const int nblk = RF_CK / kk;    // key blocks per chunk (kk <= RF_CK)
      if (tid < 16 * nblk) {
        const int q = tid & 15, bl = tid >> 4;
        double v = -INFINITY;
        for (int gg = 0; gg < gpb; ++gg) v = fmax(v, sRg[bl * gpb + gg][q]);
        const int j = c * nblk + bl;
        if (j < Nb && sg + q < ki) r64[(int64_t(f) * kk + sg + q) * Nb + j] = v;
      }
      if (tid < 16) {
        double v = -INFINITY;
#pragma unroll
        for (int gg = 0; gg < 8; ++gg) v = fmax(v, sRg[gg][tid]);
        sMc[tid] = v;
      }
      __syncthreads();
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double mc = sMc[mt * 8 + g8];
        double e = 0.0;
        if (mc != -INFINITY) {
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int x = 0; x < 2; ++x)
              if (acc[mt][nt][x] != -INFINITY) e += exp(acc[mt][nt][x] - mc);
        }
        e += __shfl_xor_sync(0xffffffffu, e, 1);
        e += __shfl_xor_sync(0xffffffffu, e, 2);
        if (kl == 0) sW[warp][mt * 8 + g8] = e;
      }
      __syncthreads();
      if (tid < 16 && sg + tid < ki) {
        const double l = sW[0][tid] + sW[1][tid] + sW[2][tid] + sW[3][tid];
        const int64_t o = (int64_t(f) * nchunks + c) * kk + sg + tid;
        mpart[o] = sMc[tid];
        lpart[o] = l;
      }
    }
    // ---- last chunk of this row: combine and reselect ----
#ifdef BLADE_RF_TIMING
    if (tid == 0) {
      const unsigned long long te = gtime();
      atomicMax(&g_rf[2], te);
      atomicMax(&g_rf[6], te - t_item);
    }
    const unsigned long long t_comb = gtime();
#endif
    __threadfence();
    __syncthreads();
    if (tid == 0) last = (atomicAdd(&done[f], 1) == nchunks - 1);
    __syncthreads();
    if (!last) continue;
    __threadfence();
    // l.14 combine in one pass, spread over all threads: (query row q, chunk
    // stripe z) merges its chunks' (M_c, l_c) online, then the 8 stripes of a
    // row are merged through shared memory
    for (int qg = 0; qg < ki; qg += 16) {  // query rows in groups of 16
      const int q = qg + (tid & 15), z = tid >> 4;  // 16 rows x 8 stripes
      double M = -INFINITY, l = 0.0;
      for (int cc = z; cc < nchunks; cc += 8) {
        const bool ok = q < ki;
        const int64_t o = (int64_t(f) * nchunks + cc) * kk + (ok ? q : 0);
        const double mc = ok ? __ldcg(&mpart[o]) : -INFINITY;
        const double lc = ok ? __ldcg(&lpart[o]) : 0.0;
        if (mc == -INFINITY) continue;
        if (mc > M) {
          l = l * exp(M - mc) + lc;  // exp(-inf) = 0 on the first chunk
          M = mc;
        } else {
          l += lc * exp(mc - M);
        }
      }
      sRg[z][q - qg] = M;
      __syncthreads();
      double Mt = sRg[0][q - qg];
#pragma unroll
      for (int zz = 1; zz < 8; ++zz) Mt = fmax(Mt, sRg[zz][q - qg]);
      __syncthreads();
      sRg[z][q - qg] = M == -INFINITY ? 0.0 : l * exp(M - Mt);
      __syncthreads();
      if (z == 0 && q < ki) {
        double lt = 0.0;
#pragma unroll
        for (int zz = 0; zz < 8; ++zz) lt += sRg[zz][q - qg];
        sMs[q] = Mt + log(lt);  // P~ = e^{L - M} / l = e^{L - (M + ln l)}
      }
      __syncthreads();
    }
    // l.17-19: P_imp[j] = max_s e^{R_sj - M_s} / l_s = e^{max_s (R_sj - M_s - ln l_s)}
    for (int j = tid; j < Nb; j += RF_THREADS) {
      double rv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)
        rv[q] = q < ki ? __ldcg(&r64[(int64_t(f) * kk + q) * Nb + j]) : -INFINITY;
      double arg = -INFINITY;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q < ki) arg = fmax(arg, rv[q] - sMs[q]);
      for (int q = 16; q < ki; ++q)  // k > 16 only
        arg = fmax(arg, __ldcg(&r64[(int64_t(f) * kk + q) * Nb + j]) - sMs[q]);
      const double best = exp(arg);
      sRow[j] = best;
      if (pimp_out) pimp_out[row * Nb + j] = float(best);
    }
    __syncthreads();
#ifdef BLADE_RF_TIMING
    const unsigned long long t_sel = gtime();
#endif
    // l.7-10 in fp64 by the whole CTA (shared-memory bitonic sort; a warp-level
    // register sort of the fp64 row measured slower: 38-45 vs 14 us per row)
    cta_select_f64<RF_THREADS>(sRow, Nb, tau, lo, hi, mask ? mask + row * Nb : nullptr,
                               kv_idx + row * Nb, kv_cnt + row,
                               reinterpret_cast<char*>(sRow + kMaxNb));
#ifdef BLADE_RF_TIMING
    if (tid == 0) {
      const unsigned long long t_done = gtime();
      atomicAdd(&g_rf[3], t_sel - t_comb);
      atomicAdd(&g_rf[4], t_done - t_sel);
      atomicAdd(&g_rf[5], 1ull);
    }
#endif
  }
#ifdef BLADE_RF_TIMING
  if (tid == 0) atomicMax(&g_rf[1], gtime());
#endif
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
  int* done = reinterpret_cast<int*>(ws + w.off_done);
  double* r64 = reinterpret_cast<double*>(ws + w.off_r64);
  double* mpart = reinterpret_cast<double*>(ws + w.off_mpart);
  double* lpart = reinterpret_cast<double*>(ws + w.off_lpart);
  const int64_t rows = p.BH * p.Nb;
  cudaError_t e;

  {  // K-mask.1 (sampling + gathered copies Q_s, K_s)
    const int64_t warps = p.BH * p.Nb * 2;
    auto kern = p.kk <= 16 ? sample_gather_kernel<D, true> : sample_gather_kernel<D, false>;
    kern<<<unsigned((warps + 7) / 8), 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
        p.BH, p.N, p.Nb, p.b, p.kk, p.seed, p.mode, p.share_qk, p.unit_offset, sample_idx, qs,
        ks, counters, p.attn_work);
  }
  // K-mask.2: tcgen05 probe (probe2.cu), every supported k and N_b
  e = launch_probe2(p.BH, p.N, p.Nb, p.b, p.kk, D, p.scale, qs, ks, pimp, stream);
  if (e != cudaSuccess) return e;
  // K-mask.3
  {  // K-mask.3, a programmatic dependent of K-mask.2 (its launch overlaps the probe's tail)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((rows + SEL_WARPS - 1) / SEL_WARPS));
    cfg.blockDim = dim3(SEL_WARPS * 32);
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, select_kernel, static_cast<const float*>(pimp), rows, p.Nb, p.tau,
                           p.lo, p.hi, p.guard, mask, kv_idx, kv_cnt, counters, flags, done,
                           p.neg_flagged);
    if (e != cudaSuccess) return e;
  }
  if (p.lpt_order) {  // before K-mask.4, so the attention stays its programmatic dependent
    e = launch_lpt_order(kv_cnt, p.BH, p.Nb, D, p.lpt_pairs, p.lpt_order, stream);
    if (e != cudaSuccess) return e;
  }
  // K-mask.4 (persistent grid; the queue length is read on the device)
  refine_kernel<D><<<148 * BLADE_RF_MINB, RF_THREADS, 0, stream>>>(
      qs, ks, p.N, p.Nb, p.b, p.kk, double(p.scale), w.nchunks, p.tau, p.lo, p.hi, counters,
      flags, done, r64, mpart, lpart, p_imp_out, mask, kv_idx, kv_cnt, n_refined);
#ifdef BLADE_RF_TIMING
  {
    static int calls = 0;
    unsigned long long h[8], z[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h, g_rf, sizeof(h));
    cudaMemcpyToSymbol(g_rf, z, sizeof(z));
    if (++calls % 10 == 0 && h[5])
      fprintf(stderr, "refine: kernel %.1f us, items end at %.1f us (max item %.1f us), %llu rows: "
              "combine %.1f us, select %.1f us per row\n", (h[1] - h[0]) * 1e-3,
              (h[2] - h[0]) * 1e-3, h[6] * 1e-3, h[5], h[3] * 1e-3 / h[5], h[4] * 1e-3 / h[5]);
  }
#endif
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

// ---------------------------------------------------------------------------
// LPT order of the attention CTAs: with content-adaptive lists the
// CTAs of a tau-mode call differ in work by up to N_b / lo; launching the
// longest first keeps the last wave short.  Items (a query block, or a pair
// of blocks for the two-block kernel) are sorted by kept-block count,
// descending, WITHIN each unit (one CTA per unit, counting sort): units stay
// in launch order, so the CTAs in flight keep sharing one unit's K and V in
// L2 (a global sort mixes every unit's K/V and measured slower on Wan).  The
// order of equal counts is arbitrary (atomics); it cannot change any result,
// every CTA writes its own rows.
// ---------------------------------------------------------------------------
namespace blade {
namespace {

constexpr int kLptBins = 2 * kMaxNb + 1;

__global__ void __launch_bounds__(256) lpt_order_kernel(const int32_t* __restrict__ kv_cnt,
                                                        int64_t BH, int Nb, int pairs,
                                                        int per_unit, int group,
                                                        int32_t* __restrict__ order) {
  __shared__ int hist[kLptBins];
  const int64_t u0 = int64_t(blockIdx.x) * group;
  const int64_t u1 = u0 + group < BH ? u0 + group : BH;
  const int items = int((u1 - u0) * per_unit);
  for (int b = threadIdx.x; b < kLptBins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  auto key = [&](int it) {
    const int64_t u = u0 + it / per_unit;
    const int x = it % per_unit;
    auto c = [&](int i) {
      const int v = kv_cnt[u * Nb + i];
      return v < 0 ? -1 - v : v;  // provisional count of a row K-mask.4 recomputes
    };
    return pairs ? c(2 * x) + (2 * x + 1 < Nb ? c(2 * x + 1) : 0) : c(x);
  };
  for (int it = threadIdx.x; it < items; it += blockDim.x) atomicAdd(&hist[key(it)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {  // descending exclusive scan: start of each count's range
    int run = 0;
    for (int b = kLptBins - 1; b >= 0; --b) {
      const int h = hist[b];
      hist[b] = run;
      run += h;
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < items; it += blockDim.x)
    order[u0 * per_unit + atomicAdd(&hist[key(it)], 1)] = int32_t(u0 * per_unit + it);
}

}  // namespace

cudaError_t launch_lpt_order(const int32_t* kv_cnt, int64_t BH, int Nb, int d, int pairs,
                             int32_t* order, cudaStream_t stream) {
  const int per_unit = pairs ? (Nb + 1) / 2 : Nb;
  // sort within groups of units whose K and V fit in about 48 MB of L2
  const double unit_kv = 2.0 * Nb * 128.0 * d * 2.0;
  int group = int(48e6 / unit_kv);
  group = group < 1 ? 1 : group;
  const int64_t ngroups = (BH + group - 1) / group;
  lpt_order_kernel<<<unsigned(ngroups), 256, 0, stream>>>(kv_cnt, BH, Nb, pairs, per_unit, group,
                                                          order);
  return cudaGetLastError();
}

}  // namespace blade
