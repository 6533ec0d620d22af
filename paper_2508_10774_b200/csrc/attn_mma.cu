// attn_mma.cu — block-sparse attention forward, legacy-tensor-path BASELINE
// (mma.sync m16n8k16, FlashAttention-2 style).  Kept as the comparison point
// the tcgen05 kernel (attn_tc.cu) must beat, and as a second independent GPU
// implementation in the parity tests.  PAPER.md P:133 (Step 2.2 (1)).
//
// CTA = one (unit u, query block i) = 128 query rows, 8 warps x 16 rows.
// Walks kv_idx[u, i, 0:kv_cnt) in list order; each kept 128-key block is
// two 64-key stages (cp.async double buffer).  fp32 online softmax in the
// log2 domain; O normalised at the end; LSE = ln sum exp(scale * s).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace blade {
#ifdef BLADE_WITH_BASELINES  // comparison baseline, not in the product build
namespace {

constexpr int AM_ROWS = 128;
constexpr int AM_KEYS = 64;

template <int D>
__global__ void __launch_bounds__(256, 1) attn_mma_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
    const __nv_bfloat16* __restrict__ V, int N, int Nb, float scale_log2,
    const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
    __nv_bfloat16* __restrict__ O, float* __restrict__ LSE) {
  extern __shared__ __align__(128) char smem[];
  char* sQ = smem;                           // [128][D]
  char* sK = sQ + AM_ROWS * D * 2;           // [2][64][D]
  char* sV = sK + 2 * AM_KEYS * D * 2;       // [2][64][D]
  constexpr int CH = D / 8;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = blockIdx.x;
  const int64_t u = blockIdx.y;
  const int64_t base = u * int64_t(N) * D;
  const int32_t* list = kv_idx + (u * Nb + i) * int64_t(Nb);
  const int cnt = kv_cnt[u * Nb + i];
  const int ntiles = cnt * 2;

  for (int e = tid; e < AM_ROWS * CH; e += 256) {
    const int r = e / CH, c = e % CH;
    const int gr = i * AM_ROWS + r;
    cp_async16(smem_u32(sQ) + swz<D>(r, c), Q + base + int64_t(min(gr, N - 1)) * D + c * 8,
               gr < N ? 16 : 0);
  }
  auto load_kv = [&](int t, int stage) {
    const int j = list[t >> 1];
    const int key0 = j * 128 + (t & 1) * AM_KEYS;
    const uint32_t kb = smem_u32(sK + stage * AM_KEYS * D * 2);
    const uint32_t vb = smem_u32(sV + stage * AM_KEYS * D * 2);
    for (int e = tid; e < AM_KEYS * CH; e += 256) {
      const int r = e / CH, c = e % CH;
      const int gr = key0 + r;
      const int64_t off = base + int64_t(min(gr, N - 1)) * D + c * 8;
      cp_async16(kb + swz<D>(r, c), K + off, gr < N ? 16 : 0);
      cp_async16(vb + swz<D>(r, c), V + off, gr < N ? 16 : 0);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const int g = lane >> 2, qd = lane & 3;
  uint32_t qa[D / 16][4];
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) load_kv(t + 1, (t + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const int r = warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int c = ks * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ) + swz<D>(r, c), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
      }
    }
    const uint32_t kb = smem_u32(sK + (t & 1) * AM_KEYS * D * 2);
    const uint32_t vb = smem_u32(sV + (t & 1) * AM_KEYS * D * 2);
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + 8 * (lane >> 4);
        const int c = ks * 2 + ((lane >> 3) & 1);
        ldsm_x4(kb + swz<D>(r, c), b0, b1, b2, b3);
        mma_bf16(s[2 * np], qa[ks], b0, b1);
        mma_bf16(s[2 * np + 1], qa[ks], b2, b3);
      }
    }
    const int key0 = list[t >> 1] * 128 + (t & 1) * AM_KEYS;
    const bool tail = key0 + AM_KEYS > N;
    float tmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool ok = !tail || key0 + n * 8 + qd * 2 + h < N;
        s[n][h] = ok ? s[n][h] * scale_log2 : -INFINITY;
        s[n][2 + h] = ok ? s[n][2 + h] * scale_log2 : -INFINITY;
        tmax[0] = fmaxf(tmax[0], s[n][h]);
        tmax[1] = fmaxf(tmax[1], s[n][2 + h]);
      }
    }
    float corr[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float tm = tmax[hr];
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 2));
      const float m_new = fmaxf(m_run[hr], tm);
      // a fully masked 64-key half-tile keeps m_new = -inf: use 0 as the shift
      const float msub = m_new == -INFINITY ? 0.f : m_new;
      corr[hr] = ex2(m_run[hr] - msub);
      m_run[hr] = m_new;
      float acc = 0.f;
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        s[n][2 * hr] = ex2(s[n][2 * hr] - msub);
        s[n][2 * hr + 1] = ex2(s[n][2 * hr + 1] - msub);
        acc += s[n][2 * hr] + s[n][2 * hr + 1];
      }
      l_run[hr] = l_run[hr] * corr[hr] + acc;
    }
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= corr[0]; o[n][1] *= corr[0];
      o[n][2] *= corr[1]; o[n][3] *= corr[1];
    }
    // O += P V   (P from registers as the A operand, 4 k-steps of 16 keys)
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kt][0], s[2 * kt][1]);
      pa[1] = pack_bf16(s[2 * kt][2], s[2 * kt][3]);
      pa[2] = pack_bf16(s[2 * kt + 1][0], s[2 * kt + 1][1]);
      pa[3] = pack_bf16(s[2 * kt + 1][2], s[2 * kt + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int r = kt * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int c = dp * 2 + (lane >> 4);
        ldsm_x4_t(vb + swz<D>(r, c), b0, b1, b2, b3);
        mma_bf16(o[2 * dp], pa, b0, b1);
        mma_bf16(o[2 * dp + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    float l = l_run[hr];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const float inv = 1.f / l;
    const int r = i * AM_ROWS + warp * 16 + g + 8 * hr;
    if (r < N) {
      __nv_bfloat16* orow = O + base + int64_t(r) * D;
#pragma unroll
      for (int n = 0; n < D / 8; ++n)
        *reinterpret_cast<uint32_t*>(orow + n * 8 + qd * 2) =
            pack_bf16(o[n][2 * hr] * inv, o[n][2 * hr + 1] * inv);
      if (LSE && qd == 0) LSE[u * N + r] = (m_run[hr] + log2f(l)) * 0.69314718055994531f;
    }
  }
}

template <int D>
cudaError_t launch_d(const AttnProblem& p, const void* q, const void* k, const void* v,
                     const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                     cudaStream_t stream) {
  const size_t smem = size_t(AM_ROWS) * D * 2 + 4 * size_t(AM_KEYS) * D * 2;
  cudaError_t e = cudaFuncSetAttribute(attn_mma_kernel<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(p.Nb), unsigned(p.BH));
  attn_mma_kernel<D><<<grid, 256, smem, stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
      reinterpret_cast<const __nv_bfloat16*>(v), p.N, p.Nb, p.scale * kLog2e, kv_idx, kv_cnt,
      reinterpret_cast<__nv_bfloat16*>(o), lse);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_mma(const AttnProblem& p, const void* q, const void* k,
                            const void* v, const int32_t* kv_idx, const int32_t* kv_cnt,
                            void* o, float* lse, cudaStream_t stream) {
  if (p.d == 64) return launch_d<64>(p, q, k, v, kv_idx, kv_cnt, o, lse, stream);
  if (p.d == 128) return launch_d<128>(p, q, k, v, kv_idx, kv_cnt, o, lse, stream);
  return cudaErrorInvalidValue;
}

#else
cudaError_t launch_attn_mma(const AttnProblem&, const void*, const void*, const void*,
                            const int32_t*, const int32_t*, void*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
#endif  // BLADE_WITH_BASELINES

}  // namespace blade
