// gt_pool.cu — MeanPool_n of K and V for ASA with global tokens (PAPER.md
// P:135 Step 2.2 (2): "K_aug = Concat(K, MeanPool_n(K)) (and similarly for
// V)").  Window w covers tokens [w n, min((w+1) n, N)) (reading R-18); the
// pooled row is the fp32 mean of its n_w tokens rounded once to bf16
// (reading R-19: K_aug has the input dtype).
//
// HBM-bound: every K and V element is read once, N_g rows are written.  CTA
// = one (window, unit, K|V); 256 threads = RP row lanes x (D/8) column lanes,
// each load a 16-byte vector (a warp reads 2 or 4 whole 256/128-byte rows:
// fully coalesced); the RP partial sums are combined through shared memory.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace blade {
namespace {

template <int D>
__global__ void __launch_bounds__(256) gt_pool_kernel(const __nv_bfloat16* __restrict__ k,
                                                      const __nv_bfloat16* __restrict__ v, int N,
                                                      int window, int Ng,
                                                      __nv_bfloat16* __restrict__ kg,
                                                      __nv_bfloat16* __restrict__ vg) {
  constexpr int CL = D / 8;     // 16-byte column lanes per row
  constexpr int RP = 256 / CL;  // row lanes
  __shared__ float part[RP][D + 4];
  const int w = blockIdx.x;
  const int64_t u = blockIdx.y;
  const __nv_bfloat16* src = blockIdx.z == 0 ? k : v;
  __nv_bfloat16* dst = blockIdx.z == 0 ? kg : vg;
  const int cl = threadIdx.x % CL, rl = threadIdx.x / CL;
  const int r0 = w * window;
  const int r1 = min(r0 + window, N);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const __nv_bfloat16* base = src + (u * N) * int64_t(D) + cl * 8;
#pragma unroll 4
  for (int r = r0 + rl; r < r1; r += RP) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(base + int64_t(r) * D));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      acc[2 * e] += f.x;
      acc[2 * e + 1] += f.y;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[rl][cl * 8 + e] = acc[e];
  __syncthreads();
  if (threadIdx.x < D) {
    const int c = threadIdx.x;
    float t = 0.f;
#pragma unroll 8
    for (int z = 0; z < RP; ++z) t += part[z][c];
    const float mean = __fdiv_rn(t, float(r1 - r0));
    dst[(u * Ng + w) * int64_t(D) + c] = __float2bfloat16_rn(mean);
  }
}

}  // namespace

cudaError_t launch_gt_pool(const void* k, const void* v, int64_t BH, int N, int d, int window,
                           void* kg, void* vg, cudaStream_t stream) {
  const int Ng = (N + window - 1) / window;
  dim3 grid(unsigned(Ng), unsigned(BH), 2u);
  auto K = reinterpret_cast<const __nv_bfloat16*>(k);
  auto V = reinterpret_cast<const __nv_bfloat16*>(v);
  auto KG = reinterpret_cast<__nv_bfloat16*>(kg);
  auto VG = reinterpret_cast<__nv_bfloat16*>(vg);
  if (d == 128)
    gt_pool_kernel<128><<<grid, 256, 0, stream>>>(K, V, N, window, Ng, KG, VG);
  else if (d == 64)
    gt_pool_kernel<64><<<grid, 256, 0, stream>>>(K, V, N, window, Ng, KG, VG);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace blade
