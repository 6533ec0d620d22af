// Microbenchmark: achievable L2 -> shared-memory TMA bandwidth (all SMs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2508_10774_b200/csrc \
//        scripts/tma_bench.cu -o scripts/tma_bench.bin
// Each CTA (one per SM) streams 32 KB tiles (two 64 x 128 bf16 boxes, 128-byte
// swizzle, the attention kernel's K/V tile) of a [units, rows, 128] bf16
// tensor through a ring of smem slots, waiting only on the full barriers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc_ptx.cuh"
#include "tma_host.h"

using namespace blade;

constexpr int kSlots = 6;
constexpr int kTile = 32768;

__global__ void __launch_bounds__(32, 1) tma_stream(const __grid_constant__ CUtensorMap tm,
                                                    int tiles_per_unit, int units, int iters,
                                                    long long* cyc) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[kSlots];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) tc::mbar_init(full + s, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  const int u = (blockIdx.x * 13 + 5) % units;
  for (int it = 0; it < iters; ++it) {
    const int s = it % kSlots;
    if (it >= kSlots) tc::mbar_wait(full + s, ((it / kSlots) - 1) & 1);
    tc::mbar_arrive_expect_tx(full + s, kTile);
    const int row = (((it * 2654435761u) ^ (blockIdx.x * 40503u)) % tiles_per_unit) * 128;
    tc::tma_load_3d(smem + s * kTile, &tm, full + s, 0, row, u);
    tc::tma_load_3d(smem + s * kTile + 16384, &tm, full + s, 64, row, u);
  }
  for (int it = iters; it < iters + kSlots; ++it) {
    const int s = it % kSlots;
    tc::mbar_wait(full + s, ((it / kSlots) - 1) & 1);
  }
  cyc[blockIdx.x] = clock64() - t0;
}

#include <stdlib.h>
int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int units = argc > 1 ? atoi(argv[1]) : 2, N = 32768, D = 128;  // 8 MB per unit
  void* buf;
  cudaMalloc(&buf, size_t(units) * N * D * 2);
  cudaMemset(buf, 0, size_t(units) * N * D * 2);
  CUtensorMap tm;
  if (!make_tile_map(&tm, buf, units, N, D)) { printf("tensor map failed\n"); return 1; }
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int smem = kSlots * kTile + 1024;
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ctas : {148, 74, 296}) {
    const int iters = 2000;
    tma_stream<<<ctas, 32, smem>>>(tm, N / 128, units, 100, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_stream<<<ctas, 32, smem>>>(tm, N / 128, units, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ctas=%d: %.2f TB/s L2->smem (%s)\n", ctas,
           double(ctas) * iters * kTile / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
