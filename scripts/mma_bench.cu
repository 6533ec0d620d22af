// Microbenchmark: tcgen05.mma throughput per instruction on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2508_10774_b200/csrc \
//        scripts/mma_bench.cu -o build/mma_bench && build/mma_bench
// One CTA per SM; one thread issues R back-to-back MMAs (K = 16 bf16) of shape
// 128 x N with A from smem (SS) or TMEM (TS), then waits on a commit barrier.
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc_ptx.cuh"

using namespace blade;

template <int N, bool kTS>
__global__ void __launch_bounds__(128, 1) mma_loop(int reps, long long* cycles) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 64 * 1024 / 4; e += 128) reinterpret_cast<uint32_t*>(smem)[e] = 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = tc::idesc_bf16(128, N, 0, 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
        if (kTS)
          tc::mma_ts(tmem, tmem + 256 + ks * 8, tc::sw128_desc(b + off, 16, 1024), id, 1);
        else
          tc::mma_ss(tmem, tc::sw128_desc(a + off, 16, 1024), tc::sw128_desc(b + off, 16, 1024),
                     id, 1);
      }
    }
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int N, bool kTS>
void run(int ctas) {
  const int reps = 2000;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * ctas);
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(mma_loop<N, kTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_loop<N, kTS><<<ctas, 128, smem>>>(10, d);  // warm
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("warm launch failed: %s\n", cudaGetErrorString(err)); return; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<N, kTS><<<ctas, 128, smem>>>(reps, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  const double instr = double(reps) * 8;
  const double flop = 2.0 * 128 * N * 16 * instr * ctas;
  printf("%s N=%3d ctas=%3d: %.1f cycles/instr (clock64), %.1f TFLOP/s (events), err=%s\n",
         kTS ? "TS" : "SS", N, ctas, double(h[0]) / instr, flop / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  run<64, false>(148);
  run<128, false>(148);
  run<256, false>(148);
  run<64, true>(148);
  run<128, true>(148);
  run<256, true>(148);
  run<128, true>(1);
  run<256, true>(1);
  return 0;
}
