// Microbenchmark: FP64 FMA and exp() throughput per SM on this GPU.
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void dfma_loop(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-7);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_loop(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999999f, 1e-7f);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dexp_loop(double* out, int iters) {
  double s = 0, x = -threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) { s += exp(x); x -= 1e-4; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int it = 20000;
  dfma_loop<<<148 * 4, 256>>>(d, 10); cudaEventRecord(e0); dfma_loop<<<148 * 4, 256>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("DFMA: %.2f TFLOP/s\n", 2.0 * 8 * it * 148 * 4 * 256 / (ms * 1e-3) / 1e12);
  ffma_loop<<<148 * 4, 256>>>((float*)d, 10); cudaEventRecord(e0); ffma_loop<<<148 * 4, 256>>>((float*)d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("FFMA: %.2f TFLOP/s\n", 2.0 * 8 * it * 148 * 4 * 256 / (ms * 1e-3) / 1e12);
  dexp_loop<<<148 * 4, 256>>>(d, 10); cudaEventRecord(e0); dexp_loop<<<148 * 4, 256>>>(d, 2000); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("exp(double): %.2f Gexp/s\n", 1.0 * 2000 * 148 * 4 * 256 / (ms * 1e-3) / 1e9);
  return 0;
}
