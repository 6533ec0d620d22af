// Microbenchmark: issue cost of tcgen05.mma from one thread (clock64 around
// the issue of a group of MMAs) and completion time, for the operand forms
// the attention kernels use.  One CTA per SM, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2508_10774_b200/csrc \
//        scripts/mma_issue_bench.cu -o scripts/mma_issue_bench.bin
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc_ptx.cuh"

using namespace blade;

// mode 0: SS  M128 N128 (S = Q K^T with Q in smem)
// mode 1: TS  M128 N128 (A from TMEM)
// mode 2: TS  M128 N64  (P V with d = 64)
// mode 3: SS  M128 N64
// mode 4: TS  M128 N128, a commit after every MMA
// mode 5: SS  M128 N256
// mode 6: TS  M128 N128, B MN-major (the P V form with d = 128)
// mode 7: TS  M128 N64,  B MN-major (the P V form with d = 64)
// mode 8: as 7, but every group of 8 is committed and waited for (cold start each group)
// mode 9: SS  M128 N128 groups of 4 (S with d = 64), committed and waited for each group
// mode 10: the attention skeleton of one block: groups of 8 SS (S, N128) and 8 TS (P V,
//          N128, B MN-major) alternating, a commit after each group, no waits
// mode 11: as 10 without the per-group commits
// mode 12: as 10 with two blocks (S_A, PV_A, S_B, PV_B into separate TMEM columns)
template <int MODE>
__global__ void __launch_bounds__(128, 1) issue_loop(int groups, long long* out) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar, bar_g;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 96 * 1024 / 4; e += 128) reinterpret_cast<uint32_t*>(smem)[e] = 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&bar_g, 1);
    tc::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tslot;
  if (MODE >= 10 && threadIdx.x == 0) {
    constexpr uint32_t idS = tc::idesc_bf16(128, 128, 0, 0), idO = tc::idesc_bf16(128, 128, 0, 1);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t_start = clock64();
    for (int g = 0; g < groups; ++g) {
      const int blk = MODE == 12 ? (g & 1) : 0;
      const uint32_t dS = tmem + blk * 128, dO = tmem + 256 + blk * 128;
      if ((g >> (MODE == 12 ? 1 : 0)) & 1) {  // P V group
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc::mma_ts(dO, dS + 64 + ks * 8, tc::sw128_desc(b + ks * 2048, 16384, 1024), idO, 1);
      } else {  // S group
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          tc::mma_ss(dS, tc::sw128_desc(a + off, 16, 1024), tc::sw128_desc(b + off, 16, 1024),
                     idS, ks > 0);
        }
      }
      if (MODE != 11) tc::commit(&bar_g);  // arrivals nobody waits for
    }
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x * 2] = 0;
    out[blockIdx.x * 2 + 1] = clock64() - t_start;
  } else if (threadIdx.x == 0) {
    constexpr int N = (MODE == 2 || MODE == 3 || MODE == 7 || MODE == 8) ? 64 : (MODE == 5 ? 256 : 128);
    constexpr bool kMN = MODE == 6 || MODE == 7 || MODE == 8;
    constexpr int G = MODE == 9 ? 4 : 8;
    constexpr uint32_t id = tc::idesc_bf16(128, N, 0, kMN ? 1 : 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long issue = 0, t_start = clock64();
    for (int g = 0; g < groups; ++g) {
      const long long t0 = clock64();
#pragma unroll
      for (int ks = 0; ks < G; ++ks) {
        const uint32_t off = (ks & 3) * 32;
        if (kMN)
          tc::mma_ts(tmem, tmem + 256 + ks * 8, tc::sw128_desc(b + ks * 2048, 16384, 1024), id,
                     1);
        else if (MODE == 1 || MODE == 2 || MODE == 4)
          tc::mma_ts(tmem, tmem + 256 + ks * 8, tc::sw128_desc(b + off, 16, 1024), id, 1);
        else
          tc::mma_ss(tmem, tc::sw128_desc(a + off, 16, 1024), tc::sw128_desc(b + off, 16, 1024),
                     id, 1);
        if (MODE == 4) tc::commit(&bar);
      }
      issue += clock64() - t0;
      if (MODE == 8 || MODE == 9) {
        tc::commit(&bar);
        tc::mbar_wait(&bar, g & 1);
      }
    }
    if (MODE != 8 && MODE != 9) {
      tc::commit(&bar);
      tc::mbar_wait(&bar, 0);
    }
    const long long t_end = clock64();
    out[blockIdx.x * 2] = issue;
    out[blockIdx.x * 2 + 1] = t_end - t_start;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run(const char* name) {
  const int groups = 500;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 2 * 148);
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(issue_loop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  issue_loop<MODE><<<148, 128, smem>>>(groups, d);
  cudaError_t err = cudaDeviceSynchronize();
  long long h[2 * 148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double n = groups * (MODE == 9 ? 4.0 : 8.0);  // modes 10-12: 8 MMAs per group too
  printf("%-28s issue %.1f cyc/MMA, total %.1f cyc/MMA (%s)\n", name, h[0] / n, h[1] / n,
         cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  run<0>("SS M128 N128");
  run<1>("TS M128 N128");
  run<2>("TS M128 N64");
  run<3>("SS M128 N64");
  run<4>("TS M128 N128 + commit each");
  run<5>("SS M128 N256");
  run<6>("TS M128 N128 B MN-major");
  run<7>("TS M128 N64 B MN-major");
  run<8>("PV d64 group, cold each");
  run<9>("S d64 group of 4, cold each");
  run<10>("skeleton 1 block, commits");
  run<11>("skeleton 1 block, no commits");
  run<12>("skeleton 2 blocks, commits");
  return 0;
}
