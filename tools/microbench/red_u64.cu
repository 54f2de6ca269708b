// Throughput of red.global.add.u64 (the int64 fixed-point S accumulation of spmm_tc / the streaming
// f1 kernel) into an L2-resident array: warp instructions whose 32 lanes hit 32 consecutive
// 8-byte slots (the column-part pattern) and 32 slots k apart (the row-part pattern, S[p][c]).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/microbench/red_u64.cu -o red_u64
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void red_bench(long long *S, int64_t slots, int iters, int lane_stride) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t x = (uint64_t)warp * 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < iters; ++i) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    const int64_t base = (int64_t)((x >> 20) % (uint64_t)(slots - 32 * lane_stride));
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(S + base + (int64_t)lane * lane_stride), "l"(1ll) : "memory");
  }
}

int main() {
  const int64_t slots = 2 * 1024 * 1024;  // 16 MB: L2-resident
  long long *S;
  cudaMalloc(&S, slots * 8);
  cudaMemset(S, 0, slots * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int stride : {1, 10, 64}) {
    const int blocks = 148 * 8, threads = 256, iters = 2000;
    red_bench<<<blocks, threads>>>(S, slots, 10, stride);
    cudaEventRecord(a);
    red_bench<<<blocks, threads>>>(S, slots, iters, stride);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * threads * iters;
    printf("lane stride %2d: %.3e red.add.u64 per s (%.1f ms)\n", stride, ops / (ms * 1e-3), ms);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
