// TMEM read bandwidth on one SM (tcgen05.ld.32x32b.x32): how fast can epilogue warps drain a
// TMEM accumulator? One CTA per SM, W warps (warp w reads lanes 32 (w % 4) ...), each warp loads
// NLD x 32 columns per round; bytes per SM clock reported. Decides whether a fused kernel can
// afford to drain its accumulators more than once per tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/microbench/tmem_ld.cu -o tmem_ld
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int NCOLS>
__global__ void tmem_bench(int rounds, int nwarps_active, unsigned long long *cycles, float *sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot;
  float acc = 0.f;
  unsigned long long t0 = 0, t1 = 0;
  __syncthreads();
  if (threadIdx.x == 0) t0 = clock64();
  if (warp < nwarps_active) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col0 = (uint32_t)((warp >> 2) * NCOLS) & 511u;
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int c = 0; c < NCOLS; c += 32) {
        float v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
            "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
            "%30, %31}, [%32];"
            : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
              "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
              "=f"(v[14]), "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]),
              "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]),
              "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
            : "r"(base + lane_base + ((col0 + (uint32_t)c) & 511u)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) acc += v[q];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

int main() {
  const int blocks = 148, rounds = 2000;
  unsigned long long *cyc;
  float *sink;
  cudaMalloc(&cyc, blocks * 8);
  cudaMalloc(&sink, blocks * 1024 * 4);
  for (int nw : {4, 8, 16}) {
    for (int pass = 0; pass < 2; ++pass) {
      tmem_bench<128><<<blocks, 512>>>(rounds, nw, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
    }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, mn = ~0ull;
    for (int b = 0; b < blocks; ++b) {
      mx = h[b] > mx ? h[b] : mx;
      mn = h[b] < mn ? h[b] : mn;
    }
    const double bytes = (double)nw * 32 * 128 * 4 * rounds;  // per SM
    printf("warps %2d: %.1f B/clk per SM (min cycles %llu, max %llu)\n", nw, bytes / (double)mx, mn, mx);
  }
  return 0;
}
