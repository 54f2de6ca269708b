// kpp.cuh -- f3: K-means++ seeding in feature space (P:567 names it as future
// work). D^2 sampling with ||phi(x) - phi(c)||^2 = K(x,x) - 2 K(x,c) + K(c,c), in fp64 from the
// fp32 points (so the sampling sees exact-to-rounding distances, not the fp16x3 K tiles):
//   kpp_dist: one warp per point: distance to the newest center, running min D(x) and its
//             lowest-index argmin label;
//   kpp_pick: one CTA: fixed-order fp64 sums of max(D, 0) over contiguous chunks, prefix over
//             the chunks, then the smallest index whose running sum exceeds u * total.
// The uniforms u are inputs (kkm_seed_kmeanspp), so the oracle consumes the same draws.
#pragma once
#include <climits>
#include "common.cuh"

namespace kkm {

__device__ __forceinline__ double kpp_kappa(int kind, double gamma, double coef0, int degree, double dot,
                                            double r2) {
  if (kind == 0) return dot;
  if (kind == 1) {
    const double b = gamma * dot + coef0;
    double v = 1.0;
    for (int e = 0; e < degree; ++e) v *= b;
    return v;
  }
  return exp(-gamma * r2);
}

// t: index of the newest center c (point index); t == 0 initialises D and labels.
__global__ void kpp_dist_kernel(const float *__restrict__ Xf, int64_t ldf, int64_t n, int64_t d,
                                const int64_t *__restrict__ centers, int t, int kind, double gamma, double coef0,
                                int degree, double *__restrict__ D, int32_t *__restrict__ labels) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const int64_t c = centers[t];
  const float *x = Xf + i * ldf, *y = Xf + c * ldf;
  double sxy = 0.0, sxx = 0.0, syy = 0.0, r2 = 0.0;
  for (int64_t q = lane; q < d; q += 32) {
    const double a = x[q], b = y[q];
    sxy += a * b;
    sxx += a * a;
    syy += b * b;
    r2 += (a - b) * (a - b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sxy += __shfl_xor_sync(0xffffffffu, sxy, o);
    sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
    syy += __shfl_xor_sync(0xffffffffu, syy, o);
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  }
  if (lane == 0) {
    const double kxx = kind == 2 ? 1.0 : kpp_kappa(kind, gamma, coef0, degree, sxx, 0.0);
    const double kcc = kind == 2 ? 1.0 : kpp_kappa(kind, gamma, coef0, degree, syy, 0.0);
    const double dist = kxx - 2.0 * kpp_kappa(kind, gamma, coef0, degree, sxy, r2) + kcc;
    if (t == 0 || dist < D[i]) {
      D[i] = dist;
      labels[i] = t;
    }
  }
}

// One CTA of 1024 threads: centers[t + 1] = inverse-CDF pick of u over max(D, 0); if the total
// is 0 (no point left at positive distance), the previous center again.
__global__ void __launch_bounds__(1024) kpp_pick_kernel(const double *__restrict__ D, int64_t n, double u, int t,
                                                        int64_t *__restrict__ centers) {
  __shared__ double part[1024];
  __shared__ double base[1024];
  __shared__ long long found;
  const int tid = threadIdx.x;
  const int64_t L = (n + 1023) / 1024;
  const int64_t a = tid * L < n ? tid * L : n, b = a + L < n ? a + L : n;
  double s = 0.0;
  for (int64_t i = a; i < b; ++i) s += D[i] > 0.0 ? D[i] : 0.0;
  part[tid] = s;
  if (tid == 0) found = LLONG_MAX;
  __syncthreads();
  if (tid == 0) {  // fixed-order prefix over the chunks
    double run = 0.0;
    for (int q = 0; q < 1024; ++q) {
      base[q] = run;
      run += part[q];
    }
    part[0] = run;  // total (part[0] is no longer needed as a chunk sum: base holds the prefix)
  }
  __syncthreads();
  const double total = part[0];
  if (total <= 0.0) {
    if (tid == 0) centers[t + 1] = centers[t];
    return;
  }
  const double target = u * total;
  // the chunk whose running sums cross target scans its points in order
  double run = base[tid];
  for (int64_t i = a; i < b; ++i) {
    run += D[i] > 0.0 ? D[i] : 0.0;
    if (run > target) {
      atomicMin(&found, (long long)i);
      break;
    }
  }
  __syncthreads();
  if (tid == 0) {
    long long pick = found;
    if (pick == LLONG_MAX)  // rounding at the top end: the last point with D > 0
      for (int64_t i = n - 1; i >= 0; --i)
        if (D[i] > 0.0) {
          pick = i;
          break;
        }
    centers[t + 1] = pick;
  }
}

}  // namespace kkm
