// gemm_simt.cuh -- a1 correctness baseline (KKM_PREC_FP32_SIMT): K = kappa(X X^T)
// with fp32 CUDA-core FMA, 128x128 CTA tile, 8x8 per thread, kappa fused in the
// epilogue (Eqs. b, k P:92-103). The tensor-core path is gemm_tc.cuh.
#pragma once
#include "common.cuh"

namespace kkm {

constexpr int SG_BM = 128, SG_BN = 128, SG_BK = 8;

// out[(i - i0) * ldo + (j - j0)] = kappa(x_i . x_j) for i in [i0, i0 + m), j in
// [j0, j0 + ncov); entries with j >= n (column padding) are written as 0.
__global__ void __launch_bounds__(256) gemm_simt_kernel(const float *__restrict__ X, int64_t ldx,
                                                        int64_t n, int64_t d, int64_t i0,
                                                        int64_t m, int64_t j0, int64_t ncov,
                                                        const float *__restrict__ norms,
                                                        KappaParams kp, float *__restrict__ out,
                                                        int64_t ldo) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t bi = i0 + (int64_t)blockIdx.y * SG_BM;  // first global row of the tile
  const int64_t bj = j0 + (int64_t)blockIdx.x * SG_BN;  // first global column
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;

  const int lr = tid >> 1;         // tile row this thread loads
  const int lk = (tid & 1) * 4;    // first k of its 4-element slice
  const int64_t ga = bi + lr, gb = bj + lr;
  const bool va = ga < i0 + m && ga < n, vb = gb < n;
  for (int64_t k0 = 0; k0 < d; k0 += SG_BK) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t kk = k0 + lk + u;
      As[lk + u][lr] = (va && kk < d) ? X[ga * ldx + kk] : 0.f;
      Bs[lk + u][lr] = (vb && kk < d) ? X[gb * ldx + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][ty * 4 + u];
        a[4 + u] = As[kk][64 + ty * 4 + u];
        b[u] = Bs[kk][tx * 4 + u];
        b[4 + u] = Bs[kk][64 + tx * 4 + u];
      }
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[p][q] = fmaf(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int64_t i = bi + (p < 4 ? ty * 4 + p : 64 + ty * 4 + (p - 4));
    if (i >= i0 + m) continue;
    const float ni = norms[i];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t j = bj + (q < 4 ? tx * 4 + q : 64 + tx * 4 + (q - 4));
      if (j >= j0 + ncov) continue;
      float v = (j < n && i < n) ? kappa_epilogue(kp, acc[p][q], ni, norms[j], i == j) : 0.f;
      out[(i - i0) * ldo + (j - j0)] = v;
    }
  }
}

}  // namespace kkm
