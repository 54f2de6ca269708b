// sort.cuh -- per-iteration preparation of the streaming path: a stable counting sort of the
// points by label (cluster-sorted order p -> point perm[p], segment starts seg[c]) and the
// gather of the split operands / per-point constants into that order, so that the fused
// GEMM's B operand walks the clusters one after another.
#pragma once
#include "common.cuh"

namespace kkm {

constexpr int SORT_BLOCK = 1024;  // points per block of the counting sort

// blockcount[b * k + c] = #{j in block b : labels[j] == c}
__global__ void sort_count_kernel(const int32_t *__restrict__ labels, int64_t n, int k,
                                  int32_t *__restrict__ blockcount) {
  extern __shared__ int32_t h[];
  for (int c = threadIdx.x; c < k; c += blockDim.x) h[c] = 0;
  __syncthreads();
  const int64_t j0 = (int64_t)blockIdx.x * SORT_BLOCK;
  for (int t = threadIdx.x; t < SORT_BLOCK; t += blockDim.x) {
    const int64_t j = j0 + t;
    if (j < n) atomicAdd(&h[labels[j]], 1);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) blockcount[(int64_t)blockIdx.x * k + c] = h[c];
}

// Per-cluster totals over the sorted set: tot[c] = sum_b blockcount[b][c] (block-wide sum).
__device__ int32_t cluster_total(const int32_t *__restrict__ blockcount, int nb, int k, int c, int32_t *buf) {
  int32_t s = 0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += blockcount[(int64_t)b * k + c];
  buf[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < (unsigned)w) buf[threadIdx.x] += buf[threadIdx.x + w];
    __syncthreads();
  }
  const int32_t t = buf[0];
  __syncthreads();
  return t;
}

// One block per cluster c (+ block k writes seg): blockoff[b][c] = seg[c] + sum_{b' < b}
// blockcount[b'][c]; seg[c] = sum_{c' < c} (points of cluster c' in the set), seg[k] = set size.
// blockDim.x must be a power of two.
__global__ void sort_scan_kernel(const int32_t *__restrict__ blockcount, int nb, int k,
                                 int32_t *__restrict__ blockoff, int32_t *__restrict__ seg) {
  const int c = blockIdx.x;
  extern __shared__ int32_t buf[];
  __shared__ int32_t base;
  __shared__ int32_t carry;
  int32_t s = 0;
  for (int cc = 0; cc < (c < k ? c : k); ++cc) {
    const int32_t t = cluster_total(blockcount, nb, k, cc, buf);
    if (c == k && threadIdx.x == 0) seg[cc] = s;
    s += t;
  }
  if (c == k) {
    if (threadIdx.x == 0) seg[k] = s;
    return;
  }
  if (threadIdx.x == 0) {
    base = s;
    carry = 0;
  }
  __syncthreads();
  // block-wide exclusive scan over b in tiles of blockDim.x
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int b = b0 + threadIdx.x;
    const int32_t v = b < nb ? blockcount[(int64_t)b * k + c] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // Hillis-Steele inclusive scan
      int32_t add = threadIdx.x >= (unsigned)off ? buf[threadIdx.x - off] : 0;
      __syncthreads();
      buf[threadIdx.x] += add;
      __syncthreads();
    }
    if (b < nb) blockoff[(int64_t)b * k + c] = base + carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += buf[threadIdx.x];
    __syncthreads();
  }
}

// Stable scatter: point j of block b goes to blockoff[b][c] + (rank of j among the block's
// points of cluster c, in index order). perm[p] = j, pos[j] = p. 256 threads, 4 points each,
// processed as 4 rounds of 256 consecutive points.
__global__ void __launch_bounds__(256) sort_scatter_kernel(const int32_t *__restrict__ labels, int64_t n,
                                                           int k, const int32_t *__restrict__ blockoff,
                                                           int32_t *__restrict__ perm,
                                                           int32_t *__restrict__ pos) {
  extern __shared__ int32_t sm[];
  int32_t *running = sm;            // [k] running offset for the block
  int32_t *wcount = sm + k;         // [8 warps][k] per-round counts
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < k; c += blockDim.x) running[c] = blockoff[(int64_t)blockIdx.x * k + c];
  __syncthreads();
  const int64_t j0 = (int64_t)blockIdx.x * SORT_BLOCK;
  for (int round = 0; round < SORT_BLOCK / 256; ++round) {
    const int64_t j = j0 + round * 256 + threadIdx.x;
    const int lab = j < n ? labels[j] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, lab);
    const int rank_in_warp = __popc(same & ((1u << lane) - 1u));
    for (int c = threadIdx.x; c < 8 * k; c += blockDim.x) wcount[c] = 0;
    __syncthreads();
    if (lab >= 0 && rank_in_warp == 0) wcount[warp * k + lab] = __popc(same);
    __syncthreads();
    if (lab >= 0) {
      int32_t before = 0;
      for (int w = 0; w < warp; ++w) before += wcount[w * k + lab];
      const int32_t p = running[lab] + before + rank_in_warp;
      perm[p] = (int32_t)j;
      pos[j] = p;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      int32_t tot = 0;
      for (int w = 0; w < 8; ++w) tot += wcount[w * k + c];
      running[c] += tot;
    }
    __syncthreads();
  }
}

// Sorted copies of the set [b0, b0 + n): Xs[p] = X[b0 + perm[p]] for the hi and lo operands
// (dp 16-bit values per row, uint4 vectors), vs[p] = v[b0 + perm[p]] for norms and rscale.
// Rows p in [n, npad) are zeroed.
__global__ void gather_rows_kernel(const uint16_t *__restrict__ Xhi, const uint16_t *__restrict__ Xlo,
                                   const float *__restrict__ norms, const float *__restrict__ rscale,
                                   const int32_t *__restrict__ perm, int64_t b0, int64_t n, int64_t npad,
                                   int64_t dp, uint16_t *__restrict__ Shi, uint16_t *__restrict__ Slo,
                                   float *__restrict__ snorms, float *__restrict__ srscale) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= npad) return;
  const int64_t nv = dp / 8;  // uint4 per row
  uint4 *dh = reinterpret_cast<uint4 *>(Shi + p * dp);
  uint4 *dl = reinterpret_cast<uint4 *>(Slo + p * dp);
  if (p < n) {
    const int64_t j = b0 + perm[p];
    const uint4 *sh = reinterpret_cast<const uint4 *>(Xhi + j * dp);
    const uint4 *sl = reinterpret_cast<const uint4 *>(Xlo + j * dp);
    for (int64_t v = lane; v < nv; v += 32) {
      dh[v] = sh[v];
      dl[v] = sl[v];
    }
    if (lane == 0) {
      snorms[p] = norms[j];
      srscale[p] = rscale[j];
    }
  } else {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t v = lane; v < nv; v += 32) {
      dh[v] = z;
      dl[v] = z;
    }
    if (lane == 0) {
      snorms[p] = 0.f;
      srscale[p] = 1.f;
    }
  }
}

}  // namespace kkm
