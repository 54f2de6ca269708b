// spmm.cuh -- a2 on a materialised K: S(i, c) = sum_{j : cl(j) = c} K(i, j), the
// unnormalised E = K V^T of Eq. (e) (V of Eq. v: one nonzero
// 1/|L_c| per column, so E(i,c) = S(i,c) / |L_c|, applied in update.cuh).
//
// HBM-bound: every iteration streams the rank's K block (n_local x n fp32) once.
// Design:
//   * persistent CTAs, one per SM; a work item = R consecutive rows (8 for KP <= 10, else 4)
//     x one column split; the last warp is a producer that streams 2048-column chunks of
//     those rows plus the matching labels into a 3-stage (R = 8) / 5-stage (R = 4) shared-
//     memory ring with 1-D bulk copies (cp.async.bulk, the TMA engine) completing on
//     mbarriers, so ~200 KB per SM are in flight without registers;
//   * 4 consumer warps read the chunk from shared memory (conflict-free LDS.128) and reduce
//     it into per-lane accumulators acc[row][cluster] with a one-hot mask:
//     acc += K(i, j) * [cl(j) == c], two columns per FFMA2 (fma.rn.f32x2), so the cost per
//     element is ~KP/2 FFMA2 + KP/R mask ops and no divergent indexing;
//   * fp32 within a lane (<= 512 columns per split), fixed-order shuffle tree across
//     lanes, fp64 across the consumer warps in fixed order -> deterministic.
#pragma once
#include "common.cuh"

namespace kkm {

template <int KP>
struct SpRows;
constexpr int SP_MAX_CHUNKS_PER_SPLIT = 128;  // bounds fp32 terms per lane (<= 512 per lane)
constexpr int SP_KPMAX = 16;

// R rows per work item: the one-hot masks are per column and shared by all R rows, so more
// rows amortise them; R is bounded by the 2 R KP accumulator registers.
template <int KP>
struct SpRows {
  static constexpr int R = KP <= 10 ? 8 : 4;     // 2 R KP accumulator registers per thread
  static constexpr int CH = 2048;                 // columns per chunk (fewer stage handshakes)
  static constexpr int STAGES = R == 8 ? 3 : 5;  // 216 / 200 KB of K + labels in flight
  // 4 consumer warps + the producer keep <= 2 warps per SM sub-partition (16K registers each),
  // so 8-row items get their ~230 registers (measured: 4 warps also beat 8 for 4-row items)
  static constexpr int CW = 4;
  static constexpr int THREADS = (CW + 1) * 32;
};

template <int KP>
constexpr size_t spmm_smem_bytes() {
  return (size_t)SpRows<KP>::STAGES * (SpRows<KP>::R + 1) * SpRows<KP>::CH * 4 +
         SpRows<KP>::CW * SpRows<KP>::R * SP_KPMAX * 4 + 2 * SpRows<KP>::STAGES * 8 + 64;
}

// Spart[(s * rows_pad + i) * k + c0 + c] for clusters c0 .. c0 + KP - 1 (c0 + c < k).
template <int KP>
__global__ void __launch_bounds__(SpRows<KP>::THREADS, 1)
    spmm_onehot_kernel(const float *__restrict__ K, int64_t ldk, int64_t nrows,
                       const int32_t *__restrict__ labels, int k, int c0, int nsplit,
                       int chunks_per_split, int64_t rows_pad, double *__restrict__ Spart) {
  constexpr int SP_ROWS = SpRows<KP>::R;
  constexpr int SP_STAGES = SpRows<KP>::STAGES;
  constexpr int SP_CWARPS = SpRows<KP>::CW;
  constexpr int SP_CH = SpRows<KP>::CH;
  extern __shared__ __align__(128) uint8_t smem[];
  float *ring = reinterpret_cast<float *>(smem);  // [STAGES][ROWS + 1][CH]
  float *red = ring + (size_t)SP_STAGES * (SP_ROWS + 1) * SP_CH;  // [CWARPS][ROWS][KPMAX]
  uint64_t *full = reinterpret_cast<uint64_t *>(red + SP_CWARPS * SP_ROWS * SP_KPMAX);
  uint64_t *empty = full + SP_STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (ldk + SP_CH - 1) / SP_CH;
  const int64_t ngroups = (nrows + SP_ROWS - 1) / SP_ROWS;
  const int64_t nitems = ngroups * nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SP_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SP_CWARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0;
  if (warp == SP_CWARPS) {
    // ---------------- producer: one elected lane issues the bulk copies
    if (lane == 0) {
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int64_t g = item / nsplit;
        const int s = (int)(item % nsplit);
        const int64_t q0 = (int64_t)s * chunks_per_split;
        const int64_t q1 = q0 + chunks_per_split < nchunks ? q0 + chunks_per_split : nchunks;
        const int64_t r0 = g * SP_ROWS;
        const int nr = (int)(nrows - r0 < SP_ROWS ? nrows - r0 : SP_ROWS);
        for (int64_t q = q0; q < q1; ++q) {
          const int64_t col0 = q * SP_CH;
          const uint32_t cols = (uint32_t)(ldk - col0 < SP_CH ? ldk - col0 : SP_CH);
          mbar_wait(&empty[stage], phase ^ 1);
          float *st = ring + (size_t)stage * (SP_ROWS + 1) * SP_CH;
          mbar_arrive_expect_tx(&full[stage], (uint32_t)(nr + 1) * cols * 4u);
          bulk_g2s(st + SP_ROWS * SP_CH, labels + col0, cols * 4u, &full[stage]);
          for (int r = 0; r < nr; ++r)
            bulk_g2s(st + r * SP_CH, K + (r0 + r) * ldk + col0, cols * 4u, &full[stage]);
          if (++stage == SP_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int64_t g = item / nsplit;
    const int s = (int)(item % nsplit);
    const int64_t q0 = (int64_t)s * chunks_per_split;
    const int64_t q1 = q0 + chunks_per_split < nchunks ? q0 + chunks_per_split : nchunks;
    float2 acc[SP_ROWS][KP];
#pragma unroll
    for (int r = 0; r < SP_ROWS; ++r)
#pragma unroll
      for (int c = 0; c < KP; ++c) acc[r][c] = make_float2(0.f, 0.f);

    for (int64_t q = q0; q < q1; ++q) {
      const int64_t col0 = q * SP_CH;
      const int cols = (int)(ldk - col0 < SP_CH ? ldk - col0 : SP_CH);
      mbar_wait(&full[stage], phase);
      const float *st = ring + (size_t)stage * (SP_ROWS + 1) * SP_CH;
      const int4 *lab4 = reinterpret_cast<const int4 *>(st + SP_ROWS * SP_CH);
      const int nquads = cols >> 2;
      for (int v = warp * 32 + lane; v < nquads; v += SP_CWARPS * 32) {
        const int4 l = lab4[v];
        float4 x[SP_ROWS];
#pragma unroll
        for (int r = 0; r < SP_ROWS; ++r) x[r] = reinterpret_cast<const float4 *>(st + r * SP_CH)[v];
#pragma unroll
        for (int c = 0; c < KP; ++c) {
          const int cc = c0 + c;
          const float m0 = mask_eq(l.x, cc), m1 = mask_eq(l.y, cc);
          const float m2 = mask_eq(l.z, cc), m3 = mask_eq(l.w, cc);
          // the two updates of acc[r][c] are SP_ROWS instructions apart (FFMA2 latency)
#pragma unroll
          for (int r = 0; r < SP_ROWS; ++r) ffma2(acc[r][c], x[r].x, x[r].y, m0, m1);
#pragma unroll
          for (int r = 0; r < SP_ROWS; ++r) ffma2(acc[r][c], x[r].z, x[r].w, m2, m3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == SP_STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    // ---- fixed-order reduction: lanes (shuffle tree, fp32) then warps (fp64)
#pragma unroll
    for (int r = 0; r < SP_ROWS; ++r)
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        float v = warp_sum(acc[r][c].x + acc[r][c].y);
        if (lane == 0) red[(warp * SP_ROWS + r) * SP_KPMAX + c] = v;
      }
    asm volatile("bar.sync 1, %0;" ::"n"(SP_CWARPS * 32));
    const int64_t r0 = g * SP_ROWS;
    for (int t = threadIdx.x; t < SP_ROWS * KP; t += SP_CWARPS * 32) {
      const int r = t / KP, c = t % KP;
      if (r0 + r < nrows && c0 + c < k) {
        double sum = 0.0;
        for (int w = 0; w < SP_CWARPS; ++w) sum += (double)red[(w * SP_ROWS + r) * SP_KPMAX + c];
        Spart[((int64_t)s * rows_pad + r0 + r) * k + c0 + c] = sum;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(SP_CWARPS * 32));
  }
}

}  // namespace kkm

namespace kkm {

// labB[t] = labels[t] for t < nB, -1 on [nB, len): the B set's labels at the K-tile pitch.
__global__ void copy_labels_kernel(const int32_t *__restrict__ labels, int64_t nB, int64_t len,
                                   int32_t *__restrict__ labB) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < len) labB[t] = t < nB ? labels[t] : -1;
}

// 1.5D: out[t] = sum over the pr pieces of the column in rank order, piece gi from the own Scol,
// the others from the received buffer (rbuf[ip * bk + t]).
__global__ void column_sum_kernel(const double *__restrict__ Scol, const double *__restrict__ rbuf, int pr, int gi,
                                  int64_t bk, double *__restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= bk) return;
  double s = 0.0;
  for (int ip = 0; ip < pr; ++ip) s += ip == gi ? Scol[(int64_t)gi * bk + t] : rbuf[(int64_t)ip * bk + t];
  out[t] = s;
}

// Scol[r][c] = sum_s Spart[s][r][c] (fixed order) for r < nA, 0 on [nA, rows_pad).
__global__ void split_sum_kernel(const double *__restrict__ Spart, int nsplit, int64_t nA, int64_t rows_pad,
                                 int k, double *__restrict__ Scol) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows_pad * k) return;
  const int64_t r = t / k;
  double s = 0.0;
  if (r < nA)
    for (int p = 0; p < nsplit; ++p) s += Spart[(int64_t)p * rows_pad * k + t];
  Scol[t] = s;
}

}  // namespace kkm

// =====================================================================================
// SpMM v2: label-sorted 32-column groups (k-independent, ~0.5 instructions per element).
//
// Once per iteration `group_code_kernel` stably sorts every aligned group of 32 columns by
// label (one warp per group) and packs, for each sorted position p of group g,
//   code[32 g + p] = src | lab << 8 | rem << 16 | head << 24
// src = the group lane holding that column, lab = its label (255 for padding columns),
// rem = positions left in its label segment after p, head = p starts a segment. The consumer
// reads K[i][32 g + src] (a permutation of 32 consecutive words: conflict-free), reduces each
// segment with a 5-step (or fewer, warp-uniform) shfl_down suffix scan limited by rem, and the
// segment-head lanes add the segment sums to fp64 shared-memory accumulators acc[row][lab].
// =====================================================================================
namespace kkm {

constexpr int SG_ROWS = 8;        // rows per work item
constexpr int SG_CH = 1024;       // columns per chunk
constexpr int SG_STAGES = 4;
constexpr int SG_CWARPS = 16;
constexpr int SG_THREADS = (SG_CWARPS + 1) * 32;
constexpr int SG_MAX_K = 64;
constexpr int SG_MAX_CHUNKS_PER_SPLIT = 256;  // fp64 accumulators: splits only for balance

inline size_t sg_smem_bytes(int k) {
  return (size_t)SG_STAGES * (SG_ROWS + 1) * SG_CH * 4 + (size_t)SG_CWARPS * SG_ROWS * k * 8 +
         2 * SG_STAGES * 8 + 64;
}

// One warp per 32-column group of [0, len); labels beyond nB are padding (lab 255).
__global__ void group_code_kernel(const int32_t *__restrict__ labels, int64_t nB, int64_t len,
                                  uint32_t *__restrict__ codes) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g * 32 >= len) return;
  const int64_t col = g * 32 + lane;
  const int L = col < nB ? labels[col] : 255;
  const unsigned eq = __match_any_sync(0xffffffffu, L);
  const int within = __popc(eq & ((1u << lane) - 1u));
  int less = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) less += __shfl_sync(0xffffffffu, L, j) < L;
  const int rank = less + within;
  const int rem = less + __popc(eq) - 1 - rank;
  const uint32_t code = (uint32_t)lane | ((uint32_t)L << 8) | ((uint32_t)rem << 16) | ((uint32_t)(within == 0) << 24);
  codes[g * 32 + rank] = code;
}

// Spart[(s * rows_pad + i) * k + c] = sum over the split's columns j with cl_j = c of K[i][j].
__global__ void __launch_bounds__(SG_THREADS, 1)
    spmm_group_kernel(const float *__restrict__ K, int64_t ldk, int64_t nrows,
                      const uint32_t *__restrict__ codes, int k, int nsplit, int chunks_per_split,
                      int64_t rows_pad, double *__restrict__ Spart) {
  extern __shared__ __align__(128) uint8_t smem[];
  float *ring = reinterpret_cast<float *>(smem);  // [STAGES][ROWS + 1][CH] (last row: codes)
  double *acc = reinterpret_cast<double *>(ring + (size_t)SG_STAGES * (SG_ROWS + 1) * SG_CH);  // [CWARPS][ROWS][k]
  uint64_t *full = reinterpret_cast<uint64_t *>(acc + SG_CWARPS * SG_ROWS * k);
  uint64_t *empty = full + SG_STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (ldk + SG_CH - 1) / SG_CH;
  const int64_t ngroups = (nrows + SG_ROWS - 1) / SG_ROWS;
  const int64_t nitems = ngroups * nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SG_CWARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0;
  if (warp == SG_CWARPS) {
    if (lane == 0) {
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int64_t gi = item / nsplit;
        const int s = (int)(item % nsplit);
        const int64_t q0 = (int64_t)s * chunks_per_split;
        const int64_t q1 = q0 + chunks_per_split < nchunks ? q0 + chunks_per_split : nchunks;
        const int64_t r0 = gi * SG_ROWS;
        const int nr = (int)(nrows - r0 < SG_ROWS ? nrows - r0 : SG_ROWS);
        for (int64_t q = q0; q < q1; ++q) {
          const int64_t col0 = q * SG_CH;
          const uint32_t cols = (uint32_t)(ldk - col0 < SG_CH ? ldk - col0 : SG_CH);
          mbar_wait(&empty[stage], phase ^ 1);
          float *st = ring + (size_t)stage * (SG_ROWS + 1) * SG_CH;
          mbar_arrive_expect_tx(&full[stage], (uint32_t)(nr + 1) * cols * 4u);
          bulk_g2s(st + SG_ROWS * SG_CH, codes + col0, cols * 4u, &full[stage]);
          for (int r = 0; r < nr; ++r)
            bulk_g2s(st + r * SG_CH, K + (r0 + r) * ldk + col0, cols * 4u, &full[stage]);
          if (++stage == SG_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  double *wacc = acc + (size_t)warp * SG_ROWS * k;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int64_t gi = item / nsplit;
    const int s = (int)(item % nsplit);
    const int64_t q0 = (int64_t)s * chunks_per_split;
    const int64_t q1 = q0 + chunks_per_split < nchunks ? q0 + chunks_per_split : nchunks;
    for (int t = lane; t < SG_ROWS * k; t += 32) wacc[t] = 0.0;
    __syncwarp();
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t col0 = q * SG_CH;
      const int cols = (int)(ldk - col0 < SG_CH ? ldk - col0 : SG_CH);
      mbar_wait(&full[stage], phase);
      const float *st = ring + (size_t)stage * (SG_ROWS + 1) * SG_CH;
      const uint32_t *cd = reinterpret_cast<const uint32_t *>(st + SG_ROWS * SG_CH);
      for (int g = warp; g < (cols >> 5); g += SG_CWARPS) {
        const uint32_t code = cd[g * 32 + lane];
        const int src = (int)(code & 0xFFu), lab = (int)((code >> 8) & 0xFFu);
        const int rem = (int)((code >> 16) & 0xFFu);
        const bool head = (code >> 24) != 0u && lab < k;
        // warp-uniform number of scan steps: enough for the group's longest segment
        const int maxrem = __reduce_max_sync(0xffffffffu, (unsigned)rem);
        const int steps = 32 - __clz(maxrem);  // ceil(log2(maxrem + 1))
        const float *colp = st + g * 32 + src;
        float v[SG_ROWS];
#pragma unroll
        for (int r = 0; r < SG_ROWS; ++r) v[r] = colp[r * SG_CH];
        // segmented suffix scan, the 8 rows interleaved so their shuffles overlap
#pragma unroll
        for (int o = 1, st_ = 0; o < 32; o <<= 1, ++st_) {
          if (st_ < steps) {
            float t[SG_ROWS];
#pragma unroll
            for (int r = 0; r < SG_ROWS; ++r) t[r] = __shfl_down_sync(0xffffffffu, v[r], o);
            if (o <= rem) {
#pragma unroll
              for (int r = 0; r < SG_ROWS; ++r) v[r] += t[r];
            }
          }
        }
        if (head) {
#pragma unroll
          for (int r = 0; r < SG_ROWS; ++r) wacc[r * k + lab] += (double)v[r];
        }
        __syncwarp();  // order this group's accumulator updates before the next group's
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == SG_STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(SG_CWARPS * 32));
    const int64_t r0 = gi * SG_ROWS;
    for (int t = threadIdx.x; t < SG_ROWS * k; t += SG_CWARPS * 32) {
      const int r = t / k, c = t % k;
      if (r0 + r < nrows) {
        double sum = 0.0;
        for (int w = 0; w < SG_CWARPS; ++w) sum += acc[((size_t)w * SG_ROWS + r) * k + c];
        Spart[((int64_t)s * rows_pad + r0 + r) * k + c] = sum;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(SG_CWARPS * 32));
  }
}

}  // namespace kkm
