// sym.cuh -- f1: a2 over a materialised K that stores only its upper triangle.
// K is symmetric, so S(i, c) = sum_{j: cl(j) = c} K(i, j) splits, for i in band I
// (rows [I TB, (I+1) TB)), into
//   row part:    sum over the stored columns j >= I TB of band I (the diagonal tile K_II is
//                stored whole), by the labels of the columns;
//   column part: sum over the bands I' < I of K(i', i) = K(i, i') for i' in band I', by the
//                labels of the ROWS i' -- i.e. label-segmented column sums of band I'.
// Band I is stored row-major, TB rows x ldb_I = ceil32(n - I TB) columns (column 0 = point
// I TB), written once by the a1 GEMM (one launch per band): ~n^2/2 floats instead of n^2.
//
// Per iteration:
//   band_sort:  per band, a stable counting sort of its rows by label, cut into row groups of
//               at most R rows that never straddle a label (so a group has ONE label);
//   spmm_sym:   the one-hot FFMA2 mainloop of spmm_onehot_kernel (spmm.cuh) over (band, group,
//               column split) items -- rows fetched in sorted order by per-row bulk copies --
//               plus, per 4-column quad, the group's column sum (one float4 store per R x 4
//               block, skipped on the diagonal tile): +1/R of the K bytes written as partials;
//   sym_colsum: per band, stored column and label, the fp64 sum of that label's group partials;
//   sym_reduce: S(i, :) = row partials (fp64 over splits) + the column sums of every owned band
//               I' < band(i), in fixed order.
// All sums fixed-order: bitwise reproducible.
#pragma once
#include "common.cuh"
#include "spmm.cuh"

namespace kkm {

constexpr int SYM_TB = 1024;  // band height (rows) = width of the diagonal tile

// One owned band.
struct SymBand {
  int64_t koff;    // float offset of the band in the K buffer
  int64_t cpoff;   // float offset of the band's column partials ([G_max][ldb - TB])
  int64_t item0;   // first work item of the band
  int64_t csoff;   // double offset of the band's per-label column sums ([k][ldb - TB])
  int32_t band;    // band index I
  int32_t ldb;     // stored columns (row pitch), ceil32(n - I TB)
  int32_t nsplit;  // column splits of the band
  int32_t cps;     // chunks per split
  int32_t row0;    // 16-bit storage (spmm_tc): first row of a 512-row piece of the band; else 0
  int32_t rows;    // stored rows
};

// Row group descriptor: sorted positions [p0, p0 + cnt) of the band, all with label lab.
struct SymGroup {
  int32_t p0, cnt, lab, pad;
};

// spmm_sym_kernel shape: R = 8 rows per group; 8 consumer warps = 2 cluster halves (KP/2
// clusters each, so 2 R KP/2 accumulator registers) x 4 column quarters, + 1 producer warp.
// Two consumer warps per SM sub-partition hide each other's dependency stalls (with one,
// the kernel was latency bound at ~38 % issue and 64 % of HBM bandwidth).
constexpr int SYM_R = 8;
constexpr int SYM_CW = 8;
constexpr int SYM_STAGES = 3;
constexpr int SYM_CH = 2048;
constexpr int SYM_THREADS = (SYM_CW + 1) * 32;
inline int sym_rows(int) { return SYM_R; }
inline int sym_gmax(int k) { return SYM_TB / SYM_R + k; }

// grid: one CTA of SYM_TB threads per band (all bands). perm[I TB + p] = band-local row at
// sorted position p (stable); groups[I][g], ngroups[I], gfirst[I][c]. Rows beyond n are
// left out.
__global__ void __launch_bounds__(SYM_TB) band_sort_kernel(const int32_t *__restrict__ labels, int64_t n, int k,
                                                           int R, int gmax, int32_t *__restrict__ perm,
                                                           SymGroup *__restrict__ groups,
                                                           int32_t *__restrict__ ngroups,
                                                           int32_t *__restrict__ gfirst) {
  extern __shared__ int32_t sm[];
  int32_t *wcnt = sm;                   // [32 warps][k]
  int32_t *seg = sm + 32 * k;           // [k + 1] segment starts
  int32_t *gst = seg + k + 1;           // [k + 1] first group of each label
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t I = blockIdx.x;
  const int64_t row = I * SYM_TB + t;
  const int l = row < n ? labels[row] : -1;
  for (int i = t; i < 32 * k; i += SYM_TB) wcnt[i] = 0;
  __syncthreads();
  unsigned same = __match_any_sync(0xffffffffu, l);
  const int rank_in_warp = __popc(same & ((1u << lane) - 1u));
  if (l >= 0 && rank_in_warp == 0) wcnt[warp * k + l] = __popc(same);
  __syncthreads();
  if (t < k) {  // exclusive prefix over warps of label t; total into seg
    int s = 0;
    for (int w = 0; w < 32; ++w) {
      const int c = wcnt[w * k + t];
      wcnt[w * k + t] = s;
      s += c;
    }
    seg[t + 1] = s;
  }
  __syncthreads();
  if (t == 0) {
    seg[0] = 0;
    gst[0] = 0;
    for (int c = 0; c < k; ++c) {
      const int cnt = seg[c + 1];
      seg[c + 1] = seg[c] + cnt;
      gst[c + 1] = gst[c] + (cnt + R - 1) / R;
    }
    ngroups[I] = gst[k];
  }
  __syncthreads();
  if (t <= k) gfirst[I * (k + 1) + t] = gst[t];  // groups of label c: [gfirst[c], gfirst[c+1])
  if (l >= 0) perm[I * SYM_TB + seg[l] + wcnt[warp * k + l] + rank_in_warp] = t;
  // groups of label c: [gst[c], gst[c+1]), R rows each (the last one of a label shorter)
  for (int g = t; g < gmax; g += SYM_TB) {
    SymGroup gr{0, 0, 0, 0};
    if (g < gst[k]) {
      int c = 0;
      while (g >= gst[c + 1]) ++c;
      const int p0 = seg[c] + (g - gst[c]) * R;
      gr.p0 = p0;
      gr.cnt = min(R, seg[c + 1] - p0);
      gr.lab = c;
    }
    groups[I * gmax + g] = gr;
  }
}

// Items: for each owned band b (bands[b]), gmax groups x nsplit splits (empty groups skipped).
// Spart[(s * rows_pad + row) * k + c] (fp64) for the group's rows, s < bands[b].nsplit;
// colpart[cpoff + g * (ldb - TB) + (col - TB)] (fp32) for the stored columns col >= TB.
// work[0] (next item), work[1] (CTAs past the end): zero between launches (reset at the end).
template <int KP>
__global__ void __launch_bounds__(SYM_THREADS, 1)
    spmm_sym_kernel(const float *__restrict__ K, const SymBand *__restrict__ bands, int nbands, int64_t nitems,
                    const int32_t *__restrict__ labels, const int32_t *__restrict__ perm,
                    const SymGroup *__restrict__ groups, int gmax, int k, int64_t rows_pad,
                    double *__restrict__ Spart, float *__restrict__ colpart, int32_t *__restrict__ work) {
  constexpr int R = SYM_R, STAGES = SYM_STAGES, CW = SYM_CW, CH = SYM_CH;
  constexpr int KH = KP / 2;  // clusters per half
  extern __shared__ __align__(128) uint8_t smem[];
  float *ring = reinterpret_cast<float *>(smem);              // [STAGES][R + 1][CH]
  float *red = ring + (size_t)STAGES * (R + 1) * CH;          // [CW][R][KH]
  uint64_t *full = reinterpret_cast<uint64_t *>(red + CW * R * (SP_KPMAX / 2));
  uint64_t *empty = full + STAGES;
  __shared__ int4 s_item[STAGES];  // (band b, group g, split s) of a stage's item; b < 0: no more items
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // item -> (band b, group g, split s)
  auto decode = [&](int64_t item, int &b, int &g, int &s) {
    int lo = 0, hi = nbands - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (bands[mid].item0 <= item) lo = mid;
      else hi = mid - 1;
    }
    b = lo;
    const int64_t li = item - bands[b].item0;
    g = (int)(li / bands[b].nsplit);
    s = (int)(li % bands[b].nsplit);
  };

  int stage = 0;
  uint32_t phase = 0;
  if (warp == CW) {
    if (lane == 0) {
      // dynamic item scheduling: items are taken in order (largest bands first) by whichever
      // CTA is free (static round-robin left SMs idle at the end: a2 kernel 1.33 -> 1.26 ms)
      for (;;) {
        const int64_t item = atomicAdd(work, 1);
        if (item >= nitems) break;
        int b, g, s;
        decode(item, b, g, s);
        const SymBand bd = bands[b];
        const SymGroup gr = groups[(int64_t)bd.band * gmax + g];
        if (gr.cnt == 0) continue;
        const int nchunks = (bd.ldb + CH - 1) / CH;
        const int q0 = s * bd.cps;
        const int q1 = q0 + bd.cps < nchunks ? q0 + bd.cps : nchunks;
        const int32_t *pr = perm + (int64_t)bd.band * SYM_TB + gr.p0;
        const float *Kb = K + bd.koff;
        const int32_t *lab = labels + (int64_t)bd.band * SYM_TB;
        int64_t roff[R];
#pragma unroll
        for (int r = 0; r < R; ++r) roff[r] = r < gr.cnt ? (int64_t)pr[r] * bd.ldb : 0;
        for (int q = q0; q < q1; ++q) {
          const int col0 = q * CH;
          const uint32_t cols = (uint32_t)(bd.ldb - col0 < CH ? bd.ldb - col0 : CH);
          mbar_wait(&empty[stage], phase ^ 1);
          float *st = ring + (size_t)stage * (R + 1) * CH;
          s_item[stage] = make_int4(b, g, s, 0);
          mbar_arrive_expect_tx(&full[stage], (uint32_t)(gr.cnt + 1) * cols * 4u);
          bulk_g2s(st + R * CH, lab + col0, cols * 4u, &full[stage]);
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < gr.cnt) bulk_g2s(st + r * CH, Kb + roff[r] + col0, cols * 4u, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      mbar_wait(&empty[stage], phase ^ 1);  // end marker for the consumers
      s_item[stage] = make_int4(-1, 0, 0, 0);
      mbar_arrive(&full[stage]);
      // the last CTA past the end resets the scheduler for the next launch
      if (atomicAdd(work + 1, 1) == (int)gridDim.x - 1) {
        work[0] = 0;
        work[1] = 0;
      }
    }
    return;
  }

  const int half = warp >> 2, quarter = warp & 3;
  const int cbase = half * KH;
  for (;;) {
    mbar_wait(&full[stage], phase);  // the item's first stage (or the end marker)
    const int4 it = s_item[stage];
    if (it.x < 0) break;
    const int b = it.x, g = it.y, s = it.z;
    const int band = bands[b].band, ldb = bands[b].ldb, cps = bands[b].cps;
    const int nr = groups[(int64_t)band * gmax + g].cnt;
    const int nchunks = (ldb + CH - 1) / CH;
    const int q0 = s * cps;
    const int q1 = q0 + cps < nchunks ? q0 + cps : nchunks;
    float *cp = colpart + bands[b].cpoff + (int64_t)g * (ldb - SYM_TB) - SYM_TB;  // indexed by band column
    float2 acc[R][KH];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < KH; ++c) acc[r][c] = make_float2(0.f, 0.f);

    for (int q = q0; q < q1; ++q) {
      const int col0 = q * CH;
      const int cols = ldb - col0 < CH ? ldb - col0 : CH;
      mbar_wait(&full[stage], phase);
      const float *st = ring + (size_t)stage * (R + 1) * CH;
      const int4 *lab4 = reinterpret_cast<const int4 *>(st + R * CH);
      const int nquads = cols >> 2;
      // the column sums alternate between the cluster halves by (warp-uniform) quad step, so
      // both halves carry the same work
      int step = q;
      for (int v = quarter * 32 + lane; v < nquads; v += 4 * 32, ++step) {
        const bool colsums = (step & 1) == half;
        const int4 l = lab4[v];
        float4 x[R];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = reinterpret_cast<const float4 *>(st + r * CH)[v];
        const int colb = col0 + 4 * v;  // band column of the quad
        if (colsums && colb >= SYM_TB) {  // column part (not on the diagonal tile)
          float2 s01 = make_float2(x[0].x, x[0].y), s23 = make_float2(x[0].z, x[0].w);
          if (nr == R) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
              s01 = f2add(s01, make_float2(x[r].x, x[r].y));
              s23 = f2add(s23, make_float2(x[r].z, x[r].w));
            }
          } else {  // rows >= nr of the stage are stale (static indices: x stays in registers)
#pragma unroll
            for (int r = 1; r < R; ++r)
              if (r < nr) {
                s01 = f2add(s01, make_float2(x[r].x, x[r].y));
                s23 = f2add(s23, make_float2(x[r].z, x[r].w));
              }
          }
          __stcs(reinterpret_cast<float4 *>(cp + colb), make_float4(s01.x, s01.y, s23.x, s23.y));
        }
#pragma unroll
        for (int c = 0; c < KH; ++c) {
          const int cc = cbase + c;
          const float m0 = mask_eq(l.x, cc), m1 = mask_eq(l.y, cc);
          const float m2 = mask_eq(l.z, cc), m3 = mask_eq(l.w, cc);
#pragma unroll
          for (int r = 0; r < R; ++r) ffma2(acc[r][c], x[r].x, x[r].y, m0, m1);
#pragma unroll
          for (int r = 0; r < R; ++r) ffma2(acc[r][c], x[r].z, x[r].w, m2, m3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    // fixed-order reduction: lanes (shuffle tree, fp32), then the 4 column quarters (fp64)
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < KH; ++c) {
        float v = warp_sum(acc[r][c].x + acc[r][c].y);
        if (lane == 0) red[(warp * R + r) * KH + c] = v;
      }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
    const int32_t *pr = perm + (int64_t)band * SYM_TB + groups[(int64_t)band * gmax + g].p0;
    for (int t = threadIdx.x; t < R * KP; t += CW * 32) {
      const int r = t / KP, c = t % KP;
      if (r < nr && c < k) {
        const int h = c / KH, cl = c % KH;
        double sum = 0.0;
        for (int w = 0; w < 4; ++w) sum += (double)red[((h * 4 + w) * R + r) * KH + cl];
        const int64_t row = (int64_t)band * SYM_TB + pr[r];
        Spart[((int64_t)s * rows_pad + row) * k + c] = sum;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
  }
}

constexpr size_t spmm_sym_smem_bytes() {
  return (size_t)SYM_STAGES * (SYM_R + 1) * SYM_CH * 4 + SYM_CW * SYM_R * (SP_KPMAX / 2) * 4 + 2 * SYM_STAGES * 8 + 64;
}

// Column part, step 1: per owned band (blockIdx.y), label c (blockIdx.z) and 4 stored
// off-diagonal columns j .. j+3 (thread; w = ldb - TB is a multiple of 32), the fp64 sum over
// the band's row groups of label c (a contiguous range, gfirst) in order:
// colsum[csoff + c * w + j] (0 if the band has no rows of label c).
__global__ void sym_colsum_kernel(const float *__restrict__ colpart, const SymBand *__restrict__ bands,
                                  const int32_t *__restrict__ gfirst, int k, double *__restrict__ colsum) {
  const SymBand bd = bands[blockIdx.y];
  const int64_t w = bd.ldb - SYM_TB;
  const int64_t j = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (j >= w) return;
  const int c = blockIdx.z;
  const int g0 = gfirst[bd.band * (k + 1) + c], g1 = gfirst[bd.band * (k + 1) + c + 1];
  const float *cp = colpart + bd.cpoff + j;
  double r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
#pragma unroll 4
  for (int g = g0; g < g1; ++g) {
    const float4 v = __ldcs(reinterpret_cast<const float4 *>(cp + (int64_t)g * w));
    r0 += (double)v.x;
    r1 += (double)v.y;
    r2 += (double)v.z;
    r3 += (double)v.w;
  }
  double *o = colsum + bd.csoff + (int64_t)c * w + j;
  o[0] = r0;
  o[1] = r1;
  o[2] = r2;
  o[3] = r3;
}

// Step 2, one thread per (row i < rows_pad, label c = blockIdx.y); rows >= n get zeros.
// band_desc[I] = index of band I in `bands` if owned, else -1. S[i][c] (fp64) = this rank's
// contributions to S(i, c): the row partials of its own band (splits in order) + the column
// sums of the owned bands I' < band(i) (in order).
__global__ void sym_reduce_kernel(const double *__restrict__ Spart, const double *__restrict__ colsum,
                                  const SymBand *__restrict__ bands, const int32_t *__restrict__ band_desc,
                                  int64_t n, int64_t rows_pad, int k, double *__restrict__ S) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= rows_pad) return;
  double acc = 0.0;
  if (i < n) {
    const int I = (int)(i / SYM_TB);
    const int bi = band_desc[I];
    if (bi >= 0)
      for (int s = 0; s < bands[bi].nsplit; ++s) acc += Spart[((int64_t)s * rows_pad + i) * k + c];
    for (int Ip = 0; Ip < I; ++Ip) {
      const int bp = band_desc[Ip];
      if (bp < 0) continue;
      const int64_t w = bands[bp].ldb - SYM_TB;
      acc += colsum[bands[bp].csoff + (int64_t)c * w + (i - (int64_t)Ip * SYM_TB - SYM_TB)];
    }
  }
  S[i * k + c] = acc;
}

}  // namespace kkm

namespace kkm {

// ---- f1 on the streaming path (tc2_stream_sym_kernel): exact int64 fixed-point S.
// max over the n rows of norms[] (one CTA) -> *out.
__global__ void max_norm_kernel(const float *__restrict__ norms, int64_t n, float *__restrict__ out) {
  __shared__ float red[32];
  float m = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, norms[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
  }
}

// Original order: Sorig[i][c] = Sfix[pos[i]][c] for i < n, 0 on [n, rows) (int64, exact);
// if Sd != NULL also Sd[i][c] = Sorig * inv_scale (fp64).
__global__ void fx_unpermute_kernel(const long long *__restrict__ Sfix, const int32_t *__restrict__ pos, int64_t n,
                                    int64_t rows, int k, double inv_scale, long long *__restrict__ Sorig,
                                    double *__restrict__ Sd) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * k) return;
  const int64_t i = t / k;
  const int c = (int)(t % k);
  const long long v = i < n ? Sfix[(int64_t)pos[i] * k + c] : 0ll;
  if (Sorig) Sorig[t] = v;
  if (Sd) Sd[t] = (double)v * inv_scale;
}

__global__ void fx_to_double_kernel(const long long *__restrict__ S, int64_t count, double inv_scale,
                                    double *__restrict__ Sd) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) Sd[t] = (double)S[t] * inv_scale;
}

}  // namespace kkm
