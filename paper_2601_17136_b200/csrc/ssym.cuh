// ssym.cuh -- f1 on the streaming path: the upper triangle of the label-sorted K, recomputed per
// iteration on CTA pairs (the tc2.cuh mainloop) and reduced in the epilogue; K is never stored.
//
// A = B = the label-sorted points (sort.cuh), so the sorted K is symmetric and only pair
// tiles (tm, tn >= tm) are computed. Every tile adds
//   row part:    S(p, c) += sum_{q in tile, q in segment c} K(p, q)            (Eq. e)
//   column part: S(q, r) += sum_{p in tile, p in segment r} K(p, q)   (tn > tm; K(p,q) = K(q,p))
// in int64 fixed point (value x 2^s with n max K_ii 2^s < 2^61; red.add: integer addition is
// associative, so S is bitwise independent of the order, the grid and the rank count).
//
// Epilogue (16 warps: 4 TMEM lane quarters x 4 column quarters of 64; thread = row):
//  1. drain: the tile's main + correction accumulators (64 + 64 columns per thread) are read from
//     TMEM and summed into 64 registers, then TMEM goes straight back to the MMA warp -- the only
//     part of the epilogue serial with the tensor core (single-buffered TMEM: the fp16x3
//     correction accumulator fills the second half);
//  2. per 32-column chunk, overlapped with the next tile's MMAs: kappa (Eqs. b, k; A1/A23), the row
//     part as ONE running fp64 sum per thread that is flushed (one red.add) whenever the column
//     segment changes -- columns are label-sorted, so a row sweeps its unit's columns segment
//     after segment and no per-cluster register array is needed (any k); the column part by a
//     31-shuffle reduce-scatter butterfly over the warp's 32 rows (one label, almost always) and
//     one red.add per column; a warp whose rows straddle a segment boundary (<= k - 1 of them)
//     adds its elements one by one.
// Work units (tm, tn0, ntn) cover the upper triangle in aligned blocks of column tiles; the host
// orders a rank's units block-major, so the ~74 pairs running at once sweep the SAME block of B
// tiles (L2-resident) with different row tiles.
#pragma once
#include "tc2.cuh"

namespace kkm {

constexpr int SS_EPI_WARPS = 16;
constexpr int SS_THREADS = (2 + SS_EPI_WARPS) * 32;
constexpr int SS_COLS = 64;  // columns per epilogue warp
constexpr size_t SS_COLC_BYTES = 2 * SS_COLS * 4;  // per warp: norms + rscale of its 64 columns
constexpr size_t SS_SEG_BYTES = (size_t)(KKM_MAX_K + 1) * 4;
constexpr size_t SS_EXTRA = SS_EPI_WARPS * SS_COLC_BYTES + (SS_SEG_BYTES + 15) / 16 * 16;
constexpr size_t SS_SMEM = (size_t)T2_STAGES * T2_STAGE_BYTES + SS_EXTRA + 1024 + 128;

// Per-column constants of columns [j, j + 64) into cn[0..64) (norms) / cn[64..128) (rscale).
__device__ __forceinline__ void ss_stage_columns(float *cn, const float *__restrict__ norms,
                                                 const float *__restrict__ rscale, int64_t j, int64_t nvalid,
                                                 bool need_norm, int lane) {
  const int64_t p0 = j + 2 * lane;
  float2 nv = make_float2(0.f, 0.f), rv = make_float2(1.f, 1.f);
  if (p0 < nvalid) {
    if (need_norm) nv.x = __ldg(norms + p0);
    if (rscale) rv.x = __ldg(rscale + p0);
  }
  if (p0 + 1 < nvalid) {
    if (need_norm) nv.y = __ldg(norms + p0 + 1);
    if (rscale) rv.y = __ldg(rscale + p0 + 1);
  }
  __syncwarp();
  reinterpret_cast<float2 *>(cn)[lane] = nv;
  reinterpret_cast<float2 *>(cn + SS_COLS)[lane] = rv;
  __syncwarp();
}

// Last segment c in [0, k) with seg[c] <= p (seg[0] = 0 <= p).
__device__ __forceinline__ int ss_segment_of(const int32_t *seg, int k, int64_t p) {
  int lo = 0, hi = k - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid] <= p) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ long long ss_fix(double v, double fx) { return __double2ll_rn(v * fx); }

// One 32-column chunk of a tile (columns p0 .. p0 + 31, this thread's row p): kappa, the row part
// into the running sum (flushed on a segment change), the column part (off-diagonal tiles).
// cn: the chunk's column norms at cn[0..32) and rscale at cn[SS_COLS..SS_COLS + 32).
__device__ __forceinline__ void ss_chunk(float (&x)[32], int64_t p0, const float *cn, const KappaParams &kp,
                                         const RowK &rk, bool diag, int64_t p, bool row_ok, int64_t n,
                                         const int32_t *seg, int k, int &cseg, int &cur, double &run, int r0, int r1,
                                         int mylab, int lane, double fx_scale, long long *__restrict__ Sfix) {
  if (p0 >= n) return;
  kappa_chunk_sum(x, cn, cn + SS_COLS, kp, rk);
  if (diag && kp.kind == 2 && p >= p0 && p < p0 + 32) {  // kappa(x_p, x_p) = 1 exactly (A1)
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (p0 + q == p) x[q] = 1.f;
  }
  if (p0 + 32 > n) {
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (p0 + q >= n) x[q] = 0.f;
  }
  if (!row_ok) {
#pragma unroll
    for (int q = 0; q < 32; ++q) x[q] = 0.f;
  }
  // row part: the chunk's columns are segments c0 .. c1 (the warp's pointer only moves forward)
  const int64_t p1 = p0 + 31 < n ? p0 + 31 : n - 1;
  while (cseg + 1 < k && seg[cseg + 1] <= p0) ++cseg;
  const int c0 = cseg;
  int c1 = c0;
  while (c1 + 1 < k && seg[c1 + 1] <= p1) ++c1;
  if (c0 == c1) {
    float2 s2 = make_float2(x[0], x[1]);
#pragma unroll
    for (int q = 2; q < 32; q += 2) s2 = f2add(s2, make_float2(x[q], x[q + 1]));
    if (c0 != cur) {
      if (cur >= 0 && row_ok) red_add_s64(Sfix + p * k + cur, ss_fix(run, fx_scale));
      run = 0.0;
      cur = c0;
    }
    run += (double)(s2.x + s2.y);
  } else {
    for (int cc = c0; cc <= c1; ++cc) {
      const int64_t lo = seg[cc] - p0, hi = (cc + 1 < k ? (int64_t)seg[cc + 1] : n) - p0;
      float sum = 0.f;
#pragma unroll
      for (int q = 0; q < 32; ++q) sum += (q >= lo && q < hi) ? x[q] : 0.f;
      if (cc != cur) {
        if (cur >= 0 && row_ok) red_add_s64(Sfix + p * k + cur, ss_fix(run, fx_scale));
        run = 0.0;
        cur = cc;
      }
      run += (double)sum;
    }
  }
  if (diag) return;
  // column part: column p0 + l gets the sum over the warp's rows of each row label
  if (r0 == r1) {  // one label (almost always): the butterfly consumes x
    const float cs = lane_column_sum(x, lane);
    if (p0 + lane < n) red_add_s64(Sfix + (p0 + lane) * k + r0, ss_fix((double)cs, fx_scale));
  } else if (row_ok) {  // the rows straddle a segment boundary: element by element
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (p0 + q < n) red_add_s64(Sfix + (p0 + q) * k + mylab, ss_fix((double)x[q], fx_scale));
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SS_THREADS, 1)
    ssym_kernel(const __grid_constant__ CUtensorMap t_hi, const __grid_constant__ CUtensorMap t_lo, uint32_t idesc,
                int nkb, int64_t n, const float *__restrict__ snorms, const float *__restrict__ srscale,
                const int32_t *__restrict__ seg_g, int k, KappaParams kp, T2SymSched sc, double fx_scale,
                long long *__restrict__ Sfix) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *extra;
  const T2Smem s = t2_carve(smem_raw, (uint32_t)SS_EXTRA, &extra);
  float *colc = reinterpret_cast<float *>(extra);
  int32_t *seg = reinterpret_cast<int32_t *>(extra + SS_EPI_WARPS * SS_COLC_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const bool fp16 = srscale != nullptr;
  for (int c = threadIdx.x; c <= k; c += blockDim.x) seg[c] = seg_g[c];
  t2_setup(s, warp, 2 * SS_EPI_WARPS);
  const uint32_t tmem_base = *s.tmem_slot;

  if (warp == 0) {
    if (lane == 0) t2_producer(sc, s, &t_hi, &t_lo, &t_hi, &t_lo, nkb, cr, 1);
  } else if (warp == 1) {
    if (lane == 0 && cr == 0) t2_mma(sc, s, nkb, idesc, tmem_base);
  } else {
    const int e = warp - 2;
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int colq = e >> 2;        // its 64-column quarter of the 256-column tile
    float *cn = colc + e * (2 * SS_COLS);
    const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colq * SS_COLS);
    const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    int64_t it = 0;
    for (int64_t u = cl; u < sc.nitems; u += ncl) {
      const int4 U = sc.units[u];
      const int tm = U.x, tn0 = U.y, tn1 = U.y + U.z;
      const int64_t rw = (int64_t)tm * T2_BM + (int64_t)cr * 128 + quarter * 32;  // warp's first row
      const int64_t p = rw + lane;                                                 // this thread's row
      const bool row_ok = p < n;
      const float ni = row_ok ? snorms[p] : 0.f;
      const float rsi = (fp16 && row_ok) ? srscale[p] : 1.f;
      const RowK rk = make_rowk(kp, rsi, ni);
      // labels of the warp's rows (sorted: segments r0 .. r1) and of this row
      const int64_t plast = rw + 31 < n ? rw + 31 : n - 1;
      const int r0 = rw < n ? ss_segment_of(seg, k, rw) : 0;
      const int r1 = rw < n ? ss_segment_of(seg, k, plast) : 0;
      const int mylab = row_ok ? ss_segment_of(seg, k, p) : r0;
      // the row part's running sum: segment `cur` of the columns seen last, flushed on change
      double run = 0.0;
      int cur = -1;
      int cseg = ss_segment_of(seg, k, (int64_t)tn0 * 256 + colq * SS_COLS < n ? (int64_t)tn0 * 256 + colq * SS_COLS : n - 1);
      for (int tn = tn0; tn < tn1; ++tn, ++it) {
        const int64_t pbase = (int64_t)tn * 256 + colq * SS_COLS;
        const bool diag = tn == tm;
        ss_stage_columns(cn, snorms, fp16 ? srscale : nullptr, pbase, n, kp.kind == 2, lane);
        mbar_wait(s.tfull, (uint32_t)(it & 1));
        tc_fence_after();
        // 1. drain main + correction into registers, give TMEM back
        float va[32], vb[32];
        {
          float w[32];
          tmem_ld32_nowait(tq, va);
          tmem_ld32_nowait(tq + 256u, w);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            const float2 t = f2add(make_float2(va[q], va[q + 1]), make_float2(w[q], w[q + 1]));
            va[q] = t.x;
            va[q + 1] = t.y;
          }
          tmem_ld32_nowait(tq + 32u, vb);
          tmem_ld32_nowait(tq + 256u + 32u, w);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            const float2 t = f2add(make_float2(vb[q], vb[q + 1]), make_float2(w[q], w[q + 1]));
            vb[q] = t.x;
            vb[q + 1] = t.y;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(s.tempty, 0);
        if (rw >= n) continue;
        // 2. per chunk: kappa, row part, column part
        ss_chunk(va, pbase, cn, kp, rk, diag, p, row_ok, n, seg, k, cseg, cur, run, r0, r1, mylab, lane, fx_scale,
                 Sfix);
        ss_chunk(vb, pbase + 32, cn + 32, kp, rk, diag, p, row_ok, n, seg, k, cseg, cur, run, r0, r1, mylab, lane,
                 fx_scale, Sfix);
      }
      if (cur >= 0 && row_ok) red_add_s64(Sfix + p * k + cur, ss_fix(run, fx_scale));
    }
  }
  t2_teardown(s, warp, tmem_base);
}

inline int ssym_launch(TcStream &g, const uint16_t *Shi, const uint16_t *Slo, bool fp16, int64_t rows, int64_t dp,
                       int64_t n, const float *snorms, const float *srscale, const int32_t *seg, int k,
                       const KappaParams &kp, const int4 *units, int64_t nunits, double fx_scale, long long *Sfix,
                       cudaStream_t st, int64_t *launches) {
  if (!tc_encode_fn()) {
    TcGemm tmp;
    if (tc_make_maps(tmp, Shi, Slo, fp16, rows, dp)) return 1;
  }
  if (g.ahi != Shi || g.alo != Slo || g.bhi != Shi || g.blo != Slo || g.fp16 != fp16 || g.arows != rows ||
      g.brows != rows) {
    if (ts_encode(&g.a_hi, Shi, fp16, rows, dp) || ts_encode(&g.a_lo, Slo, fp16, rows, dp)) return 1;
    g.b_hi = g.a_hi;
    g.b_lo = g.a_lo;
    g.ahi = g.bhi = Shi;
    g.alo = g.blo = Slo;
    g.fp16 = fp16;
    g.arows = g.brows = rows;
  }
  if (!g.num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (nunits <= 0) return 0;
  if (k > KKM_MAX_K) {
    tc_err_slot() = "ssym_launch: k > KKM_MAX_K";
    return 1;
  }
  if (ensure_smem_attr((const void *)ssym_kernel, SS_SMEM) != cudaSuccess) {
    tc_err_slot() = "cudaFuncSetAttribute(ssym_kernel) failed";
    return 1;
  }
  T2SymSched sc;
  sc.units = units;
  sc.nitems = nunits;
  const int64_t clusters = nunits < g.num_sms / 2 ? nunits : g.num_sms / 2;
  ssym_kernel<<<(unsigned)(2 * clusters), SS_THREADS, SS_SMEM, st>>>(
      g.a_hi, g.a_lo, t2_idesc(fp16), (int)(dp / TC_BK), n, snorms, fp16 ? srscale : nullptr, seg, k, kp, sc,
      fx_scale, Sfix);
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace kkm
