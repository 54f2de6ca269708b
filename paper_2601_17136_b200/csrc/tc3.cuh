// tc3.cuh -- the a1 tensor-core kernels on the chained mainloop (chain.cuh): the materialised GEMM
// + kappa epilogue (store; or the diagonal only: the tensor core's self dots), and the full
// (non-symmetric) fused streaming kernel. Same arithmetic per element as ssym.cuh, so every path
// computes b = x.y with identical chain boundaries (DESIGN A9).
//
// Epilogue layout (16 warps): warp e = 2 .. 17 reads TMEM lane quarter (warp & 3) and the 64-column
// quarter (e >> 2) of the 256-column tile; thread = row.
#pragma once
#include "chain.cuh"

namespace kkm {

constexpr uint32_t T3_STAGING_BYTES = 32 * 32;  // per warp: one TMA store box of 32 rows x 32 bytes
constexpr size_t T3_GEMM_EXTRA = CH_EPI_WARPS * (CH_COLC_BYTES + T3_STAGING_BYTES);
constexpr size_t T3_GEMM_SMEM = (size_t)T2_STAGES * T2_STAGE_BYTES + T3_GEMM_EXTRA + 1024 + 128;

// ---------------------------------------------------------------- materialised GEMM + kappa
// Output maps: [m x ncov] views of the region's K (row pitch ldo), fp32 boxes of 32 rows x 8
// columns or fp16 boxes of 32 rows x 16 columns, 32-byte swizzle (tc3_encode_out_map).
// oscale == 0: fp32 output; > 0: fp16 K * oscale, planes == 1 (hi only) or 2 (hi, lo = RN(K' - hi)
// through the second map). diag_out != NULL: no stores, diag_out[i] = kappa(x_i, x_i) of the tiles.
template <class Sched, int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CH_THREADS, 1)
    tc3_gemm_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
                    const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_out2,
                    const CUtensorMap *__restrict__ omaps, uint32_t idesc, int nkb, int nch, int64_t n,
                    const float *__restrict__ norms, const float *__restrict__ rscale, KappaParams kp, Sched sc,
                    float oscale, int planes, float *__restrict__ diag_out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *extra;
  const ChSmem s = ch_carve(smem_raw, (uint32_t)T3_GEMM_EXTRA, &extra);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  ch_setup(s, warp, 2 * CH_EPI_WARPS);
  const uint32_t tmem_base = *s.tmem_slot;
  if (warp < 2) {
    ch_producer_mma(sc, s, warp, lane, cr, &tm_hi, &tm_lo, &tm_hi, &tm_lo, nkb, nch, idesc, tmem_base);
  } else {
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int colq = e >> 2;
    float *cn = reinterpret_cast<float *>(extra) + e * (2 * CH_COLS);
    uint8_t *stg = extra + CH_EPI_WARPS * CH_COLC_BYTES + e * T3_STAGING_BYTES;
    const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colq * CH_COLS);
    const uint64_t evict = l2_policy_evict_first();
    const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const uint32_t swz = ((uint32_t)lane >> 2) & 1u;  // 32-byte swizzle of this row's two 16-byte units
    int64_t chain = 0;
    for (int64_t u = cl; u < sc.nitems; u += ncl) {
      int tm, tn, ridx;
      int64_t i0, m, j0, ncov;
      sc.region(u, tm, tn, i0, m, j0, ncov, ridx);
      const CUtensorMap *out1 = ridx < 0 ? &tm_out : omaps + (int64_t)ridx * planes;
      const CUtensorMap *out2 = ridx < 0 ? &tm_out2 : out1 + 1;
      const int64_t ibase = i0 + (int64_t)tm * T2_BM + (int64_t)cr * 128 + quarter * 32;
      const int64_t i = ibase + lane;
      const bool row_ok = i < i0 + m && i < n;
      const float ni = (row_ok && KIND == 2) ? norms[i] : 0.f;
      const float rsi = (rscale && row_ok) ? rscale[i] : 1.f;
      const RowK rk = make_rowk(kp, rsi, ni);
      const int64_t jw = j0 + (int64_t)tn * 256 + colq * CH_COLS;
      ch_stage_columns(cn, norms, rscale, jw, n, KIND == 2, lane);
      float va[32], vb[32];
      ch_drain(s, tq, nch, chain, va, vb, lane);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float(&v)[32] = c ? vb : va;
        const int64_t jb = jw + 32 * c;
        if (jb >= j0 + ncov || ibase >= i0 + m) continue;
        ch_kappa<KIND>(v, cn + 32 * c, cn + CH_COLS + 32 * c, kp, rk);
        if (diag_out) {
          if (row_ok && i >= jb && i < jb + 32) {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (jb + q == i) diag_out[i] = v[q];
          }
          continue;
        }
        if (KIND == 2 && i >= jb && i < jb + 32) {  // kappa(x_i, x_i) = 1 exactly (A1)
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (jb + q == i) v[q] = 1.f;
        }
        if (!row_ok || jb + 32 > n) {  // partial chunk / invalid row: padding is 0
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (!row_ok || jb + q >= n) v[q] = 0.f;
        }
        if (oscale > 0.f) {  // fp16 planes: boxes of 16 columns
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] *= oscale;
          for (int pl = 0; pl < planes; ++pl) {
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
              if (jb + 16 * hb >= j0 + ncov) continue;
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int u2 = 0; u2 < 2; ++u2) {
                uint32_t hw[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                  const int q = 16 * hb + 8 * u2 + 2 * e2;
                  const __half2 h2 = __floats2half2_rn(v[q], v[q + 1]);
                  hw[e2] = *reinterpret_cast<const uint32_t *>(&h2);
                  if (pl == 0 && planes > 1) {  // the residual for the lo plane (exact in fp32)
                    const float2 f = __half22float2(h2);
                    v[q] -= f.x;
                    v[q + 1] -= f.y;
                  }
                }
                *reinterpret_cast<uint4 *>(stg + lane * 32 + (((uint32_t)u2 ^ swz) << 4)) =
                    make_uint4(hw[0], hw[1], hw[2], hw[3]);
              }
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(pl ? out2 : out1, (int)(jb + 16 * hb - j0), (int)(ibase - i0), stg, evict);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              }
            }
          }
          continue;
        }
#pragma unroll
        for (int hb = 0; hb < 4; ++hb) {  // fp32: boxes of 8 columns
          if (jb + 8 * hb >= j0 + ncov) continue;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) {
            const int q = 8 * hb + 4 * u2;
            *reinterpret_cast<float4 *>(stg + lane * 32 + (((uint32_t)u2 ^ swz) << 4)) =
                make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(out1, (int)(jb + 8 * hb - j0), (int)(ibase - i0), stg, evict);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  ch_teardown(warp, tmem_base);
}

// [m x ncov] view of out (row pitch ldo elements) for tc3_gemm_kernel's stores: fp32 boxes of
// 32 rows x 8 columns (ldo % 4 == 0) or fp16 boxes of 32 rows x 16 columns (ldo % 8 == 0).
inline int tc3_encode_out_map(CUtensorMap *map, void *out, int64_t m, int64_t ncov, int64_t ldo, bool half_out) {
  if (tc_encode_ready()) return 1;
  cuuint64_t dims[2] = {(cuuint64_t)ncov, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)ldo * (half_out ? 2 : 4)};
  cuuint32_t box[2] = {half_out ? 16u : 8u, 32u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = tc_encode_fn()(map, half_out ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                              2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tc_err_slot() = "cuTensorMapEncodeTiled (output) failed";
    return 1;
  }
  return 0;
}

template <class Sched>
inline int tc3_gemm_run(TcGemm &g, bool fp16, const float *rscale, int64_t dp, int64_t n, const CUtensorMap &o1,
                        const CUtensorMap &o2, const CUtensorMap *omaps, const Sched &sc, const float *norms,
                        const KappaParams &kp, float oscale, int planes, float *diag_out, cudaStream_t st,
                        int64_t *launches, int ckb) {
  if (sc.nitems <= 0) return 0;
  if (!g.num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int nkb = (int)(dp / TC_BK);
  const int nch = ch_chains(nkb, ckb > 0 ? ckb : CH_CKB);
  const int64_t clusters = sc.nitems < g.num_sms / 2 ? sc.nitems : g.num_sms / 2;
  const unsigned grid = (unsigned)(2 * clusters);
  const int rc = ch_dispatch_kind(kp, [&](auto kind_tag) -> int {
    constexpr int KIND = decltype(kind_tag)::value;
    if (ensure_smem_attr((const void *)tc3_gemm_kernel<Sched, KIND>, T3_GEMM_SMEM) != cudaSuccess) return 1;
    tc3_gemm_kernel<Sched, KIND><<<grid, CH_THREADS, T3_GEMM_SMEM, st>>>(
        g.map_hi, g.map_lo, o1, o2, omaps, t2_idesc(fp16), nkb, nch, n, norms, fp16 ? rscale : nullptr, kp, sc, oscale,
        planes, diag_out);
    return 0;
  });
  if (rc) {
    tc_err_slot() = "cudaFuncSetAttribute(tc3_gemm_kernel) failed";
    return 1;
  }
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// One region: K[i0 : i0 + m, j0 : j0 + ncov] into out (row pitch ldo); same contract as round 1's
// tc2_gemm_launch. oscale > 0: fp16 K * oscale (hi), with out_lo also lo = RN(K * oscale - hi).
inline int tc3_gemm_launch(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16, const float *rscale,
                           int64_t rows, int64_t dp, int64_t n, int64_t i0, int64_t m, int64_t j0, int64_t ncov,
                           const float *norms, const KappaParams &kp, void *out, int64_t ldo, cudaStream_t st,
                           int64_t *launches, float oscale = 0.f, void *out_lo = nullptr, int ckb = 0) {
  if (g.hi != Xhi || g.lo != Xlo || g.fp16 != fp16)
    if (tc_make_maps(g, Xhi, Xlo, fp16, rows, dp)) return 1;
  if ((ldo & (oscale > 0.f ? 7 : 3)) || (reinterpret_cast<uintptr_t>(out) & 15)) {
    tc_err_slot() = "tcgen05 GEMM output needs 16-byte alignment and 16-byte aligned rows";
    return 1;
  }
  if (tc3_encode_out_map(&g.map_out, out, m, ncov, ldo, oscale > 0.f)) return 1;
  g.map_out2 = g.map_out;
  if (out_lo && tc3_encode_out_map(&g.map_out2, out_lo, m, ncov, ldo, true)) return 1;
  T2GemmSched sc;
  sc.tiles_m = (int)((m + T2_BM - 1) / T2_BM);
  sc.tiles_n = (int)((ncov + 255) / 256);
  sc.nitems = (int64_t)sc.tiles_m * sc.tiles_n;
  sc.i0 = i0;
  sc.j0 = j0;
  sc.m = m;
  sc.ncov = ncov;
  return tc3_gemm_run(g, fp16, rscale, dp, n, g.map_out, g.map_out2, nullptr, sc, norms, kp, oscale,
                      out_lo ? 2 : 1, nullptr, st, launches, ckb);
}

// Several output regions (the f1 band pieces) in ONE launch; regs_dev / omaps on the device, omaps
// encoded with tc3_encode_out_map (nreg * planes of them).
inline int tc3_gemm_launch_multi(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16, const float *rscale,
                                 int64_t rows, int64_t dp, int64_t n, const T2Region *regs_dev, int nreg,
                                 int64_t nitems, const CUtensorMap *omaps, const float *norms, const KappaParams &kp,
                                 float oscale, int planes, cudaStream_t st, int64_t *launches, int ckb = 0) {
  if (nitems <= 0) return 0;
  if (g.hi != Xhi || g.lo != Xlo || g.fp16 != fp16)
    if (tc_make_maps(g, Xhi, Xlo, fp16, rows, dp)) return 1;
  T2MultiSched sc;
  sc.nitems = nitems;
  sc.nreg = nreg;
  sc.reg = regs_dev;
  return tc3_gemm_run(g, fp16, rscale, dp, n, g.map_hi, g.map_hi, omaps, sc, norms, kp, oscale, planes, nullptr, st,
                      launches, ckb);
}

// out[i] = the tensor core's x_i . x_i (linear kernel), i < n: the SAME chained mainloop and
// epilogue arithmetic as every off-diagonal b = x_i . x_j. The Gaussian kernel's norms, so that
// r^2 = n_i + n_j - 2 b carries the accumulation error of like terms (DESIGN A9).
inline int tc3_self_dots(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16, const float *rscale,
                         int64_t rows, int64_t dp, int64_t n, float *out, cudaStream_t st, int64_t *launches,
                         int ckb = 0) {
  if (n <= 0) return 0;
  if (g.hi != Xhi || g.lo != Xlo || g.fp16 != fp16)
    if (tc_make_maps(g, Xhi, Xlo, fp16, rows, dp)) return 1;
  T2DiagSched sc;
  sc.n = n;
  sc.nitems = (n + T2_BM - 1) / T2_BM;
  KappaParams lin{};
  lin.kind = 0;
  return tc3_gemm_run(g, fp16, rscale, dp, n, g.map_hi, g.map_hi, nullptr, sc, out, lin, 0.f, 1, out, st, launches,
                      ckb);
}

// ---------------------------------------------------------------- full streaming kernel
// A = rows [row0, row0 + nloc) of a split operand (Xhi/Xlo), B = a label-sorted set of nB points
// (Shi/Slo) with segments seg[0..k]; work units = (256-row pair tile, split of the sorted columns)
// (T2StreamSched). Sx[r][c] (int64 fixed point, r = A row - row0, row pitch k) += 2^s times
// sum_{q in segment c} kappa(a_r, b_q) -- Eqs. (b), (k), (e); one running sum per row flushed at
// segment changes (ch_row_part). pos (may be NULL): sorted position of A row i for b0 <= i <
// b0 + npos, where kappa(x_i, x_i) = 1 exactly (A1). K(A, B) is never stored.
constexpr size_t T3_STREAM_RING_OFF = CH_EPI_WARPS * CH_COLC_BYTES + ((size_t)(KKM_MAX_K + 1) * 4 + 15) / 16 * 16;
constexpr size_t T3_STREAM_EXTRA = T3_STREAM_RING_OFF + CH_RING_BYTES;
constexpr size_t T3_STREAM_SMEM = (size_t)T2_STAGES * T2_STAGE_BYTES + T3_STREAM_EXTRA + 1024 + 128;

template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CH_THREADS, 1)
    tc3_stream_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                      const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                      uint32_t idesc, int nkb, int nch, int64_t nB, int64_t b0, int64_t nloc,
                      const float *__restrict__ norms, const float *__restrict__ rscale,
                      const float *__restrict__ snorms, const float *__restrict__ srscale,
                      const int32_t *__restrict__ pos, int64_t npos, const int32_t *__restrict__ seg_g, int k,
                      KappaParams kp, T2StreamSched sc, bool dyn, int32_t *__restrict__ work, float fx,
                      long long *__restrict__ Sx) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *extra;
  const ChSmem s = ch_carve(smem_raw, (uint32_t)T3_STREAM_EXTRA, &extra);
  float *colc = reinterpret_cast<float *>(extra);
  int32_t *seg = reinterpret_cast<int32_t *>(extra + CH_EPI_WARPS * CH_COLC_BYTES);
  const ChRing ring = ch_ring_carve(extra + T3_STREAM_RING_OFF, dyn, sc.nitems, work);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const bool fp16 = rscale != nullptr;
  for (int c = threadIdx.x; c <= k; c += blockDim.x) seg[c] = seg_g[c];
  ch_ring_init(ring);
  ch_setup(s, warp, 2 * CH_EPI_WARPS);  // (its cluster barrier also publishes seg and the ring's init)
  const uint32_t tmem_base = *s.tmem_slot;
  if (warp == 0) {
    if (lane == 0) ch_ring_producer(sc, ring, s, cr, &ta_hi, &ta_lo, &tb_hi, &tb_lo, nkb);
  } else if (warp == 1) {
    if (lane == 0 && cr == 0) ch_ring_mma(sc, ring, s, nkb, nch, idesc, tmem_base);
  } else {
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int colq = e >> 2;
    float *cn = colc + e * (2 * CH_COLS);
    const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colq * CH_COLS);
    int64_t chain = 0;
    for (int64_t iu = 0;; ++iu) {
      const int64_t u = ring.take(iu, lane == 0);
      if (u < 0) break;
      int tm, tn0, ntn;
      sc.unit(u, tm, tn0, ntn);
      const int tn1 = tn0 + ntn;
      const int64_t r = (int64_t)tm * T2_BM + (int64_t)cr * 128 + quarter * 32 + lane;  // A-set row
      const bool row_ok = r < nloc;
      const int64_t i = sc.row0 + r;
      const float ni = (row_ok && KIND == 2) ? norms[i] : 0.f;
      const float rsi = (fp16 && row_ok) ? rscale[i] : 1.f;
      const RowK rk = make_rowk(kp, rsi, ni);
      const int64_t mypos = (row_ok && KIND == 2 && pos && i >= b0 && i < b0 + npos) ? pos[i - b0] : -1;
      long long run = 0;
      int cur = -1;
      const int64_t pfirst = (int64_t)tn0 * 256 + colq * CH_COLS;
      int cseg = ch_segment_of(seg, k, pfirst < nB ? pfirst : (nB > 0 ? nB - 1 : 0));
      for (int tn = tn0; tn < tn1; ++tn) {
        const int64_t pbase = (int64_t)tn * 256 + colq * CH_COLS;
        ch_stage_columns(cn, snorms, fp16 ? srscale : nullptr, pbase, nB, KIND == 2, lane);
        float va[32], vb[32];
        ch_drain(s, tq, nch, chain, va, vb, lane);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float(&x)[32] = c ? vb : va;
          const int64_t p0 = pbase + 32 * c;
          if (p0 >= nB) continue;
          ch_kappa<KIND>(x, cn + 32 * c, cn + CH_COLS + 32 * c, kp, rk);
          if (KIND == 2 && mypos >= p0 && mypos < p0 + 32) {  // kappa(x_i, x_i) = 1 exactly (A1)
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (p0 + q == mypos) x[q] = 1.f;
          }
          if (p0 + 32 > nB) {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (p0 + q >= nB) x[q] = 0.f;
          }
          ch_row_part(x, p0, nB, seg, k, cseg, cur, run, row_ok, Sx + r * k, fx);
        }
      }
      if (cur >= 0 && row_ok) red_add_s64(Sx + r * k + cur, run);
    }
  }
  ch_teardown(warp, tmem_base);
}

// Streaming on CTA pairs: A = rows_a rows (Xhi/Xlo, norms, rscale), output rows [row0, row0 + nloc);
// B = the label-sorted operand (Shi/Slo, snorms, srscale; rows_b rows) holding nB points in k
// segments seg[0..k]. Sx: [>= nloc][k] int64, zeroed by the caller; fx = 2^s with
// nB max|K| 2^s < 2^61. splits: column splits per pair row tile (load balance / L2 reuse).
inline int tc3_stream_launch(TcStream &g, const uint16_t *Xhi, const uint16_t *Xlo, const uint16_t *Shi,
                             const uint16_t *Slo, bool fp16, int64_t rows_a, int64_t rows_b, int64_t dp, int64_t nB,
                             int64_t b0, int64_t row0, int64_t nloc, const float *norms, const float *rscale,
                             const float *snorms, const float *srscale, const int32_t *pos, int64_t npos,
                             const int32_t *seg, int k, const KappaParams &kp, double fx,
                             long long *Sx, cudaStream_t st, int64_t *launches, int ckb = 0) {
  if (!tc_encode_fn()) {
    TcGemm tmp;
    if (tc_make_maps(tmp, Xhi, Xlo, fp16, rows_a, dp)) return 1;
  }
  if (g.ahi != Xhi || g.alo != Xlo || g.bhi != Shi || g.blo != Slo || g.fp16 != fp16 || g.arows != rows_a ||
      g.brows != rows_b) {
    if (ts_encode(&g.a_hi, Xhi, fp16, rows_a, dp) || ts_encode(&g.a_lo, Xlo, fp16, rows_a, dp) ||
        ts_encode(&g.b_hi, Shi, fp16, rows_b, dp) || ts_encode(&g.b_lo, Slo, fp16, rows_b, dp))
      return 1;
    g.ahi = Xhi;
    g.alo = Xlo;
    g.bhi = Shi;
    g.blo = Slo;
    g.fp16 = fp16;
    g.arows = rows_a;
    g.brows = rows_b;
  }
  if (!g.num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (nloc <= 0 || nB <= 0) return 0;
  if (k > KKM_MAX_K) {
    tc_err_slot() = "tc3_stream_launch: k > KKM_MAX_K";
    return 1;
  }
  if (!g.work) {  // the dynamic schedule's two counters (zero between launches: the kernel resets them)
    if (cudaMalloc((void **)&g.work, 16) != cudaSuccess || cudaMemset(g.work, 0, 16) != cudaSuccess) {
      g.work = nullptr;
      tc_err_slot() = "cudaMalloc (stream unit counter) failed";
      return 1;
    }
  }
  // units of W column tiles in G-row supertiles (T2StreamSched), taken dynamically: the ~74 units
  // in flight cover ~G A tiles and a few W-groups of B tiles (as ssym.cuh; KKM_TS_G / KKM_TS_W /
  // KKM_SSYM_STATIC for A/B runs)
  T2StreamSched sc;
  sc.tiles_m = (int)((nloc + T2_BM - 1) / T2_BM);
  sc.tiles_n = (int)((nB + 255) / 256);
  sc.G = 32;
  sc.W = 16;
  if (const char *e = std::getenv("KKM_TS_G")) sc.G = std::max(1, std::atoi(e));
  if (const char *e = std::getenv("KKM_TS_W")) sc.W = std::max(1, std::atoi(e));
  sc.ncb = (sc.tiles_n + sc.W - 1) / sc.W;
  sc.nitems = (int64_t)sc.tiles_m * sc.ncb;
  sc.row0 = row0;
  sc.hint = 1;  // L2 evict_last on the operand loads
  const bool dyn = std::getenv("KKM_SSYM_STATIC") == nullptr;
  const int64_t clusters = sc.nitems < g.num_sms / 2 ? sc.nitems : g.num_sms / 2;
  const unsigned grid = (unsigned)(2 * clusters);
  const int nkb = (int)(dp / TC_BK);
  const int nch = ch_chains(nkb, ckb > 0 ? ckb : CH_CKB);
  const float *rs = fp16 ? rscale : nullptr;
  const float *srs = fp16 ? srscale : nullptr;
  const int rc = ch_dispatch_kind(kp, [&](auto kind_tag) -> int {
    constexpr int KIND = decltype(kind_tag)::value;
    if (ensure_smem_attr((const void *)tc3_stream_kernel<KIND>, T3_STREAM_SMEM) != cudaSuccess) return 1;
    tc3_stream_kernel<KIND><<<grid, CH_THREADS, T3_STREAM_SMEM, st>>>(
        g.a_hi, g.a_lo, g.b_hi, g.b_lo, t2_idesc(fp16), nkb, nch, nB, b0, nloc, norms, rs, snorms, srs, pos, npos, seg,
        k, kp, sc, dyn, g.work, (float)fx, Sx);
    return 0;
  });
  if (rc) {
    tc_err_slot() = "cudaFuncSetAttribute(tc3_stream_kernel) failed";
    return 1;
  }
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace kkm
