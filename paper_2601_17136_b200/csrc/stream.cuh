// stream.cuh -- fused streaming a1+a2 (K never stored): for the rank's rows i and all points j
// in cluster-sorted order p (sort.cuh), S(i, c) = sum_{p in segment c} kappa(x_i . x_perm[p])
// (Eqs. b, k, e), the paper's sliding-window recompute done tile by tile
// in TMEM instead of b x n block rows in HBM.
//
// Same tensor-core mainloop as gemm_tc.cuh (TMA producer warp, single-thread tcgen05.mma issuer,
// fp16x3 / bf16x3 with the main and correction TMEM accumulators). Work unit = one 128-row tile
// x one split of the sorted column range; the epilogue warps (thread = row, 8 warps = 4 lane
// quarters x 2 column halves) apply kappa to each 32-column chunk and add its sum into the row's
// per-cluster fp64 accumulator. Chunks lie inside one cluster except at the <= k-1 segment
// boundaries, which are handled by a warp-uniform per-segment split, so the reduction costs
// ~1 FADD per element. Partials go to Spart[2*split + half][row][c], reduced in fixed order by
// finalize_kernel exactly like the materialised SpMM's output.
#pragma once
#include "gemm_tc.cuh"

namespace kkm {

constexpr size_t TS_COLC_BYTES = TC_EPI_WARPS * 256 * 4;  // per warp: 128 x (norm_j, rscale_j)
constexpr size_t TS_SMEM = (size_t)TC_STAGES * TC_STAGE_BYTES + TS_COLC_BYTES + 1024 /*align*/ +
                           128 /*barriers*/ + 65 * 4 /*seg*/;

template <int KMAX>
__device__ __forceinline__ void acc_add(double (&acc)[KMAX], int c, double s) {
#pragma unroll
  for (int cc = 0; cc < KMAX; ++cc)
    if (cc == c) acc[cc] += s;
}

template <int KMAX>
__global__ void __launch_bounds__(TC_THREADS_V2, 1)
    tc_stream_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                     const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                     uint32_t idesc, int nkb, int64_t n, int64_t b0, int64_t row0, int64_t nloc,
                     int64_t rows_pad,
                     const float *__restrict__ norms, const float *__restrict__ rscale,
                     const float *__restrict__ snorms, const float *__restrict__ srscale,
                     const int32_t *__restrict__ pos, const int32_t *__restrict__ seg_g, int k,
                     KappaParams kp, int tiles_m, int tiles_n, int nsplit, int tps,
                     double *__restrict__ Spart) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  uint8_t *smem = smem_raw + pad;
  float *colc = reinterpret_cast<float *>(smem + TC_STAGES * TC_STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + TC_STAGES * TC_STAGE_BYTES + TS_COLC_BYTES);
  uint64_t *empty = full + TC_STAGES;
  uint64_t *tfull = empty + TC_STAGES;
  uint64_t *tempty = tfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);
  int32_t *seg = reinterpret_cast<int32_t *>(tmem_slot + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nunits = (int64_t)tiles_m * nsplit;
  const bool fp16 = rscale != nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, TC_EPI_WARPS);
    fence_barrier_init();
  }
  for (int c = threadIdx.x; c <= k; c += blockDim.x) seg[c] = seg_g[c];
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t keep = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int tm = (int)(u / nsplit), sp = (int)(u % nsplit);
        const int tn0 = sp * tps, tn1 = min(tiles_n, tn0 + tps);
        const int ra = (int)(row0 + (int64_t)tm * TC_BM);
        for (int tn = tn0; tn < tn1; ++tn) {
          const int rb = tn * TC_BN;
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t *st = smem + stage * TC_STAGE_BYTES;
            mbar_arrive_expect_tx(&full[stage], TC_STAGE_BYTES);
            const int kc = kb * TC_BK;
            tma_load_2d_hint(st, &ta_hi, kc, ra, &full[stage], keep);
            tma_load_2d_hint(st + TC_A_BYTES, &ta_lo, kc, ra, &full[stage], keep);
            tma_load_2d_hint(st + 2 * TC_A_BYTES, &tb_hi, kc, rb, &full[stage], keep);
            tma_load_2d_hint(st + 3 * TC_A_BYTES, &tb_hi, kc, rb + 128, &full[stage], keep);
            tma_load_2d_hint(st + 2 * TC_A_BYTES + TC_B_BYTES, &tb_lo, kc, rb, &full[stage], keep);
            tma_load_2d_hint(st + 3 * TC_A_BYTES + TC_B_BYTES, &tb_lo, kc, rb + 128, &full[stage], keep);
            if (++stage == TC_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t it = 0;
      const uint32_t d_main = tmem_base, d_corr = tmem_base + (uint32_t)TC_BN;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int sp = (int)(u % nsplit);
        const int tn0 = sp * tps, tn1 = min(tiles_n, tn0 + tps);
        for (int tn = tn0; tn < tn1; ++tn, ++it) {
          mbar_wait(tempty, (uint32_t)(it & 1) ^ 1u);
          tc_fence_after();
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + stage * TC_STAGE_BYTES);
            const uint32_t a_hi = st, a_lo = st + TC_A_BYTES;
            const uint32_t b_hi = st + 2 * TC_A_BYTES, b_lo = b_hi + TC_B_BYTES;
#pragma unroll
            for (int kk = 0; kk < TC_BK / 16; ++kk) {
              const uint32_t ko = (uint32_t)kk * 32u;
              const uint32_t acc = (kb == 0 && kk == 0) ? 0u : 1u;
              umma_f16(d_corr, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_lo + ko), idesc, acc);
              umma_f16(d_corr, umma_desc_sw128(a_lo + ko), umma_desc_sw128(b_hi + ko), idesc, 1u);
              umma_f16(d_main, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_hi + ko), idesc, acc);
            }
            umma_commit(&empty[stage]);
            if (++stage == TC_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(tfull);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int half = e >> 2;
    float *cn = colc + e * 256;  // [0,128): norm_j, [128,256): rscale_j of this warp's columns
    int64_t it = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int tm = (int)(u / nsplit), sp = (int)(u % nsplit);
      const int tn0 = sp * tps, tn1 = min(tiles_n, tn0 + tps);
      const int64_t r = (int64_t)tm * TC_BM + quarter * 32 + lane;  // local row
      const bool row_ok = r < nloc;
      const int64_t i = row0 + r;
      const float ni = row_ok ? norms[i] : 0.f;
      const float rsi = (fp16 && row_ok) ? rscale[i] : 1.f;
      const int64_t mypos = (row_ok && kp.kind == 2 && i >= b0 && i < b0 + n) ? pos[i - b0] : -1;
      double acc[KMAX];
#pragma unroll
      for (int c = 0; c < KMAX; ++c) acc[c] = 0.0;
      for (int tn = tn0; tn < tn1; ++tn, ++it) {
        const int64_t pbase = (int64_t)tn * TC_BN + half * 128;  // first sorted column of the warp
        // stage the per-column constants of my 128 columns (float4, lane-parallel)
        {
          const int64_t p = pbase + lane * 4;
          float4 nv = make_float4(0.f, 0.f, 0.f, 0.f), rv = make_float4(1.f, 1.f, 1.f, 1.f);
          if (p + 3 < n) {
            if (kp.kind == 2) nv = *reinterpret_cast<const float4 *>(snorms + p);
            if (fp16) rv = *reinterpret_cast<const float4 *>(srscale + p);
          } else {
            float *pn = &nv.x, *pr = &rv.x;
            for (int q = 0; q < 4; ++q)
              if (p + q < n) {
                if (kp.kind == 2) pn[q] = snorms[p + q];
                if (fp16) pr[q] = srscale[p + q];
              }
          }
          __syncwarp();
          reinterpret_cast<float4 *>(cn)[lane] = nv;
          reinterpret_cast<float4 *>(cn + 128)[lane] = rv;
          __syncwarp();
        }
        mbar_wait(tfull, (uint32_t)(it & 1));
        tc_fence_after();
        const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          const int col = half * 128 + c * 32;
          float v[32];
          tmem_ld_sum32(tq + (uint32_t)col, tq + (uint32_t)(TC_BN + col), v);
          const int64_t p0 = pbase + c * 32;
          if (p0 >= n) continue;
          const float *cnn = cn + c * 32, *crs = cn + 128 + c * 32;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 nj = reinterpret_cast<const float4 *>(cnn)[q4];
            const float4 rj = reinterpret_cast<const float4 *>(crs)[q4];
            const float njs[4] = {nj.x, nj.y, nj.z, nj.w}, rjs[4] = {rj.x, rj.y, rj.z, rj.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int q = q4 * 4 + t;
              const float b = fp16 ? v[q] * (rsi * rjs[t]) : v[q];
              const float kv = kappa_epilogue(kp, b, ni, njs[t], p0 + q == mypos);
              v[q] = (p0 + q < n) ? kv : 0.f;
            }
          }
          // warp-uniform segment structure of the chunk [p0, p1]
          const int64_t p1 = p0 + 31 < n ? p0 + 31 : n - 1;
          int c0 = 0, c1 = 0;
          for (int cc = 1; cc < k; ++cc) {
            if (seg[cc] <= p0) c0 = cc;
            if (seg[cc] <= p1) c1 = cc;
          }
          if (c0 == c1) {
            float s = 0.f;
#pragma unroll
            for (int q = 0; q < 32; ++q) s += v[q];
            acc_add<KMAX>(acc, c0, (double)s);
          } else {
            for (int cc = c0; cc <= c1; ++cc) {
              const int64_t lo = seg[cc] - p0, hi = seg[cc + 1] - p0;
              float s = 0.f;
#pragma unroll
              for (int q = 0; q < 32; ++q) s += (q >= lo && q < hi) ? v[q] : 0.f;
              acc_add<KMAX>(acc, cc, (double)s);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
      if (row_ok) {
        double *dst = Spart + ((int64_t)(2 * sp + half) * rows_pad + r) * k;
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
          if (c < k) dst[c] = acc[c];
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ---------------------------------------------------------------- host side
struct TcStream {
  const void *ahi = nullptr, *alo = nullptr, *bhi = nullptr, *blo = nullptr;
  bool fp16 = false;
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
  bool attr4 = false, attr8 = false, attr16 = false;
  int num_sms = 0;
};

inline int ts_encode(CUtensorMap *m, const void *ptr, bool fp16, int64_t rows, int64_t dp) {
  cuuint64_t dims[2] = {(cuuint64_t)dp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)dp * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, 128u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = tc_encode_fn()(m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                              (void *)ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tc_err_slot() = "cuTensorMapEncodeTiled (stream operand) failed";
    return 1;
  }
  return 0;
}

template <int KMAX>
inline int ts_launch_k(TcStream &g, bool &attr, int grid, cudaStream_t st, uint32_t idesc, int nkb, int64_t n,
                       int64_t b0, int64_t row0, int64_t nloc, int64_t rows_pad, const float *norms,
                       const float *rscale,
                       const float *snorms, const float *srscale, const int32_t *pos, const int32_t *seg,
                       int k, const KappaParams &kp, int tiles_m, int tiles_n, int nsplit, int tps,
                       double *Spart) {
  if (!attr) {
    if (cudaFuncSetAttribute(tc_stream_kernel<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)TS_SMEM) != cudaSuccess) {
      tc_err_slot() = "cudaFuncSetAttribute(tc_stream_kernel) failed";
      return 1;
    }
    attr = true;
  }
  tc_stream_kernel<KMAX><<<grid, TC_THREADS_V2, TS_SMEM, st>>>(
      g.a_hi, g.a_lo, g.b_hi, g.b_lo, idesc, nkb, n, b0, row0, nloc, rows_pad, norms, rscale, snorms, srscale,
      pos, seg, k, kp, tiles_m, tiles_n, nsplit, tps, Spart);
  return 0;
}

// Spart[2*split + half][r][c] (row pitch rows_pad) for rows r in [0, nloc) (global row0 + r)
// against the n sorted columns of the set starting at global point b0.
inline int tc_stream_launch(TcStream &g, const uint16_t *Xhi, const uint16_t *Xlo, const uint16_t *Shi,
                            const uint16_t *Slo, bool fp16, int64_t rows, int64_t dp, int64_t n,
                            int64_t b0, int64_t row0, int64_t nloc, int64_t rows_pad,
                            const float *norms, const float *rscale,
                            const float *snorms, const float *srscale, const int32_t *pos,
                            const int32_t *seg, int k, const KappaParams &kp, int nsplit, double *Spart,
                            cudaStream_t st, int64_t *launches) {
  if (!tc_encode_fn()) {  // resolve the driver entry point once
    TcGemm tmp;
    if (tc_make_maps(tmp, Xhi, Xlo, fp16, rows, dp)) return 1;
  }
  if (g.ahi != Xhi || g.alo != Xlo || g.bhi != Shi || g.blo != Slo || g.fp16 != fp16) {
    if (ts_encode(&g.a_hi, Xhi, fp16, rows, dp) || ts_encode(&g.a_lo, Xlo, fp16, rows, dp) ||
        ts_encode(&g.b_hi, Shi, fp16, rows, dp) || ts_encode(&g.b_lo, Slo, fp16, rows, dp))
      return 1;
    g.ahi = Xhi;
    g.alo = Xlo;
    g.bhi = Shi;
    g.blo = Slo;
    g.fp16 = fp16;
  }
  if (!g.num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (nloc <= 0) return 0;
  const int tiles_m = (int)((nloc + TC_BM - 1) / TC_BM);
  const int tiles_n = (int)((n + TC_BN - 1) / TC_BN);
  const int tps = (tiles_n + nsplit - 1) / nsplit;
  const int64_t nunits = (int64_t)tiles_m * nsplit;
  const int grid = (int)(nunits < g.num_sms ? nunits : g.num_sms);
  const uint32_t idesc = tc_idesc(fp16);
  const int nkb = (int)(dp / TC_BK);
  int rc;
  if (k <= 4)
    rc = ts_launch_k<4>(g, g.attr4, grid, st, idesc, nkb, n, b0, row0, nloc, rows_pad, norms,
                         fp16 ? rscale : nullptr,
                        snorms, srscale, pos, seg, k, kp, tiles_m, tiles_n, nsplit, tps, Spart);
  else if (k <= 8)
    rc = ts_launch_k<8>(g, g.attr8, grid, st, idesc, nkb, n, b0, row0, nloc, rows_pad, norms,
                         fp16 ? rscale : nullptr,
                        snorms, srscale, pos, seg, k, kp, tiles_m, tiles_n, nsplit, tps, Spart);
  else
    rc = ts_launch_k<16>(g, g.attr16, grid, st, idesc, nkb, n, b0, row0, nloc, rows_pad, norms,
                         fp16 ? rscale : nullptr,
                         snorms, srscale, pos, seg, k, kp, tiles_m, tiles_n, nsplit, tps, Spart);
  if (rc) return rc;
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// Splits of the sorted column range: enough work units for a full last wave.
inline int ts_choose_splits(int64_t nloc, int64_t n, int num_sms) {
  const int64_t tiles_m = (nloc + TC_BM - 1) / TC_BM;
  const int64_t tiles_n = (n + TC_BN - 1) / TC_BN;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 8 && s <= tiles_n; ++s) {
    const int64_t units = tiles_m * s;
    const int64_t waves = (units + num_sms - 1) / num_sms;
    const double eff = (double)units / (double)(waves * num_sms) - 0.002 * s;  // mild preference for fewer splits
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

}  // namespace kkm
