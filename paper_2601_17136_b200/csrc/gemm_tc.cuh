// gemm_tc.cuh -- a1 on the 5th-generation tensor cores: K = kappa(X X^T) (Eqs. b, k,
// P:92-104) with X split into bf16 hi + lo (reading A9) and
//     B = X_hi X_hi^T + X_hi X_lo^T + X_lo X_hi^T      (3 bf16 MMAs, fp32 TMEM accumulation)
// so the product error is ~2^-16 relative instead of bf16's 2^-8.
//
// Kernel anatomy: persistent, one CTA per SM, warp-specialised.
//   warp 0      TMA producer: per 64-wide K block loads A_hi, A_lo (128 rows) and B_hi,
//               B_lo (256 rows) into a 2-stage smem ring (128B-swizzled, K-major), L2
//               evict-last so the operands stay resident while K streams out
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//               M=128 N=256 K=16, 12 per K block (4 k-steps x 3 products), hi*hi into the
//               main TMEM accumulator and hi*lo + lo*hi into a correction accumulator;
//               tcgen05.commit -> mbarrier releases smem stages / publishes the tile
//   warps 2..9  epilogue: tcgen05.ld 32x32b (thread = row, 8 warps = 4 lane quarters x 2
//               column halves), main + correction, per-column factors from smem (LDS.128
//               broadcast), kappa, 64B-swizzled smem staging and TMA bulk-tensor stores
//               (L2 evict-first) of 32x16 fp32 boxes of K.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace kkm {

constexpr int TC_BM = 128;   // UMMA M (rows of K per tile)
constexpr int TC_BN = 256;   // UMMA N (columns of K per tile)
constexpr int TC_BK = 64;    // K block = one 128-byte swizzle atom of bf16
constexpr int TC_STAGES = 2;
constexpr uint32_t TC_A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
constexpr uint32_t TC_B_BYTES = TC_BN * TC_BK * 2;  // 32 KB
constexpr uint32_t TC_STAGE_BYTES = 2 * TC_A_BYTES + 2 * TC_B_BYTES;  // 96 KB
constexpr int TC_GROUP_M = 32;  // tile raster: groups of 32 row tiles sweep the column tiles

// instruction descriptor, kind::f16: D fp32, A/B bf16 (format 1) or fp16 (format 0), both
// K-major, N = 256, M = 128
constexpr uint32_t tc_idesc(bool fp16) {
  return (1u << 4) | ((fp16 ? 0u : 1u) << 7) | ((fp16 ? 0u : 1u) << 10) |
         ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane (no wait: call tmem_wait_ld()
// before reading v).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, float (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
        "=f"(v[14]), "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]),
        "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]),
        "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// main + correction accumulators of 32 columns, summed (fp32 RN).
__device__ __forceinline__ void tmem_ld_sum32(uint32_t t_main, uint32_t t_corr, float (&v)[32]) {
  float w[32];
  tmem_ld32_nowait(t_main, v);
  tmem_ld32_nowait(t_corr, w);
  tmem_wait_ld();
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] += w[q];
}

// Lane-parallel load of 128 per-column constants (norm_j, rscale_j) of columns [j, j+128) into
// smem cn[0..128) / cn[128..256); missing columns get (0, 1). Ends with __syncwarp.
__device__ __forceinline__ void stage_column_constants(float *cn, const float *__restrict__ norms,
                                                       const float *__restrict__ rscale, int64_t j,
                                                       int64_t nvalid, bool need_norm, int lane) {
  const int64_t p = j + lane * 4;
  float4 nv = make_float4(0.f, 0.f, 0.f, 0.f), rv = make_float4(1.f, 1.f, 1.f, 1.f);
  float *pn = &nv.x, *pr = &rv.x;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (p + q < nvalid) {
      if (need_norm) pn[q] = __ldg(norms + p + q);
      if (rscale) pr[q] = __ldg(rscale + p + q);
    }
  __syncwarp();
  reinterpret_cast<float4 *>(cn)[lane] = nv;
  reinterpret_cast<float4 *>(cn + 128)[lane] = rv;
  __syncwarp();
}

// Tile t -> (row tile, column tile): groups of TC_GROUP_M row tiles, column-major inside a
// group, so the ~148 concurrent tiles share A and B operands through L2.
__device__ __forceinline__ void tc_tile_coords(int64_t t, int tiles_m, int tiles_n, int &tm, int &tn) {
  const int64_t per_group = (int64_t)TC_GROUP_M * tiles_n;
  const int64_t g = t / per_group;
  const int first_m = (int)(g * TC_GROUP_M);
  const int gm = tiles_m - first_m < TC_GROUP_M ? tiles_m - first_m : TC_GROUP_M;
  const int64_t r = t - g * per_group;
  tm = first_m + (int)(r % gm);
  tn = (int)(r / gm);
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_2d_hint(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int c0, int c1, const void *smem_src,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src)), "l"(pol)
      : "memory");
}

constexpr int TC_EPI_WARPS = 8;
constexpr int TC_THREADS_V2 = (2 + TC_EPI_WARPS) * 32;
constexpr uint32_t TC_STAGING_BYTES = 32 * 16 * 4;  // per epilogue warp: 32 rows x 16 fp32 (SW64 box)
constexpr uint32_t TC_COLC_BYTES = 256 * 4;          // per epilogue warp: 128 x (norm_j, rscale_j)
constexpr size_t TC_SMEM_V2 = (size_t)TC_STAGES * TC_STAGE_BYTES +
                              TC_EPI_WARPS * (TC_STAGING_BYTES + TC_COLC_BYTES) + 1024 /*align*/ +
                              128 /*barriers*/;

// out[(i - i0) * ldo + (j - j0)] = kappa(x_i . x_j), i in [i0, i0+m), j in [j0, j0+ncov),
// 0 for j >= n, written by TMA stores through `tm_out` (an fp32 [m x ncov] view of out).
// A rows start at i0, B rows at j0 (global point indices). rscale (fp16 split, else NULL):
// x_i . x_j = acc * rscale[i] * rscale[j], exact powers of two.
// TMEM: the hi*hi products accumulate in columns [0, 256), the small hi*lo + lo*hi
// corrections in [256, 512): the tensor core's fp32 accumulation truncates once per MMA
// relative to the running sum, so keeping the corrections out of the main sum cuts the
// one-signed error of b by ~3x; the two are added in fp32 (RN).
__global__ void __launch_bounds__(TC_THREADS_V2, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
                   const __grid_constant__ CUtensorMap tm_out, uint32_t idesc, int nkb, int64_t n,
                   int64_t i0, int64_t m, int64_t j0, int64_t ncov, const float *__restrict__ norms,
                   const float *__restrict__ rscale, KappaParams kp, int tiles_m, int tiles_n) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  uint8_t *smem = smem_raw + pad;
  uint8_t *staging = smem + TC_STAGES * TC_STAGE_BYTES;
  float *colc = reinterpret_cast<float *>(staging + TC_EPI_WARPS * TC_STAGING_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(staging + TC_EPI_WARPS * (TC_STAGING_BYTES + TC_COLC_BYTES));
  uint64_t *empty = full + TC_STAGES;
  uint64_t *tfull = empty + TC_STAGES;  // accumulators ready
  uint64_t *tempty = tfull + 1;         // accumulators drained
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (int64_t)tiles_m * tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, TC_EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 1) {  // TMEM: 512 columns = main (hi*hi) + correction 128 x 256 fp32 accumulators
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
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int tm, tn;
        tc_tile_coords(t, tiles_m, tiles_n, tm, tn);
        const int ra = (int)(i0 + (int64_t)tm * TC_BM);
        const int rb = (int)(j0 + (int64_t)tn * TC_BN);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *st = smem + stage * TC_STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], TC_STAGE_BYTES);
          const int kc = kb * TC_BK;
          tma_load_2d_hint(st, &tm_hi, kc, ra, &full[stage], keep);                          // A_hi
          tma_load_2d_hint(st + TC_A_BYTES, &tm_lo, kc, ra, &full[stage], keep);             // A_lo
          tma_load_2d_hint(st + 2 * TC_A_BYTES, &tm_hi, kc, rb, &full[stage], keep);         // B_hi
          tma_load_2d_hint(st + 3 * TC_A_BYTES, &tm_hi, kc, rb + 128, &full[stage], keep);
          tma_load_2d_hint(st + 2 * TC_A_BYTES + TC_B_BYTES, &tm_lo, kc, rb, &full[stage], keep);  // B_lo
          tma_load_2d_hint(st + 3 * TC_A_BYTES + TC_B_BYTES, &tm_lo, kc, rb + 128, &full[stage], keep);
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
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
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        mbar_wait(tempty, (uint32_t)(it & 1) ^ 1u);
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * TC_STAGE_BYTES);
          const uint32_t a_hi = st, a_lo = st + TC_A_BYTES;
          const uint32_t b_hi = st + 2 * TC_A_BYTES, b_lo = b_hi + TC_B_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint32_t ko = (uint32_t)k * 32u;  // 16 elements = 32 bytes along K in the atom
            const uint32_t acc = (kb == 0 && k == 0) ? 0u : 1u;
            umma_f16(d_corr, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_lo + ko), idesc, acc);
            umma_f16(d_corr, umma_desc_sw128(a_lo + ko), umma_desc_sw128(b_hi + ko), idesc, 1u);
            umma_f16(d_main, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_hi + ko), idesc, acc);
          }
          umma_commit(&empty[stage]);  // smem stage free once these MMAs have read it
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull);  // accumulators complete
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    const int e = warp - 2;
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter + 32)
    const int half = e >> 2;       // tile columns [128*half, 128*half + 128)
    uint8_t *stg = staging + e * TC_STAGING_BYTES;
    float *cn = colc + e * 256;
    const uint64_t evict = l2_policy_evict_first();
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      int tm, tn;
      tc_tile_coords(t, tiles_m, tiles_n, tm, tn);
      const int64_t ibase = i0 + (int64_t)tm * TC_BM + quarter * 32;  // first row of this warp
      const int64_t i = ibase + lane;
      const bool row_ok = i < i0 + m && i < n;
      const float ni = row_ok ? norms[i] : 0.f;
      const float rsi = (rscale && row_ok) ? rscale[i] : 1.f;
      const int64_t jw = j0 + (int64_t)tn * TC_BN + half * 128;  // first column of this warp
      stage_column_constants(cn, norms, rscale, jw, n, kp.kind == 2, lane);
      mbar_wait(tfull, (uint32_t)(it & 1));
      tc_fence_after();
      const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col = half * 128 + c * 32;  // column offset inside the tile
        const int64_t jb = jw + c * 32;
        float v[32];
        tmem_ld_sum32(tq + (uint32_t)col, tq + (uint32_t)(TC_BN + col), v);
        if (jb >= j0 + ncov) continue;  // whole chunk outside the requested columns
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 nj = reinterpret_cast<const float4 *>(cn + c * 32)[q4];
          const float4 rj = reinterpret_cast<const float4 *>(cn + 128 + c * 32)[q4];
          const float njs[4] = {nj.x, nj.y, nj.z, nj.w}, rjs[4] = {rj.x, rj.y, rj.z, rj.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = 4 * q4 + u;
            const int64_t j = jb + q;
            const float b = rscale ? v[q] * (rsi * rjs[u]) : v[q];
            const float kv = kappa_epilogue(kp, b, ni, njs[u], i == j);
            v[q] = (row_ok && j < n) ? kv : 0.f;
          }
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // two 16-column boxes per 32-column chunk
          // the previous TMA store from this staging buffer must have finished reading it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {  // 64B-swizzled row: 16B chunk u4 at u4 ^ ((row >> 1) & 3)
            float4 *dst = reinterpret_cast<float4 *>(stg + lane * 64 + ((u4 ^ ((lane >> 1) & 3)) << 4));
            const int q = hh * 16 + 4 * u4;
            *dst = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && jb + hh * 16 < j0 + ncov) {
            tma_store_2d(&tm_out, (int)(jb + hh * 16 - j0), (int)(ibase - i0), stg, evict);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ---------------------------------------------------------------- host side
struct TcGemm {
  const void *hi = nullptr, *lo = nullptr;  // operands the tensor maps describe
  bool fp16 = false;
  CUtensorMap map_hi, map_lo;
  CUtensorMap map_out;                        // re-encoded per launch (cheap, host only)
  bool attr = false;
  int num_sms = 0;
};

inline const char *&tc_err_slot() {
  static thread_local const char *msg = "";
  return msg;
}
inline const char *tc_gemm_error() { return tc_err_slot(); }

inline PFN_cuTensorMapEncodeTiled_v12000 &tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  return f;
}

inline int tc_make_maps(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16, int64_t rows,
                        int64_t dp) {
  PFN_cuTensorMapEncodeTiled_v12000 &encode = tc_encode_fn();
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode) {
      tc_err_slot() = "cuTensorMapEncodeTiled unavailable";
      return 1;
    }
  }
  cuuint64_t dims[2] = {(cuuint64_t)dp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)dp * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, 128u};
  cuuint32_t es[2] = {1u, 1u};
  for (int w = 0; w < 2; ++w) {
    CUresult r = encode(w ? &g.map_lo : &g.map_hi,
                        fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        (void *)(w ? Xlo : Xhi), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      tc_err_slot() = "cuTensorMapEncodeTiled failed";
      return 1;
    }
  }
  g.hi = Xhi;
  g.lo = Xlo;
  g.fp16 = fp16;
  return 0;
}

// fp32 [m x ncov] view of out (row pitch ldo floats, a multiple of 4) for the TMA stores.
inline int tc_make_out_map(TcGemm &g, float *out, int64_t m, int64_t ncov, int64_t ldo) {
  cuuint64_t dims[2] = {(cuuint64_t)ncov, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)ldo * 4};
  cuuint32_t box[2] = {16u, 32u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = tc_encode_fn()(&g.map_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)out, dims, strides,
                              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tc_err_slot() = "cuTensorMapEncodeTiled (output) failed";
    return 1;
  }
  return 0;
}

// Launch over [i0, i0+m) x [j0, j0+ncov). rows = padded row count of Xhi/Xlo, dp = padded d.
// fp16: operands are the scaled fp16 split (rscale given), else the bf16 split. out must be
// 16-byte aligned with ldo % 4 == 0 (TMA store).
inline int tc_gemm_launch(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16,
                          const float *rscale, int64_t rows, int64_t dp, int64_t n, int64_t i0,
                          int64_t m, int64_t j0, int64_t ncov, const float *norms,
                          const KappaParams &kp, float *out, int64_t ldo, cudaStream_t st,
                          int64_t *launches) {
  if (g.hi != Xhi || g.lo != Xlo || g.fp16 != fp16)
    if (tc_make_maps(g, Xhi, Xlo, fp16, rows, dp)) return 1;
  if ((ldo & 3) || (reinterpret_cast<uintptr_t>(out) & 15)) {
    tc_err_slot() = "tcgen05 GEMM output needs 16-byte alignment and ldo % 4 == 0";
    return 1;
  }
  if (tc_make_out_map(g, out, m, ncov, ldo)) return 1;
  if (!g.attr) {
    if (cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM_V2) !=
        cudaSuccess) {
      tc_err_slot() = "cudaFuncSetAttribute(tc_gemm_kernel) failed";
      return 1;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
    g.attr = true;
  }
  const int tiles_m = (int)((m + TC_BM - 1) / TC_BM);
  const int tiles_n = (int)((ncov + TC_BN - 1) / TC_BN);
  const int64_t ntiles = (int64_t)tiles_m * tiles_n;
  const int grid = (int)(ntiles < g.num_sms ? ntiles : g.num_sms);
  tc_gemm_kernel<<<grid, TC_THREADS_V2, TC_SMEM_V2, st>>>(g.map_hi, g.map_lo, g.map_out, tc_idesc(fp16),
                                                          (int)(dp / TC_BK), n, i0, m, j0, ncov, norms,
                                                          fp16 ? rscale : nullptr, kp, tiles_m, tiles_n);
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace kkm
