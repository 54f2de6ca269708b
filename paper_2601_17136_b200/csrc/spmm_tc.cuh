// spmm_tc.cuh -- f4 low-precision K storage (the paper's mixed-precision future
// work P:875): a2 over the f1 upper-triangle bands (sym.cuh) stored in fp16, on the tensor cores.
//
// With K in a 16-bit type the SpMM's two reductions are dense contractions with 0/1 matrices:
//   row part:    S_row(i, c) += sum_j K(i, j) [cl_j = c]        = (K . Onehot_colsᵀ)(i, c)
//   column part: S_col(j, c) += sum_i K(i, j) [cl_i = c]        = (Kᵀ . Onehot_rowsᵀ)(j, c)
// (Eq. e with Eq. v, split by K's symmetry P:248 exactly as sym.cuh). One TMA-loaded smem tile of
// K (128 rows x 128 columns, fp16, 128-byte swizzle) is the A operand of BOTH tcgen05 MMAs: read
// K-major for the row sums (M = rows) and MN-major for the column sums (M = columns, Kᵀ) -- the
// same bytes, two descriptors. The 0/1 B operands (N = 16 labels) are built in shared memory from
// the labels. Accumulators live in TMEM (fp32); no per-element instruction touches K, so the
// kernel is a pure HBM stream of half the bytes of the fp32 bands.
//
// Work unit = (owned band, 512-row slab = 4 row tiles, split of <= 16 chunks of 128 columns).
// Per chunk: the 4 row tiles' row MMAs accumulate into D_row[tile] (over the unit's chunks), their
// column MMAs into D_col (over the 4 tiles; skipped on the diagonal block K_II, which the row
// part covers whole). D_col is drained per chunk to colpart[band][slab][c][column] and D_row at
// the unit's end to Srow[split][c][row] (fp32, both multiplied by 2^-e, the storage scale);
// ts_reduce_kernel sums them in fixed order (fp64), like sym_reduce.
//
// Warp roles (192 threads): warp 0 = producer (lane 0: unit scheduler + TMA; all lanes build the
// one-hot tiles), warp 1 = MMA issuer (lane 0) + TMEM owner, warps 2-5 = TMEM drains.
#pragma once
#include <cuda.h>

#include "gemm_tc.cuh"

namespace kkm {

constexpr int TS_TB = 1024;            // band height (rows) = SYM_TB
constexpr int TS_ROWS = 128;           // row tile
constexpr int TS_CH = 128;             // chunk columns
constexpr int TS_SLAB_TILES = 4;       // row tiles per unit (512 rows)
constexpr int TS_SPLIT_CHUNKS = 16;    // chunks per unit (2048 columns)
constexpr int TS_STAGES = 5;
constexpr uint32_t TS_TILE_BYTES = TS_ROWS * TS_CH * 2;  // 32 KB: 2 column halves x [128 rows x 128 B]
constexpr uint32_t TS_OH_BYTES = 16 * 128 * 2;           // one-hot: 2 halves x [16 labels x 128 B]
constexpr int TS_THREADS = 6 * 32;
constexpr int TS_TMEM_COLS = 256;  // D_row 2 x 64 + D_col 2 x 16

struct TsBand {
  int64_t koff;    // element offset of the band in the fp16 K buffer
  int64_t cpoff;   // float offset of the band's column partials [slabs][k][ldb - TB]
  int32_t band;    // band index I
  int32_t ldb;     // stored columns (row pitch, elements), ceil32(n - I TB)
  int32_t rows;    // stored rows, min(TB, n - I TB)
  int32_t nsplit;  // column splits
};
struct TsUnit {
  int32_t b, slab, q0, nq;  // owned-band index, 512-row slab, first chunk, chunks
};

// fp16 one-hot of 128 labels as a K-major, 128-byte-swizzled [16 x 128] UMMA operand (two 64-wide
// halves of 2 KB): element (c, e) = (lab_e == c). Lane l owns elements 4l .. 4l+3.
__device__ __forceinline__ void ts_build_onehot(uint8_t *dst, int4 l4, int lane) {
  const int e = 4 * lane;
  const int h = e >> 6, eh = e & 63;
  const int unit = eh >> 3, sub = (eh & 7) * 2;  // 16-B unit within the 128-B row, byte offset in it
  const uint16_t one = 0x3C00u;                   // fp16 1.0
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint32_t lo = (l4.x == c ? one : 0u) | ((l4.y == c ? one : 0u) << 16);
    const uint32_t hi = (l4.z == c ? one : 0u) | ((l4.w == c ? one : 0u) << 16);
    uint8_t *row = dst + h * 2048 + (c >> 3) * 1024 + (c & 7) * 128;
    *reinterpret_cast<uint2 *>(row + ((unit ^ (c & 7)) << 4) + sub) = make_uint2(lo, hi);
  }
}

__device__ __forceinline__ void ts_tma_load(void *smem_dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ts_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void ts_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// MN-major, 128-byte swizzle: 64-element MN blocks LBO bytes apart, 8-row K groups SBO = 1 KB.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
  tmem_wait_ld();
}

// kind::f16, fp16 A and B, fp32 D, M = 128, N = 16; a_mn: A is MN-major.
constexpr uint32_t ts_idesc(bool a_mn) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

struct TsSmem {
  uint8_t *stages;   // [TS_STAGES][32 KB]
  uint8_t *brow;     // [2][4 KB] one-hot of a chunk's column labels
  uint8_t *bcol;     // [2][4 tiles][4 KB] one-hot of a unit's row labels
  uint64_t *full, *empty, *browfull, *browempty, *bcolfull, *bcolempty, *dcolfull, *dcolempty, *drowfull,
      *drowempty;
  TsUnit *unit;      // [2]
  uint32_t *tmem_slot;
};

constexpr size_t TS_SMEM = 1024 + (size_t)TS_STAGES * TS_TILE_BYTES + 2 * TS_OH_BYTES +
                           2 * TS_SLAB_TILES * TS_OH_BYTES + 256;

__device__ __forceinline__ TsSmem ts_carve(uint8_t *raw) {
  const uint32_t a = smem_u32(raw);
  uint8_t *p = raw + (((a + 1023u) & ~1023u) - a);
  TsSmem s;
  s.stages = p;
  p += TS_STAGES * TS_TILE_BYTES;
  s.brow = p;
  p += 2 * TS_OH_BYTES;
  s.bcol = p;
  p += 2 * TS_SLAB_TILES * TS_OH_BYTES;
  uint64_t *b = reinterpret_cast<uint64_t *>(p);
  s.full = b;
  s.empty = b + TS_STAGES;
  s.browfull = s.empty + TS_STAGES;
  s.browempty = s.browfull + 2;
  s.bcolfull = s.browempty + 2;
  s.bcolempty = s.bcolfull + 2;
  s.dcolfull = s.bcolempty + 2;
  s.dcolempty = s.dcolfull + 2;
  s.drowfull = s.dcolempty + 2;
  s.drowempty = s.drowfull + 2;
  s.unit = reinterpret_cast<TsUnit *>(s.drowempty + 2);
  s.tmem_slot = reinterpret_cast<uint32_t *>(s.unit + 2);
  return s;
}

// maps[b]: fp16 [rows x ldb] view of owned band b, box {64 columns, 128 rows}, 128-byte swizzle
// (global memory, 64-B aligned). work[0], work[1]: zero between launches (reset at the end).
__global__ void __launch_bounds__(TS_THREADS, 1)
    spmm_tc_kernel(const CUtensorMap *__restrict__ maps, const TsBand *__restrict__ bands,
                   const TsUnit *__restrict__ units, int nunits, const int32_t *__restrict__ labels, int64_t n,
                   int k, int64_t rows_pad, float unscale, float *__restrict__ Srow, float *__restrict__ colpart,
                   int32_t *__restrict__ work) {
  extern __shared__ uint8_t smem_raw[];
  const TsSmem s = ts_carve(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TS_STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.browfull[i], 1);
      mbar_init(&s.browempty[i], 1);
      mbar_init(&s.bcolfull[i], 1);
      mbar_init(&s.bcolempty[i], 1 + 4);  // the MMA commit + the 4 drain warps
      mbar_init(&s.dcolfull[i], 1);
      mbar_init(&s.dcolempty[i], 4);
      mbar_init(&s.drowfull[i], 1);
      mbar_init(&s.drowempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s.tmem_slot)),
                 "n"(TS_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s.tmem_slot;

  if (warp == 0) {  // ---------------- producer
    int stage = 0;
    uint32_t sphase = 0;
    int64_t chunk_it = 0;
    for (int64_t uit = 0;; ++uit) {
      const int ub = (int)(uit & 1);
      const uint32_t uph = (uint32_t)(uit >> 1) & 1u;
      int ui = 0;
      if (lane == 0) ui = atomicAdd(work, 1);
      ui = __shfl_sync(0xffffffffu, ui, 0);
      mbar_wait(&s.bcolempty[ub], uph ^ 1u);
      if (ui >= nunits) {
        if (lane == 0) {
          s.unit[ub] = TsUnit{-1, 0, 0, 0};
          mbar_arrive(&s.bcolfull[ub]);
          if (atomicAdd(work + 1, 1) == (int)gridDim.x - 1) {  // last CTA past the end: reset
            work[0] = 0;
            work[1] = 0;
          }
        }
        break;
      }
      const TsUnit u = units[ui];
      const TsBand bd = bands[u.b];
      const int64_t g0 = (int64_t)bd.band * TS_TB;  // global index of band row / column 0
      const int r0 = u.slab * TS_SLAB_TILES * TS_ROWS;
      const int ntiles = min(TS_SLAB_TILES, (bd.rows - r0 + TS_ROWS - 1) / TS_ROWS);
      // row-label one-hots of the unit's tiles
      for (int t = 0; t < ntiles; ++t) {
        const int64_t r = g0 + r0 + t * TS_ROWS + 4 * lane;
        int4 l4;
        l4.x = r < n ? labels[r] : -1;
        l4.y = r + 1 < n ? labels[r + 1] : -1;
        l4.z = r + 2 < n ? labels[r + 2] : -1;
        l4.w = r + 3 < n ? labels[r + 3] : -1;
        ts_build_onehot(s.bcol + (ub * TS_SLAB_TILES + t) * TS_OH_BYTES, l4, lane);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        s.unit[ub] = u;
        mbar_arrive(&s.bcolfull[ub]);
      }
      const CUtensorMap *map = maps + u.b;
      for (int qi = 0; qi < u.nq; ++qi, ++chunk_it) {
        const int q = u.q0 + qi;
        const int rb = (int)(chunk_it & 1);
        mbar_wait(&s.browempty[rb], ((uint32_t)(chunk_it >> 1) & 1u) ^ 1u);
        const int64_t j = (int64_t)q * TS_CH + 4 * lane;  // band column
        int4 l4;
        l4.x = (j < bd.ldb && g0 + j < n) ? labels[g0 + j] : -1;
        l4.y = (j + 1 < bd.ldb && g0 + j + 1 < n) ? labels[g0 + j + 1] : -1;
        l4.z = (j + 2 < bd.ldb && g0 + j + 2 < n) ? labels[g0 + j + 2] : -1;
        l4.w = (j + 3 < bd.ldb && g0 + j + 3 < n) ? labels[g0 + j + 3] : -1;
        ts_build_onehot(s.brow + rb * TS_OH_BYTES, l4, lane);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&s.browfull[rb]);
          for (int t = 0; t < ntiles; ++t) {
            mbar_wait(&s.empty[stage], sphase ^ 1u);
            uint8_t *st = s.stages + stage * TS_TILE_BYTES;
            mbar_arrive_expect_tx(&s.full[stage], TS_TILE_BYTES);
            const int row = r0 + t * TS_ROWS;
            ts_tma_load(st, map, q * TS_CH, row, &s.full[stage]);
            ts_tma_load(st + TS_TILE_BYTES / 2, map, q * TS_CH + 64, row, &s.full[stage]);
            if (++stage == TS_STAGES) {
              stage = 0;
              sphase ^= 1u;
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t sphase = 0;
      int64_t chunk_it = 0, dcol_it = 0;
      constexpr uint32_t IROW = ts_idesc(false), ICOL = ts_idesc(true);
      for (int64_t uit = 0;; ++uit) {
        const int ub = (int)(uit & 1);
        const uint32_t uph = (uint32_t)(uit >> 1) & 1u;
        mbar_wait(&s.bcolfull[ub], uph);
        const TsUnit u = s.unit[ub];
        if (u.b < 0) break;
        const TsBand bd = bands[u.b];
        const int r0 = u.slab * TS_SLAB_TILES * TS_ROWS;
        const int ntiles = min(TS_SLAB_TILES, (bd.rows - r0 + TS_ROWS - 1) / TS_ROWS);
        mbar_wait(&s.drowempty[ub], uph ^ 1u);
        tc_fence_after();
        const uint32_t drow = tmem + (uint32_t)ub * 64u;
        const uint32_t bcol = smem_u32(s.bcol + ub * TS_SLAB_TILES * TS_OH_BYTES);
        for (int qi = 0; qi < u.nq; ++qi, ++chunk_it) {
          const int q = u.q0 + qi;
          const bool off = q * TS_CH >= TS_TB;  // the column part skips the diagonal block
          const int rb = (int)(chunk_it & 1);
          mbar_wait(&s.browfull[rb], (uint32_t)(chunk_it >> 1) & 1u);
          const int dc = (int)(dcol_it & 1);
          if (off) mbar_wait(&s.dcolempty[dc], ((uint32_t)(dcol_it >> 1) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t brow = smem_u32(s.brow + rb * TS_OH_BYTES);
          const uint32_t dcol = tmem + 128u + (uint32_t)dc * 16u;
          for (int t = 0; t < ntiles; ++t) {
            mbar_wait(&s.full[stage], sphase);
            tc_fence_after();
            const uint32_t a = smem_u32(s.stages + stage * TS_TILE_BYTES);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {  // row sums: K-major, k-steps over the 128 columns
              const uint32_t ko = (uint32_t)(ks >> 2) * (TS_TILE_BYTES / 2) + (uint32_t)(ks & 3) * 32u;
              const uint32_t bo = (uint32_t)(ks >> 2) * 2048u + (uint32_t)(ks & 3) * 32u;
              ts_mma(drow + (uint32_t)t * 16u, umma_desc_sw128(a + ko), umma_desc_sw128(brow + bo), IROW,
                     (qi > 0 || ks > 0) ? 1u : 0u);
            }
            if (off) {
              const uint32_t bc = bcol + (uint32_t)t * TS_OH_BYTES;
#pragma unroll
              for (int ks = 0; ks < 8; ++ks) {  // column sums: A = K^T (MN-major), k-steps over the rows
                const uint32_t bo = (uint32_t)(ks >> 2) * 2048u + (uint32_t)(ks & 3) * 32u;
                ts_mma(dcol, umma_desc_sw128_mn(a + (uint32_t)ks * 2048u, TS_TILE_BYTES / 2),
                       umma_desc_sw128(bc + bo), ICOL, (t > 0 || ks > 0) ? 1u : 0u);
              }
            }
            ts_commit(&s.empty[stage]);
            if (++stage == TS_STAGES) {
              stage = 0;
              sphase ^= 1u;
            }
          }
          ts_commit(&s.browempty[rb]);
          if (off) {
            ts_commit(&s.dcolfull[dc]);
            ++dcol_it;
          }
        }
        ts_commit(&s.drowfull[ub]);
        ts_commit(&s.bcolempty[ub]);
      }
    }
    __syncwarp();
  } else {  // ---------------- drains (warps 2-5: TMEM lane quarters)
    const int quarter = warp & 3;
    const uint32_t lq = (uint32_t)(quarter * 32) << 16;
    int64_t dcol_it = 0;
    for (int64_t uit = 0;; ++uit) {
      const int ub = (int)(uit & 1);
      const uint32_t uph = (uint32_t)(uit >> 1) & 1u;
      mbar_wait(&s.bcolfull[ub], uph);
      const TsUnit u = s.unit[ub];
      if (u.b < 0) break;
      const TsBand bd = bands[u.b];
      const int64_t g0 = (int64_t)bd.band * TS_TB;
      const int r0 = u.slab * TS_SLAB_TILES * TS_ROWS;
      const int ntiles = min(TS_SLAB_TILES, (bd.rows - r0 + TS_ROWS - 1) / TS_ROWS);
      const int64_t w = (int64_t)bd.ldb - TS_TB;
      for (int qi = 0; qi < u.nq; ++qi) {
        const int q = u.q0 + qi;
        if (q * TS_CH < TS_TB) continue;
        const int dc = (int)(dcol_it & 1);
        mbar_wait(&s.dcolfull[dc], (uint32_t)(dcol_it >> 1) & 1u);
        ++dcol_it;
        tc_fence_after();
        float v[16];
        tmem_ld16(tmem + 128u + (uint32_t)dc * 16u + lq, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.dcolempty[dc]);
        const int64_t jc = (int64_t)q * TS_CH + quarter * 32 + lane - TS_TB;  // off-diagonal column
        if (jc < w) {
          float *cp = colpart + bd.cpoff + (int64_t)u.slab * k * w + jc;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < k) cp[(int64_t)c * w] = v[c] * unscale;
        }
      }
      mbar_wait(&s.drowfull[ub], uph);
      tc_fence_after();
      const int p = u.q0 / TS_SPLIT_CHUNKS;
      for (int t = 0; t < ntiles; ++t) {
        float v[16];
        tmem_ld16(tmem + (uint32_t)ub * 64u + (uint32_t)t * 16u + lq, v);
        const int64_t row = g0 + r0 + t * TS_ROWS + quarter * 32 + lane;
        if (row < n) {  // Srow[p][c][row]: coalesced here and in ts_reduce_kernel
          float *o = Srow + (int64_t)p * k * rows_pad + row;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < k) o[(int64_t)c * rows_pad] = v[c] * unscale;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&s.drowempty[ub]);
        mbar_arrive(&s.bcolempty[ub]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TS_TMEM_COLS) : "memory");
  }
}

// One thread per (row i < rows_pad, label c = blockIdx.y); rows >= n get zeros. S[i][c] (fp64) =
// this rank's contributions to S(i, c): the row partials of its own band (splits in order) + the
// column partials (slabs in order) of the owned bands I' < band(i), in order.
__global__ void ts_reduce_kernel(const float *__restrict__ Srow, const float *__restrict__ colpart,
                                 const TsBand *__restrict__ bands, const int32_t *__restrict__ band_desc, int64_t n,
                                 int64_t rows_pad, int k, double *__restrict__ S) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= rows_pad) return;
  double acc = 0.0;
  if (i < n) {
    const int I = (int)(i / TS_TB);
    const int bi = band_desc[I];
    if (bi >= 0)
      for (int p = 0; p < bands[bi].nsplit; ++p) acc += (double)Srow[((int64_t)p * k + c) * rows_pad + i];
    for (int Ip = 0; Ip < I; ++Ip) {
      const int bp = band_desc[Ip];
      if (bp < 0) continue;
      const TsBand bd = bands[bp];
      const int64_t w = (int64_t)bd.ldb - TS_TB;
      const int64_t jc = i - (int64_t)Ip * TS_TB - TS_TB;
      const int slabs = (bd.rows + TS_SLAB_TILES * TS_ROWS - 1) / (TS_SLAB_TILES * TS_ROWS);
      for (int sl = 0; sl < slabs; ++sl) acc += (double)colpart[bd.cpoff + ((int64_t)sl * k + c) * w + jc];
    }
  }
  S[i * k + c] = acc;
}

// ---------------------------------------------------------------- host side
// fp16 [rows x ldb] band view for the a2 loads: box {64 columns, 128 rows}, 128-byte swizzle.
inline int ts_encode_band(CUtensorMap *m, const void *ptr, int64_t rows, int64_t ldb) {
  if (tc_encode_ready()) return 1;
  cuuint64_t dims[2] = {(cuuint64_t)ldb, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ldb * 2};
  cuuint32_t box[2] = {64u, 128u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = tc_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void *)ptr, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tc_err_slot() = "cuTensorMapEncodeTiled (fp16 band) failed";
    return 1;
  }
  return 0;
}

}  // namespace kkm
