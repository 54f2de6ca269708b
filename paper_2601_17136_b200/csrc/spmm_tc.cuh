// spmm_tc.cuh -- a2 on the tensor cores over the f1 upper-triangle bands (sym.cuh) stored in 16-bit
// planes: the default (kstore AUTO / FP16X2: hi = RN(K 2^e), lo = RN(K 2^e - hi), fp32-class) and
// f4's low-precision storage (FP16: hi only, the paper's mixed-precision future
// work P:875).
//
// With K in a 16-bit type the SpMM's two reductions are dense contractions with 0/1 matrices:
//   row part:    S_row(i, c) += sum_j K(i, j) [cl_j = c]        = (K . Onehot_colsᵀ)(i, c)
//   column part: S_col(j, c) += sum_i K(i, j) [cl_i = c]        = (Kᵀ . Onehot_rowsᵀ)(j, c)
// (Eq. e with Eq. v, split by K's symmetry P:248 exactly as sym.cuh). One TMA-loaded smem tile of
// K (128 rows x 128 columns, fp16, 128-byte swizzle) is the A operand of BOTH tcgen05 MMAs: read
// K-major for the row sums (M = rows) and MN-major for the column sums (M = columns, Kᵀ) -- the
// same bytes, two descriptors. The 0/1 B operands (N = 16 labels) are built in shared memory from
// the labels. Accumulators live in TMEM (fp32); no per-element instruction touches K, so the
// kernel is a pure HBM stream (hi + lo: the fp32 band bytes at ~0.97 of the copy peak; FP16:
// half of them). Both planes of a tile are fed as two stages into the same accumulators, lo first.
//
// Work unit = (owned band piece, 512-row slab = 4 row tiles, split of <= 8 or 16 chunks of 128 columns).
// Per chunk and row tile the row MMAs go to D_row[tile] and the column MMAs to D_col (skipped on
// the diagonal block K_II, which the row part covers whole); an accumulator holds 2 chunks (row
// sums) or 2 row tiles (column sums) and is then drained into fp64 registers: the column sums of
// a chunk over the slab's tiles and the row sums over the unit's chunks are added to S of their
// points as int64 fixed point (value x 2^-e x 2^s, `red.global.add.u64`): integer addition is
// associative, so S is bitwise independent of the schedule and of the rank count (as the
// streaming f1 kernel), and no partial arrays or reduction kernel are needed.
//
// Warp roles (224 threads): warp 0 = producer (lane 0: unit scheduler + TMA; all lanes build the
// one-hot tiles), warp 1 = row-sum MMA issuer (lane 0) + TMEM owner, warps 2-5 = TMEM drains,
// warp 6 = column-sum MMA issuer (lane 0).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "gemm_tc.cuh"

namespace kkm {

#ifndef KKM_TS_PROMO
#define KKM_TS_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
constexpr int TS_TB = 1024;            // band height (rows) = SYM_TB
constexpr int TS_ROWS = 128;           // row tile
constexpr int TS_CH = 128;             // chunk columns
constexpr int TS_SLAB_TILES = 4;       // row tiles per unit (512 rows)
constexpr uint32_t TS_TILE_BYTES = TS_ROWS * TS_CH * 2;  // 32 KB: 2 column halves x [128 rows x 128 B]
constexpr int TS_THREADS = 7 * 32;
constexpr int TS_COL_WARP = 6;     // the column-sum MMA issuer
constexpr int TS_DR_BUF = 3;       // D_row buffers (chunks in flight between the MMA and the drains)
constexpr int TS_DC_BUF = 4;       // D_col buffers (tiles in flight)
constexpr int TS_MAX_K = 32;       // labels of one launch: NL = 16 (k <= 16) or 32 (k <= 32)

// Per label count NL: one-hot operand bytes (2 halves x [NL labels x 128 B]), stage ring depth (the
// one-hots of a unit grow with NL), TMEM columns (D_row 3 x (4 tiles x NL) + D_col 4 x NL).
template <int NL>
struct TsCfg {
  static constexpr uint32_t OH_BYTES = NL * 128 * 2;
  static constexpr int STAGES = NL == 16 ? 5 : 4;
  static constexpr int TMEM_COLS = NL == 16 ? 256 : 512;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * TS_TILE_BYTES + 2 * OH_BYTES +
                                 2 * TS_SLAB_TILES * OH_BYTES + 512;  // + barriers, units, TMEM slot
};

struct TsBand {    // a stored piece of band I: rows [I TB + row0, + rows) x columns [I TB, + ldb)
  int64_t koff;    // element offset of the piece in the fp16 K buffer (per plane)
  int64_t cpoff;   // NL = 32: float offset of its slabs' column partials ([slab][NL][ldb - TB]), else 0
  int32_t band;    // band index I
  int32_t row0;    // first row of the piece within the band (0 or 512)
  int32_t ldb;     // stored columns (row pitch, elements), ceil128(n - I TB)
  int32_t rows;    // stored rows (<= 512 when the rank holds 512-row pieces)
  int32_t nsplit;  // column splits
};
struct TsUnit {
  int32_t b, slab, q0, nq;  // owned-band index, 512-row slab, first chunk, chunks
};

// fp16 one-hot of 128 labels as a K-major, 128-byte-swizzled [NL x 128] UMMA operand (two 64-wide
// halves of NL x 128 B): element (c, e) = (lab_e == c). Lane l owns elements 4l .. 4l+3.
template <int NL>
__device__ __forceinline__ void ts_build_onehot(uint8_t *dst, int4 l4, int lane) {
  const int e = 4 * lane;
  const int h = e >> 6, eh = e & 63;
  const int unit = eh >> 3, sub = (eh & 7) * 2;  // 16-B unit within the 128-B row, byte offset in it
  const uint16_t one = 0x3C00u;                   // fp16 1.0
#pragma unroll
  for (int c = 0; c < NL; ++c) {
    const uint32_t lo = (l4.x == c ? one : 0u) | ((l4.y == c ? one : 0u) << 16);
    const uint32_t hi = (l4.z == c ? one : 0u) | ((l4.w == c ? one : 0u) << 16);
    uint8_t *row = dst + h * (NL * 128) + (c >> 3) * 1024 + (c & 7) * 128;
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
__device__ __forceinline__ void ts_red_add(long long *p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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

// kind::f16, fp16 A and B, fp32 D, M = 128, N = NL; a_mn: A is MN-major.
constexpr uint32_t ts_idesc(bool a_mn, int nl) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((uint32_t)(nl >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
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

template <int NL>
__device__ __forceinline__ TsSmem ts_carve(uint8_t *raw) {
  constexpr int TS_STAGES = TsCfg<NL>::STAGES;
  constexpr uint32_t TS_OH_BYTES = TsCfg<NL>::OH_BYTES;
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
  s.dcolempty = s.dcolfull + TS_DC_BUF;
  s.drowfull = s.dcolempty + TS_DC_BUF;
  s.drowempty = s.drowfull + TS_DR_BUF;
  s.unit = reinterpret_cast<TsUnit *>(s.drowempty + TS_DR_BUF);
  s.tmem_slot = reinterpret_cast<uint32_t *>(s.unit + 2);
  return s;
}

// maps[b * planes + pl]: fp16 [rows x ldb] view of plane pl (hi, lo) of owned band b, box {64
// columns, 128 rows}, 128-byte swizzle (global memory, 64-B aligned); both planes of a tile
// accumulate into the same TMEM sums. work[0], work[1]: zero between launches (reset at the end).
// NL = 16 (k <= 16): column sums added to Sfix (int64 red.add per column and label);
// NL = 32 (16 < k <= 32): written to colpart (fp32, [slab][label][column], each entry once) and
// summed over the slabs by ts_colpart_reduce_kernel -- 2x the labels would double the per-column
// atomics, while the partials cost ~6 % of the band bytes each way.
template <int NL>
__global__ void __launch_bounds__(TS_THREADS, 1)
    spmm_tc_kernel(const CUtensorMap *__restrict__ maps, const TsBand *__restrict__ bands,
                   const TsUnit *__restrict__ units, int nunits, const int32_t *__restrict__ labels, int64_t n,
                   int k, int64_t rows_pad, double fxm, long long *__restrict__ Sfix,
                   int32_t *__restrict__ work, int planes, float *__restrict__ colpart) {
  constexpr int TS_STAGES = TsCfg<NL>::STAGES;
  constexpr uint32_t TS_OH_BYTES = TsCfg<NL>::OH_BYTES;
  constexpr int TS_TMEM_COLS = TsCfg<NL>::TMEM_COLS;
  constexpr uint32_t DR_COLS = TS_SLAB_TILES * NL;  // one D_row buffer: the slab's tiles x NL labels
  extern __shared__ uint8_t smem_raw[];
  const TsSmem s = ts_carve<NL>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TS_STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 2);  // both MMA issuers commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.browfull[i], 1);
      mbar_init(&s.browempty[i], 1);
      mbar_init(&s.bcolfull[i], 1);
      mbar_init(&s.bcolempty[i], 2 + 4);  // the 2 MMA issuers' commits + the 4 drain warps
    }
    for (int i = 0; i < TS_DC_BUF; ++i) {
      mbar_init(&s.dcolfull[i], 1);
      mbar_init(&s.dcolempty[i], 4);
    }
    for (int i = 0; i < TS_DR_BUF; ++i) {
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
        const int64_t r = g0 + bd.row0 + r0 + t * TS_ROWS + 4 * lane;
        int4 l4;
        l4.x = r < n ? labels[r] : -1;
        l4.y = r + 1 < n ? labels[r + 1] : -1;
        l4.z = r + 2 < n ? labels[r + 2] : -1;
        l4.w = r + 3 < n ? labels[r + 3] : -1;
        ts_build_onehot<NL>(s.bcol + (ub * TS_SLAB_TILES + t) * TS_OH_BYTES, l4, lane);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        s.unit[ub] = u;
        mbar_arrive(&s.bcolfull[ub]);
      }
      const CUtensorMap *map = maps + (int64_t)u.b * planes;
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
        ts_build_onehot<NL>(s.brow + rb * TS_OH_BYTES, l4, lane);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&s.browfull[rb]);
          for (int t = 0; t < ntiles; ++t)
            for (int pl = 0; pl < planes; ++pl) {
              mbar_wait(&s.empty[stage], sphase ^ 1u);
              uint8_t *st = s.stages + stage * TS_TILE_BYTES;
              mbar_arrive_expect_tx(&s.full[stage], TS_TILE_BYTES);
              const int row = r0 + t * TS_ROWS;
              // the lo plane first: its small sums reach the accumulator while the running sum is
              // still small, so only the hi plane's MMAs add truncation error relative to S (A9)
              const CUtensorMap *pm = map + (planes - 1 - pl);
              ts_tma_load(st, pm, q * TS_CH, row, &s.full[stage]);
              ts_tma_load(st + TS_TILE_BYTES / 2, pm, q * TS_CH + 64, row, &s.full[stage]);
              if (++stage == TS_STAGES) {
                stage = 0;
                sphase ^= 1u;
              }
            }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 || warp == TS_COL_WARP) {  // ---------------- MMA issuers
    // warp 1 issues the row-sum MMAs, warp 6 the column-sum MMAs (one thread each: the issue
    // rate of a single thread limited the kernel). A TMEM accumulator sums at most 2 chunks (row
    // sums) or 2 row tiles (column sums), i.e. <= 16 k-steps x planes MMAs, before it is
    // drained: the tensor core rounds every accumulation to the running fp32 sum, and over a
    // whole 2048-column unit the one-signed part of that error reached ~3e-6 of S (J 1.1e-5 off
    // at HAR); the drains add in fp64 instead (DESIGN A9, §5.5b).
    const bool rowp = warp == 1;
    if (lane == 0) {
      int stage = 0;
      uint32_t sphase = 0;
      int64_t chunk_it = 0, dcol_it = 0, drow_it = 0;
      constexpr uint32_t IROW = ts_idesc(false, NL), ICOL = ts_idesc(true, NL);
      for (int64_t uit = 0;; ++uit) {
        const int ub = (int)(uit & 1);
        const uint32_t uph = (uint32_t)(uit >> 1) & 1u;
        mbar_wait(&s.bcolfull[ub], uph);
        const TsUnit u = s.unit[ub];
        if (u.b < 0) break;
        const TsBand bd = bands[u.b];
        const int r0 = u.slab * TS_SLAB_TILES * TS_ROWS;
        const int ntiles = min(TS_SLAB_TILES, (bd.rows - r0 + TS_ROWS - 1) / TS_ROWS);
        const uint32_t bcol = smem_u32(s.bcol + ub * TS_SLAB_TILES * TS_OH_BYTES);
        for (int qi = 0; qi < u.nq; ++qi, ++chunk_it) {
          const int q = u.q0 + qi;
          const bool off = q * TS_CH >= TS_TB;  // the column part skips the diagonal block
          const int rb = (int)(chunk_it & 1);
          const int db = (int)(drow_it % TS_DR_BUF);
          const bool rfirst = (qi & 1) == 0, rlast = (qi & 1) == 1 || qi == u.nq - 1;
          if (rowp) {
            mbar_wait(&s.browfull[rb], (uint32_t)(chunk_it >> 1) & 1u);
            if (rfirst) mbar_wait(&s.drowempty[db], ((uint32_t)(drow_it / TS_DR_BUF) & 1u) ^ 1u);
            tc_fence_after();
          }
          const uint64_t brd = umma_desc_sw128(smem_u32(s.brow + rb * TS_OH_BYTES));
          const uint32_t drow = tmem + (uint32_t)db * DR_COLS;
          for (int t = 0; t < ntiles; ++t) {
            const int dc = (int)(dcol_it % TS_DC_BUF);
            const bool cfirst = (t & 1) == 0, clast = (t & 1) == 1 || t == ntiles - 1;
            const bool colp = !rowp && off;
            if (colp && cfirst) {
              mbar_wait(&s.dcolempty[dc], ((uint32_t)(dcol_it / TS_DC_BUF) & 1u) ^ 1u);
              tc_fence_after();
            }
            const uint32_t dcol = tmem + (uint32_t)(TS_DR_BUF * DR_COLS) + (uint32_t)dc * NL;
            const uint64_t bcd = umma_desc_sw128(bcol + (uint32_t)t * TS_OH_BYTES);
            for (int pl = 0; pl < planes; ++pl) {
              mbar_wait(&s.full[stage], sphase);
              tc_fence_after();
              // descriptors: one per operand, the k-steps add their (address >> 4) offsets
              const uint32_t a = smem_u32(s.stages + stage * TS_TILE_BYTES);
              if (rowp) {
                const uint64_t ad = umma_desc_sw128(a);
                const uint32_t acc0 = (!rfirst || pl > 0) ? 1u : 0u;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {  // row sums: K-major, k-steps over the 128 columns
                  const uint32_t ko = ((uint32_t)(ks >> 2) * (TS_TILE_BYTES / 2) + (uint32_t)(ks & 3) * 32u) >> 4;
                  const uint32_t bo = ((uint32_t)(ks >> 2) * (NL * 128u) + (uint32_t)(ks & 3) * 32u) >> 4;
                  ts_mma(drow + (uint32_t)t * NL, ad + ko, brd + bo, IROW, ks > 0 ? 1u : acc0);
                }
              } else if (colp) {
                const uint64_t amn = umma_desc_sw128_mn(a, TS_TILE_BYTES / 2);
                const uint32_t acc0 = (!cfirst || pl > 0) ? 1u : 0u;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {  // column sums: A = K^T (MN-major), k-steps over the rows
                  const uint32_t bo = ((uint32_t)(ks >> 2) * (NL * 128u) + (uint32_t)(ks & 3) * 32u) >> 4;
                  ts_mma(dcol, amn + (uint32_t)ks * (2048u >> 4), bcd + bo, ICOL, ks > 0 ? 1u : acc0);
                }
              }
              ts_commit(&s.empty[stage]);  // (arrives at once when this thread issued no MMA)
              if (++stage == TS_STAGES) {
                stage = 0;
                sphase ^= 1u;
              }
            }
            if (colp && clast) ts_commit(&s.dcolfull[dc]);
            if (off && clast) ++dcol_it;
          }
          if (rowp) {
            ts_commit(&s.browempty[rb]);
            if (rlast) ts_commit(&s.drowfull[db]);
          }
          if (rlast) ++drow_it;
        }
        ts_commit(&s.bcolempty[ub]);
      }
    }
    __syncwarp();
  } else if (warp < TS_COL_WARP) {  // ---------------- drains (warps 2-5: TMEM lane quarters), fp64 sums
    const int quarter = warp & 3;
    const uint32_t lq = (uint32_t)(quarter * 32) << 16;
    int64_t dcol_it = 0, drow_it = 0;
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
      // fp64 for 16 labels; fp32 (RN adds of <= 8 drained chunk-pair sums) for 32, where fp64 would not
      // fit the registers
      using RT = typename std::conditional<NL == 16, double, float>::type;
      RT racc[TS_SLAB_TILES][NL];
#pragma unroll
      for (int t = 0; t < TS_SLAB_TILES; ++t)
#pragma unroll
        for (int c = 0; c < NL; ++c) racc[t][c] = RT(0);
      for (int qi = 0; qi < u.nq; ++qi) {
        const int q = u.q0 + qi;
        if (q * TS_CH >= TS_TB) {  // the column sums of the chunk over the slab's tiles (pairs)
          RT cacc[NL];
#pragma unroll
          for (int c = 0; c < NL; ++c) cacc[c] = RT(0);
          for (int t = 0; t < ntiles; t += 2, ++dcol_it) {
            const int dc = (int)(dcol_it % TS_DC_BUF);
            mbar_wait(&s.dcolfull[dc], (uint32_t)(dcol_it / TS_DC_BUF) & 1u);
            tc_fence_after();
#pragma unroll
            for (int g = 0; g < NL / 16; ++g) {
              float v[16];
              tmem_ld16(tmem + (uint32_t)(TS_DR_BUF * DR_COLS) + (uint32_t)dc * NL + 16u * g + lq, v);
#pragma unroll
              for (int c = 0; c < 16; ++c) cacc[16 * g + c] += (RT)v[c];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.dcolempty[dc]);
          }
          const int64_t jc = (int64_t)q * TS_CH + quarter * 32 + lane - TS_TB;  // off-diagonal column
          if (jc < w) {  // the point g0 + TB + jc of a later band: its column part
            if (NL == 16) {
              long long *o = Sfix + g0 + TS_TB + jc;
#pragma unroll
              for (int c = 0; c < NL; ++c)
                if (c < k) ts_red_add(o + (int64_t)c * rows_pad, __double2ll_rn((double)cacc[c] * fxm));
            } else {  // [slab][label][column] partials of this piece's slab (u.slab)
              float *o = colpart + bd.cpoff + (int64_t)u.slab * NL * w + jc;
#pragma unroll
              for (int c = 0; c < NL; ++c) o[(int64_t)c * w] = (float)cacc[c];
            }
          }
        }
        if ((qi & 1) == 1 || qi == u.nq - 1) {  // the row sums of a chunk pair
          const int db = (int)(drow_it % TS_DR_BUF);
          mbar_wait(&s.drowfull[db], (uint32_t)(drow_it / TS_DR_BUF) & 1u);
          ++drow_it;
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < TS_SLAB_TILES; ++t)
            if (t < ntiles) {
#pragma unroll
              for (int g = 0; g < NL / 16; ++g) {
                float v[16];
                tmem_ld16(tmem + (uint32_t)db * DR_COLS + (uint32_t)t * NL + 16u * g + lq, v);
#pragma unroll
                for (int c = 0; c < 16; ++c) racc[t][16 * g + c] += (RT)v[c];
              }
            }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.drowempty[db]);
        }
      }
#pragma unroll
      for (int t = 0; t < TS_SLAB_TILES; ++t) {
        const int64_t row = g0 + bd.row0 + r0 + t * TS_ROWS + quarter * 32 + lane;
        if (t < ntiles && row < n) {  // the row part
#pragma unroll
          for (int c = 0; c < NL; ++c)
            if (c < k) ts_red_add(Sfix + (int64_t)c * rows_pad + row, __double2ll_rn((double)racc[t][c] * fxm));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.bcolempty[ub]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TS_TMEM_COLS) : "memory");
  }
}

// NL = 32: the column parts. Slabs of this rank sorted by colstart (= band start + TB): partials
// colpart[off + c w + (j - colstart)] for the points j >= colstart of later bands. Thread (4 points
// j0 .. j0 + 3, label c) sums its slabs in that fixed order (fp64) and adds the totals to Sfix[c][j]
// (int64 fixed point). colstart, w and off are multiples of 128 floats, so the 4 points share their
// slab set and every partial load is one aligned float4.
struct TsSlab {
  int64_t colstart, w, off;
};
__global__ void ts_colpart_reduce_kernel(const float *__restrict__ colpart, const TsSlab *__restrict__ slabs,
                                         int nslab, int64_t n, int k, int64_t rows_pad, double fxm,
                                         long long *__restrict__ Sfix) {
  const int64_t j0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  const int c = blockIdx.y;
  if (j0 >= n || c >= k) return;
  // the slabs with colstart <= j0 are a prefix [0, qe) of the sorted table: bound it first, so the
  // loop below has no data-dependent exit and its independent partial loads are issued 8 at a
  // time (with an early exit each thread walked its slabs one dependent load after another:
  // ~240 us at config 2, k = 32, for ~0.46 GB)
  int lo = 0, hi = nslab;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&slabs[mid].colstart) <= j0) lo = mid + 1;
    else hi = mid;
  }
  const int qe = lo;
  if (qe == 0) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 8
  for (int q = 0; q < qe; ++q) {
    const int64_t off = __ldg(&slabs[q].off), w = __ldg(&slabs[q].w), cs = __ldg(&slabs[q].colstart);
    const float4 v = __ldcs(reinterpret_cast<const float4 *>(colpart + off + (int64_t)c * w + (j0 - cs)));
    s0 += (double)v.x;
    s1 += (double)v.y;
    s2 += (double)v.z;
    s3 += (double)v.w;
  }
  long long *o = Sfix + (int64_t)c * rows_pad + j0;
  ts_red_add(o, __double2ll_rn(s0 * fxm));
  if (j0 + 1 < n) ts_red_add(o + 1, __double2ll_rn(s1 * fxm));
  if (j0 + 2 < n) ts_red_add(o + 2, __double2ll_rn(s2 * fxm));
  if (j0 + 3 < n) ts_red_add(o + 3, __double2ll_rn(s3 * fxm));
}

// Sfix[c][row] (int64 fixed point, label-major) -> Sout[row][c]: int64 (Sint, for an exact
// ReduceScatter over ranks) or fp64 times inv (Sd); rows >= n give 0.
__global__ void ts_fix_out_kernel(const long long *__restrict__ Sfix, int64_t n, int64_t rows_pad, int k,
                                  double inv, long long *__restrict__ Sint, double *__restrict__ Sd) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows_pad * k) return;
  const int64_t i = t / k;
  const int c = (int)(t % k);
  const long long v = i < n ? Sfix[(int64_t)c * rows_pad + i] : 0ll;
  if (Sint) Sint[t] = v;
  if (Sd) Sd[t] = (double)v * inv;
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
                              (CUtensorMapL2promotion)KKM_TS_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tc_err_slot() = "cuTensorMapEncodeTiled (fp16 band) failed";
    return 1;
  }
  return 0;
}

}  // namespace kkm
