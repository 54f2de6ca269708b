// tc2.cuh -- building blocks of the a1 tensor-core mainloop on CTA pairs (tcgen05 cta_group::2):
// the pair TMA producer, the UMMA instruction / commit helpers, the kappa row constants, and the
// work schedulers of the materialised GEMM, the streaming and the symmetric streaming kernels. The
// kernels themselves run the chained mainloop of chain.cuh (tc3.cuh, ssym.cuh).
//
// Why pairs: a 1-CTA M=128 x N=256 fp16x3 tile makes each SM's shared memory feed the tensor
// core ~96 B/clk of operands while the TMA writes the next stage at ~62 B/clk -- more than the
// 128 B/clk port. A cluster of 2 CTAs on one TPC runs M=256 x N=256 tiles: each CTA loads its
// 128 rows of A and its 128-row half of B, the leader CTA's single thread issues
// tcgen05.mma.cta_group::2 reading both CTAs' shared memory, and each CTA's TMEM receives its
// 128 output rows. Per SM: 64 B/clk MMA reads + 42 B/clk TMA writes, and half the L2 traffic.
// Stage ring: 3 stages x 64 KB per CTA (A_hi, A_lo, B_hi, B_lo halves); full[s] lives in the
// leader (both CTAs' TMA loads complete_tx on it), empty[s] in both CTAs (multicast commit).
#pragma once
#include "stream.cuh"

namespace kkm {

constexpr int T2_STAGES = 3;
constexpr uint32_t T2_HALF_BYTES = 128 * TC_BK * 2;            // 16 KB: 128 rows x 64 16-bit
constexpr uint32_t T2_STAGE_BYTES = 4 * T2_HALF_BYTES;          // A_hi, A_lo, B_hi, B_lo halves
constexpr int T2_BM = 256;                                      // rows per pair tile
constexpr int T2_GROUP_M = 16;                                  // raster groups of pair tiles

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
// TMA load whose completion is signalled on the leader CTA's barrier (peer bit cleared).
__device__ __forceinline__ void tma_load_2d_pair(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void umma2_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma2_commit_both(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// kind::f16 instruction descriptor for M = 256 (pair) x N = 256.
constexpr uint32_t t2_idesc(bool fp16) {
  return (1u << 4) | ((fp16 ? 0u : 1u) << 7) | ((fp16 ? 0u : 1u) << 10) | ((uint32_t)(256 >> 3) << 17) |
         ((uint32_t)(T2_BM >> 4) << 24);
}

struct T2Smem {
  uint8_t *stages;  // [T2_STAGES][A_hi | A_lo | B_hi | B_lo] x 16 KB, 1024-aligned
  uint64_t *full, *empty, *tfull, *tempty;
  uint32_t *tmem_slot;
};

// Carves the dynamic smem: stages, then `extra` bytes for the epilogue, then barriers.
__device__ __forceinline__ T2Smem t2_carve(uint8_t *smem_raw, uint32_t extra, uint8_t **extra_ptr) {
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  T2Smem s;
  s.stages = smem_raw + pad;
  *extra_ptr = s.stages + T2_STAGES * T2_STAGE_BYTES;
  s.full = reinterpret_cast<uint64_t *>(*extra_ptr + extra);
  s.empty = s.full + T2_STAGES;
  s.tfull = s.empty + T2_STAGES;
  s.tempty = s.tfull + 1;
  s.tmem_slot = reinterpret_cast<uint32_t *>(s.tempty + 1);
  return s;
}

// L2 policy of the operand loads: hint 0 normal / normal, 1 evict_last / evict_last, 2 evict_last /
// normal, 3 normal / evict_last, 4 evict_last / evict_first (A / B).
struct T2Policy {
  uint64_t a, b;
  __device__ __forceinline__ explicit T2Policy(int hint) {
    a = (hint == 1 || hint == 2 || hint == 4) ? l2_policy_evict_last() : l2_policy_evict_normal();
    b = (hint == 1 || hint == 3) ? l2_policy_evict_last() : hint == 4 ? l2_policy_evict_first() : l2_policy_evict_normal();
  }
};

// Producer body of one work item u (this CTA's halves of A and B through the stage ring).
template <class Sched>
__device__ __forceinline__ void t2_produce_item(const Sched &sc, const T2Smem &s, int64_t u, const CUtensorMap *a_hi,
                                                const CUtensorMap *a_lo, const CUtensorMap *b_hi,
                                                const CUtensorMap *b_lo, int nkb, uint32_t cr, const T2Policy &pol,
                                                int &stage, uint32_t &phase) {
  int ra, rb0, ntn;
  sc.item(u, ra, rb0, ntn);
  for (int t = 0; t < ntn; ++t) {
    const int rb = rb0 + t * 256;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait_backoff(&s.empty[stage], phase ^ 1);
      uint8_t *st = s.stages + stage * T2_STAGE_BYTES;
      if (cr == 0) mbar_arrive_expect_tx(&s.full[stage], 2 * T2_STAGE_BYTES);
      const int kc = kb * TC_BK;
      const int ar = ra + (int)cr * 128, br = rb + (int)cr * 128;
      tma_load_2d_pair(st, a_hi, kc, ar, &s.full[stage], pol.a);
      tma_load_2d_pair(st + T2_HALF_BYTES, a_lo, kc, ar, &s.full[stage], pol.a);
      tma_load_2d_pair(st + 2 * T2_HALF_BYTES, b_hi, kc, br, &s.full[stage], pol.b);
      tma_load_2d_pair(st + 3 * T2_HALF_BYTES, b_lo, kc, br, &s.full[stage], pol.b);
      if (++stage == T2_STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
}

// Producer (warp 0 lane 0 of both CTAs), static schedule: pair cl takes items cl, cl + ncl, ...
// Sched::item(u, ra, rb0, ntn): pair-tile A row base, first B row, number of 256-column tiles of
// work item u (B rows rb0 + t * 256).
template <class Sched>
__device__ __forceinline__ void t2_producer(const Sched &sc, const T2Smem &s, const CUtensorMap *a_hi,
                                            const CUtensorMap *a_lo, const CUtensorMap *b_hi,
                                            const CUtensorMap *b_lo, int nkb, uint32_t cr, int hint) {
  const T2Policy pol(hint);
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t u = cl; u < sc.nitems; u += ncl) t2_produce_item(sc, s, u, a_hi, a_lo, b_hi, b_lo, nkb, cr, pol, stage, phase);
}


// ---------------------------------------------------------------- fast epilogue math
// kappa of one 32-column chunk on packed pairs. In: v = main accumulator, w = correction
// accumulator (TMEM), cnj / crs = the chunk's per-column norms / rscale (smem). Row constants:
// rsi (1 / row scale, fp16 split), ni (row norm). No masking here: the caller zeroes invalid
// columns of partial chunks and patches the diagonal. Eqs. (b), (k); Gaussian per A1/A23.
struct RowK {
  float2 g;    // poly: gamma * rsi; linear: rsi; Gaussian: -rsi
  float2 c;    // poly: coef0; Gaussian: ni
  float scale; // Gaussian: -gamma * log2(e)
};

__device__ __forceinline__ RowK make_rowk(const KappaParams &kp, float rsi, float ni) {
  RowK r;
  if (kp.kind == 1) {
    r.g = make_float2(kp.gamma * rsi, kp.gamma * rsi);
    r.c = make_float2(kp.coef0, kp.coef0);
  } else if (kp.kind == 2) {  // n - b = fma(-rsi, t, n) with b = rsi t
    r.g = make_float2(-rsi, -rsi);
    r.c = make_float2(ni, ni);
  } else {
    r.g = make_float2(rsi, rsi);
    r.c = make_float2(0.f, 0.f);
  }
  r.scale = kp.neg_gamma_log2e;
  return r;
}

// ---------------------------------------------------------------- materialised GEMM
struct T2GemmSched {
  int64_t nitems;
  int tiles_m, tiles_n;  // pair tiles (256 rows) x 256-column tiles
  int64_t i0, j0, m, ncov;
  // the output region of work item u (one region: the kernel's tm_out / tm_out2, ridx = -1)
  __device__ __forceinline__ void region(int64_t u, int &tm, int &tn, int64_t &ri0, int64_t &rm, int64_t &rj0,
                                         int64_t &rncov, int &ridx) const {
    coords(u, tm, tn);
    ri0 = i0;
    rm = m;
    rj0 = j0;
    rncov = ncov;
    ridx = -1;
  }
  __device__ __forceinline__ void coords(int64_t u, int &tm, int &tn) const {
    const int64_t per_group = (int64_t)T2_GROUP_M * tiles_n;
    const int64_t g = u / per_group;
    const int first = (int)(g * T2_GROUP_M);
    const int gm = tiles_m - first < T2_GROUP_M ? tiles_m - first : T2_GROUP_M;
    const int64_t r = u - g * per_group;
    tm = first + (int)(r % gm);
    tn = (int)(r / gm);
  }
  __device__ __forceinline__ void item(int64_t u, int &ra, int &rb0, int &ntn) const {
    int tm, tn;
    coords(u, tm, tn);
    ra = (int)(i0 + (int64_t)tm * T2_BM);
    rb0 = (int)(j0 + (int64_t)tn * 256);
    ntn = 1;
  }
};

// Several output regions in one launch (the f1 band pieces): region r = rows [i0, i0 + m) x
// columns [j0, j0 + ncov) stored through the tensor map(s) omaps[r * planes + plane] (global
// memory); its tiles are work items [item0, item0 + tiles_m * tiles_n), row tiles fastest.
struct T2Region {
  int64_t i0, m, j0, ncov, item0;
  int32_t tiles_m, tiles_n;
};
struct T2MultiSched {
  int64_t nitems;
  int nreg;
  const T2Region *reg;
  __device__ __forceinline__ int find(int64_t u) const {
    int lo = 0, hi = nreg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (reg[mid].item0 <= u) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }
  __device__ __forceinline__ void region(int64_t u, int &tm, int &tn, int64_t &ri0, int64_t &rm, int64_t &rj0,
                                         int64_t &rncov, int &ridx) const {
    ridx = find(u);
    const T2Region g = reg[ridx];
    const int64_t lu = u - g.item0;
    tm = (int)(lu % g.tiles_m);
    tn = (int)(lu / g.tiles_m);
    ri0 = g.i0;
    rm = g.m;
    rj0 = g.j0;
    rncov = g.ncov;
  }
  __device__ __forceinline__ void item(int64_t u, int &ra, int &rb0, int &ntn) const {
    int tm, tn, r;
    int64_t i0, m, j0, nc;
    region(u, tm, tn, i0, m, j0, nc, r);
    ra = (int)(i0 + (int64_t)tm * T2_BM);
    rb0 = (int)(j0 + (int64_t)tn * 256);
    ntn = 1;
  }
};

// The diagonal pair tiles (u, u) of the n x n Gram matrix only: the tensor core's own x_i . x_i.
struct T2DiagSched {
  int64_t nitems, n;
  __device__ __forceinline__ void region(int64_t u, int &tm, int &tn, int64_t &ri0, int64_t &rm, int64_t &rj0,
                                         int64_t &rncov, int &ridx) const {
    tm = tn = (int)u;
    ri0 = rj0 = 0;
    rm = rncov = n;
    ridx = -1;
  }
  __device__ __forceinline__ void item(int64_t u, int &ra, int &rb0, int &ntn) const {
    ra = rb0 = (int)(u * T2_BM);
    ntn = 1;
  }
};

// ---------------------------------------------------------------- fused streaming kernel
// Work units of the full streaming kernel: (pair row tile, W column tiles) in a G-row supertile
// raster -- row groups of G pair tiles, each swept W column tiles at a time across its G rows --
// computed from the unit index (no table): unit u of group gi = u / (G ncb) is column block
// cb = r / gm, row gi G + r % gm (r = u - gi G ncb, gm = the group's rows, ncb = ceil(tiles_n / W)).
struct T2StreamSched {
  int64_t nitems;  // tiles_m * ncb
  int tiles_m, tiles_n, G, W, ncb;
  int64_t row0;
  int hint;        // 1: L2 evict_last on the operand loads
  __device__ __forceinline__ void unit(int64_t u, int &tm, int &tn0, int &ntn) const {
    const int64_t per_group = (int64_t)G * ncb;
    const int gi = (int)(u / per_group);
    const int64_t r = u - (int64_t)gi * per_group;
    const int gm = min(G, tiles_m - gi * G);
    const int cb = (int)(r / gm);
    tm = gi * G + (int)(r % gm);
    tn0 = cb * W;
    ntn = min(W, tiles_n - tn0);
  }
  __device__ __forceinline__ void item(int64_t u, int &ra, int &rb0, int &ntn) const {
    int tm, tn0;
    unit(u, tm, tn0, ntn);
    ra = (int)(row0 + (int64_t)tm * T2_BM);
    rb0 = tn0 * 256;
  }
};

// ---------------------------------------------------------------- f1: symmetric streaming
// A = B = the label-sorted points. Work unit u = units[u] = (tm, tn0, ntn, 0): pair row tile tm
// against the column tiles tn0 .. tn0 + ntn - 1 (tn0 >= tm: the upper triangle of the sorted
// K). Every tile adds its row sums by the column segments to Sfix[p][c] (rows p), and, unless
// it is a diagonal tile (tn == tm, whose row sums already cover both halves), its column sums
// by the row segments to Sfix[q][c] (columns q): K(p, q) = K(q, p). Sums are added in int64
// fixed point (value * 2^s, red.add: associative, so the result is bitwise independent of the
// order, of the grid and of the rank count).
struct T2SymSched {
  const int4 *units;
  int64_t nitems;
  int hint;  // L2 policy of the operand loads (t2_producer)
  __device__ __forceinline__ void item(int64_t u, int &ra, int &rb0, int &ntn) const {
    const int4 U = units[u];
    ra = U.x * T2_BM;
    rb0 = U.y * 256;
    ntn = U.z;
  }
};

// Reduce-scatter butterfly over the warp: returns, on lane l, the sum over the 32 lanes of
// t[l] (t is consumed). 31 shuffles; fixed order, deterministic.
__device__ __forceinline__ float lane_column_sum(float (&t)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < o; ++q) {
      const float send = up ? t[q] : t[q + o];
      const float keep = up ? t[q + o] : t[q];
      t[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return t[0];
}

__device__ __forceinline__ void red_add_s64(long long *p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace kkm
