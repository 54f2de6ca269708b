// tc2.cuh -- the a1 tensor-core mainloop on CTA pairs (tcgen05 cta_group::2) for both the
// materialised GEMM (store epilogue) and the fused streaming kernel (segmented-sum epilogue).
//
// Why pairs: a 1-CTA M=128 x N=256 fp16x3 tile makes each SM's shared memory feed the tensor
// core ~96 B/clk of operands while the TMA writes the next stage at ~62 B/clk -- more than the
// 128 B/clk port. A cluster of 2 CTAs on one TPC runs M=256 x N=256 tiles: each CTA loads its
// 128 rows of A and its 128-row half of B, the leader CTA's single thread issues
// tcgen05.mma.cta_group::2 reading both CTAs' shared memory, and each CTA's TMEM receives its
// 128 output rows. Per SM: 64 B/clk MMA reads + 42 B/clk TMA writes, and half the L2 traffic.
//
// Pipeline: 3 stages x 64 KB per CTA; full[s] lives in the leader (both CTAs'
// TMA loads complete_tx on it), empty[s] / tfull in both CTAs (multicast tcgen05.commit),
// tempty in the leader (16 epilogue-warp arrivals, the peer's through mapa). TMEM per CTA:
// hi*hi main accumulator [0,256) + hi*lo + lo*hi correction accumulator [256,512).
#pragma once
#include "stream.cuh"

namespace kkm {

constexpr int T2_STAGES = 3;
constexpr uint32_t T2_HALF_BYTES = 128 * TC_BK * 2;            // 16 KB: 128 rows x 64 16-bit
constexpr uint32_t T2_STAGE_BYTES = 4 * T2_HALF_BYTES;          // A_hi, A_lo, B_hi, B_lo halves
constexpr int T2_THREADS = (2 + TC_EPI_WARPS) * 32;
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

__device__ __forceinline__ void t2_setup(const T2Smem &s, int warp, uint32_t tempty_count = 2 * TC_EPI_WARPS) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < T2_STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    mbar_init(s.tfull, 1);
    mbar_init(s.tempty, tempty_count);  // every epilogue warp of both CTAs arrives
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(s.tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
}

__device__ __forceinline__ void t2_teardown(const T2Smem &s, int warp, uint32_t tmem_base) {
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's smem
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// Producer (warp 0 lane 0 of both CTAs). Sched::item(u, ra, rb0, ntn): pair-tile A row base,
// first B row, number of 256-column tiles of work item u (B rows rb0 + t * 256).
template <class Sched>
__device__ __forceinline__ void t2_producer(const Sched &sc, const T2Smem &s, const CUtensorMap *a_hi,
                                            const CUtensorMap *a_lo, const CUtensorMap *b_hi,
                                            const CUtensorMap *b_lo, int nkb, uint32_t cr, int hint) {
  const uint64_t keep = hint ? l2_policy_evict_last() : l2_policy_evict_normal();
  const uint64_t bpol = keep;  // (evict_normal on the streaming B measured slower)
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t u = cl; u < sc.nitems; u += ncl) {
    int ra, rb0, ntn;
    sc.item(u, ra, rb0, ntn);
    for (int t = 0; t < ntn; ++t) {
      const int rb = rb0 + t * 256;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&s.empty[stage], phase ^ 1);
        uint8_t *st = s.stages + stage * T2_STAGE_BYTES;
        if (cr == 0) mbar_arrive_expect_tx(&s.full[stage], 2 * T2_STAGE_BYTES);
        const int kc = kb * TC_BK;
        const int ar = ra + (int)cr * 128, br = rb + (int)cr * 128;
        tma_load_2d_pair(st, a_hi, kc, ar, &s.full[stage], keep);
        tma_load_2d_pair(st + T2_HALF_BYTES, a_lo, kc, ar, &s.full[stage], keep);
        tma_load_2d_pair(st + 2 * T2_HALF_BYTES, b_hi, kc, br, &s.full[stage], bpol);
        tma_load_2d_pair(st + 3 * T2_HALF_BYTES, b_lo, kc, br, &s.full[stage], bpol);
        if (++stage == T2_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
}

// MMA issuer (warp 1 lane 0 of the leader CTA).
template <class Sched>
__device__ __forceinline__ void t2_mma(const Sched &sc, const T2Smem &s, int nkb, uint32_t idesc,
                                       uint32_t tmem_base) {
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  int stage = 0;
  uint32_t phase = 0;
  int64_t it = 0;
  const uint32_t d_main = tmem_base, d_corr = tmem_base + 256u;
  for (int64_t u = cl; u < sc.nitems; u += ncl) {
    int ra, rb0, ntn;
    sc.item(u, ra, rb0, ntn);
    for (int t = 0; t < ntn; ++t, ++it) {
      mbar_wait(s.tempty, (uint32_t)(it & 1) ^ 1u);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&s.full[stage], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(s.stages + stage * T2_STAGE_BYTES);
        const uint32_t a_hi = st, a_lo = st + T2_HALF_BYTES;
        const uint32_t b_hi = st + 2 * T2_HALF_BYTES, b_lo = st + 3 * T2_HALF_BYTES;
#pragma unroll
        for (int k = 0; k < TC_BK / 16; ++k) {
          const uint32_t ko = (uint32_t)k * 32u;
          const uint32_t acc = (kb == 0 && k == 0) ? 0u : 1u;
          umma2_f16(d_corr, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_lo + ko), idesc, acc);
          umma2_f16(d_corr, umma_desc_sw128(a_lo + ko), umma_desc_sw128(b_hi + ko), idesc, 1u);
          umma2_f16(d_main, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_hi + ko), idesc, acc);
        }
        umma2_commit_both(&s.empty[stage]);
        if (++stage == T2_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma2_commit_both(s.tfull);
    }
  }
}


// ---------------------------------------------------------------- fast epilogue math
// kappa of one 32-column chunk on packed pairs. In: v = main accumulator, w = correction
// accumulator (TMEM), cnj / crs = the chunk's per-column norms / rscale (smem). Row constants:
// rsi (1 / row scale, fp16 split), ni (row norm). No masking here: the caller zeroes invalid
// columns of partial chunks and patches the diagonal. Eqs. (b), (k); Gaussian per A1/A23.
struct RowK {
  float2 g;    // poly: gamma * rsi; linear: rsi; Gaussian: -2 * rsi
  float2 c;    // poly: coef0; Gaussian: ni
  float scale; // Gaussian: -gamma * log2(e)
};

__device__ __forceinline__ RowK make_rowk(const KappaParams &kp, float rsi, float ni) {
  RowK r;
  if (kp.kind == 1) {
    r.g = make_float2(kp.gamma * rsi, kp.gamma * rsi);
    r.c = make_float2(kp.coef0, kp.coef0);
  } else if (kp.kind == 2) {
    r.g = make_float2(-2.f * rsi, -2.f * rsi);
    r.c = make_float2(ni, ni);
  } else {
    r.g = make_float2(rsi, rsi);
    r.c = make_float2(0.f, 0.f);
  }
  r.scale = kp.neg_gamma_log2e;
  return r;
}

__device__ __forceinline__ void kappa_chunk(float (&v)[32], const float (&w)[32], const float *cnj,
                                            const float *crs, const KappaParams &kp, const RowK &rk) {
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    const float4 rj = reinterpret_cast<const float4 *>(crs)[q4];
    const float2 r01 = make_float2(rj.x, rj.y), r23 = make_float2(rj.z, rj.w);
    float2 t01 = f2mul(f2add(make_float2(v[4 * q4], v[4 * q4 + 1]), make_float2(w[4 * q4], w[4 * q4 + 1])), r01);
    float2 t23 = f2mul(f2add(make_float2(v[4 * q4 + 2], v[4 * q4 + 3]), make_float2(w[4 * q4 + 2], w[4 * q4 + 3])), r23);
    if (kp.kind == 1) {  // (gamma b + c)^degree
      const float2 b01 = f2fma(rk.g, t01, rk.c), b23 = f2fma(rk.g, t23, rk.c);
      t01 = b01;
      t23 = b23;
      for (int e = 1; e < kp.degree; ++e) {
        t01 = f2mul(t01, b01);
        t23 = f2mul(t23, b23);
      }
    } else if (kp.kind == 2) {  // exp(-gamma max(0, ni + nj - 2 b))
      const float4 nj = reinterpret_cast<const float4 *>(cnj)[q4];
      const float2 nn01 = f2add(rk.c, make_float2(nj.x, nj.y)), nn23 = f2add(rk.c, make_float2(nj.z, nj.w));
      float2 r01 = f2fma(rk.g, t01, nn01), r23 = f2fma(rk.g, t23, nn23);
      r01 = f2mul(make_float2(fmaxf(r01.x, 0.f), fmaxf(r01.y, 0.f)), make_float2(rk.scale, rk.scale));
      r23 = f2mul(make_float2(fmaxf(r23.x, 0.f), fmaxf(r23.y, 0.f)), make_float2(rk.scale, rk.scale));
      t01 = make_float2(ex2_approx(r01.x), ex2_approx(r01.y));
      t23 = make_float2(ex2_approx(r23.x), ex2_approx(r23.y));
    } else {  // linear: b
      t01 = f2mul(t01, rk.g);
      t23 = f2mul(t23, rk.g);
    }
    v[4 * q4] = t01.x;
    v[4 * q4 + 1] = t01.y;
    v[4 * q4 + 2] = t23.x;
    v[4 * q4 + 3] = t23.y;
  }
}

// kappa_chunk for a chunk whose main + correction sum is already in v (same fp32 operations).
__device__ __forceinline__ void kappa_chunk_sum(float (&v)[32], const float *cnj, const float *crs,
                                                const KappaParams &kp, const RowK &rk) {
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    const float4 rj = reinterpret_cast<const float4 *>(crs)[q4];
    float2 t01 = f2mul(make_float2(v[4 * q4], v[4 * q4 + 1]), make_float2(rj.x, rj.y));
    float2 t23 = f2mul(make_float2(v[4 * q4 + 2], v[4 * q4 + 3]), make_float2(rj.z, rj.w));
    if (kp.kind == 1) {
      const float2 b01 = f2fma(rk.g, t01, rk.c), b23 = f2fma(rk.g, t23, rk.c);
      t01 = b01;
      t23 = b23;
      for (int e = 1; e < kp.degree; ++e) {
        t01 = f2mul(t01, b01);
        t23 = f2mul(t23, b23);
      }
    } else if (kp.kind == 2) {
      const float4 nj = reinterpret_cast<const float4 *>(cnj)[q4];
      const float2 nn01 = f2add(rk.c, make_float2(nj.x, nj.y)), nn23 = f2add(rk.c, make_float2(nj.z, nj.w));
      float2 r01 = f2fma(rk.g, t01, nn01), r23 = f2fma(rk.g, t23, nn23);
      r01 = f2mul(make_float2(fmaxf(r01.x, 0.f), fmaxf(r01.y, 0.f)), make_float2(rk.scale, rk.scale));
      r23 = f2mul(make_float2(fmaxf(r23.x, 0.f), fmaxf(r23.y, 0.f)), make_float2(rk.scale, rk.scale));
      t01 = make_float2(ex2_approx(r01.x), ex2_approx(r01.y));
      t23 = make_float2(ex2_approx(r23.x), ex2_approx(r23.y));
    } else {
      t01 = f2mul(t01, rk.g);
      t23 = f2mul(t23, rk.g);
    }
    v[4 * q4] = t01.x;
    v[4 * q4 + 1] = t01.y;
    v[4 * q4 + 2] = t23.x;
    v[4 * q4 + 3] = t23.y;
  }
}

__device__ __forceinline__ void tmem_ld2_32(uint32_t t_main, uint32_t t_corr, float (&v)[32], float (&w)[32]) {
  tmem_ld32_nowait(t_main, v);
  tmem_ld32_nowait(t_corr, w);
  tmem_wait_ld();
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

constexpr size_t T2_GEMM_EXTRA = TC_EPI_WARPS * (TC_STAGING_BYTES + TC_COLC_BYTES);
constexpr size_t T2_GEMM_SMEM = (size_t)T2_STAGES * T2_STAGE_BYTES + T2_GEMM_EXTRA + 1024 + 128;

template <class Sched>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1)
    tc2_gemm_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
                    const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_out2,
                    const CUtensorMap *__restrict__ omaps, uint32_t idesc, int nkb, int64_t n,
                    const float *__restrict__ norms, const float *__restrict__ rscale, KappaParams kp, Sched sc,
                    float oscale, int planes) {
  // oscale == 0: fp32 output; > 0: fp16 output of K' = K * oscale (f4 K storage): planes == 1
  // hi = RN(K') only, planes == 2 also lo = RN(K' - hi) through tm_out2 (hi + lo = K' to 2^-21 + 2^-24 relative)
  extern __shared__ uint8_t smem_raw[];
  uint8_t *extra;
  const T2Smem s = t2_carve(smem_raw, (uint32_t)T2_GEMM_EXTRA, &extra);
  uint8_t *staging = extra;
  float *colc = reinterpret_cast<float *>(extra + TC_EPI_WARPS * TC_STAGING_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  t2_setup(s, warp);
  const uint32_t tmem_base = *s.tmem_slot;

  if (warp == 0) {
    if (lane == 0) t2_producer(sc, s, &tm_hi, &tm_lo, &tm_hi, &tm_lo, nkb, cr, 1);
  } else if (warp == 1) {
    if (lane == 0 && cr == 0) t2_mma(sc, s, nkb, idesc, tmem_base);
  } else {
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int half = e >> 2;
    uint8_t *stg = staging + e * TC_STAGING_BYTES;
    float *cn = colc + e * 256;
    const uint64_t evict = l2_policy_evict_first();
    const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    int64_t it = 0;
    for (int64_t u = cl; u < sc.nitems; u += ncl, ++it) {
      int tm, tn, ridx;
      int64_t i0, m, j0, ncov;
      sc.region(u, tm, tn, i0, m, j0, ncov, ridx);
      const CUtensorMap *out1 = ridx < 0 ? &tm_out : omaps + (int64_t)ridx * planes;
      const CUtensorMap *out2 = ridx < 0 ? &tm_out2 : out1 + 1;
      const int64_t ibase = i0 + (int64_t)tm * T2_BM + (int64_t)cr * 128 + quarter * 32;
      const int64_t i = ibase + lane;
      const bool row_ok = i < i0 + m && i < n;
      const float ni = row_ok ? norms[i] : 0.f;
      const float rsi = (rscale && row_ok) ? rscale[i] : 1.f;
      const RowK rk = make_rowk(kp, rsi, ni);
      const int64_t jw = j0 + (int64_t)tn * 256 + half * 128;
      stage_column_constants(cn, norms, rscale, jw, n, kp.kind == 2, lane);
      mbar_wait(s.tfull, (uint32_t)(it & 1));
      tc_fence_after();
      const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col = half * 128 + c * 32;
        const int64_t jb = jw + c * 32;
        float v[32], w[32];
        tmem_ld2_32(tq + (uint32_t)col, tq + (uint32_t)(256 + col), v, w);
        if (jb >= j0 + ncov || ibase >= i0 + m) continue;
        kappa_chunk(v, w, cn + c * 32, cn + 128 + c * 32, kp, rk);
        if (kp.kind == 2 && i >= jb && i < jb + 32) {  // kappa(x_i, x_i) = 1 exactly (A1)
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (jb + q == i) v[q] = 1.f;
        }
        if (!row_ok || jb + 32 > n) {  // partial chunk / invalid row: padding is 0
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (!row_ok || jb + q >= n) v[q] = 0.f;
        }
        if (oscale > 0.f) {  // 32 x 32 fp16 boxes per chunk and plane (64-byte rows, same swizzle)
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] *= oscale;
          for (int pl = 0; pl < planes; ++pl) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4) {
              uint32_t hw[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int q = 8 * u4 + 2 * e;
                const __half2 h2 = __floats2half2_rn(v[q], v[q + 1]);
                hw[e] = *reinterpret_cast<const uint32_t *>(&h2);
                if (pl == 0 && planes > 1) {  // the residual for the lo plane (exact in fp32)
                  const float2 f = __half22float2(h2);
                  v[q] -= f.x;
                  v[q + 1] -= f.y;
                }
              }
              *reinterpret_cast<uint4 *>(stg + lane * 64 + ((u4 ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(hw[0], hw[1], hw[2], hw[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(pl ? out2 : out1, (int)(jb - j0), (int)(ibase - i0), stg, evict);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
          continue;
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {
            float4 *dst = reinterpret_cast<float4 *>(stg + lane * 64 + ((u4 ^ ((lane >> 1) & 3)) << 4));
            const int q = hh * 16 + 4 * u4;
            *dst = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && jb + hh * 16 < j0 + ncov) {
            tma_store_2d(out1, (int)(jb + hh * 16 - j0), (int)(ibase - i0), stg, evict);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(s.tempty, 0);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  t2_teardown(s, warp, tmem_base);
}

// ---------------------------------------------------------------- fused streaming kernel
struct T2StreamSched {
  int64_t nitems;
  int tiles_m, tiles_n, nsplit, tps;
  int64_t row0;
  int split_major;  // 1: consecutive work items share a split (column region) -> L2 reuse
  int hint;         // 1: L2 evict_last on the operand loads
  __device__ __forceinline__ void unit(int64_t u, int &tm, int &sp) const {
    if (split_major) {
      sp = (int)(u / tiles_m);
      tm = (int)(u % tiles_m);
    } else {
      tm = (int)(u / nsplit);
      sp = (int)(u % nsplit);
    }
  }
  __device__ __forceinline__ void item(int64_t u, int &ra, int &rb0, int &ntn) const {
    int tm, sp;
    unit(u, tm, sp);
    const int tn0 = sp * tps, tn1 = min(tiles_n, tn0 + tps);
    ra = (int)(row0 + (int64_t)tm * T2_BM);
    rb0 = tn0 * 256;
    ntn = tn1 > tn0 ? tn1 - tn0 : 0;
  }
};

constexpr size_t T2_STREAM_EXTRA = TC_EPI_WARPS * TC_COLC_BYTES + 512;  // + seg[k+1] (k <= 64), keeps the barriers 8-aligned
constexpr size_t T2_STREAM_SMEM = (size_t)T2_STAGES * T2_STAGE_BYTES + T2_STREAM_EXTRA + 1024 + 128;

template <int KMAX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1)
    tc2_stream_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                      const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                      uint32_t idesc, int nkb, int64_t n, int64_t b0, int64_t nloc, int64_t rows_pad,
                      const float *__restrict__ norms, const float *__restrict__ rscale,
                      const float *__restrict__ snorms, const float *__restrict__ srscale,
                      const int32_t *__restrict__ pos, int64_t npos, const int32_t *__restrict__ seg_g, int k,
                      KappaParams kp, T2StreamSched sc, double *__restrict__ Spart, int kstride, int c0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *extra;
  const T2Smem s = t2_carve(smem_raw, (uint32_t)T2_STREAM_EXTRA, &extra);
  float *colc = reinterpret_cast<float *>(extra);
  int32_t *seg = reinterpret_cast<int32_t *>(extra + TC_EPI_WARPS * TC_COLC_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const bool fp16 = rscale != nullptr;
  // B holds the clusters [c0, c0 + k) of the sorted operand, starting at sorted row seg_g[0]
  const int32_t sbase = seg_g[0];
  for (int c = threadIdx.x; c <= k; c += blockDim.x) seg[c] = seg_g[c] - sbase;
  t2_setup(s, warp);  // (its cluster barrier also publishes seg)
  const uint32_t tmem_base = *s.tmem_slot;

  if (warp == 0) {
    if (lane == 0) t2_producer(sc, s, &ta_hi, &ta_lo, &tb_hi, &tb_lo, nkb, cr, sc.hint);
  } else if (warp == 1) {
    if (lane == 0 && cr == 0) t2_mma(sc, s, nkb, idesc, tmem_base);
  } else {
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int half = e >> 2;
    float *cn = colc + e * 256;
    const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    int64_t it = 0;
    for (int64_t u = cl; u < sc.nitems; u += ncl) {
      int tm, sp;
      sc.unit(u, tm, sp);
      const int tn0 = sp * sc.tps, tn1 = min(sc.tiles_n, tn0 + sc.tps);
      const int64_t r = (int64_t)tm * T2_BM + (int64_t)cr * 128 + quarter * 32 + lane;  // A-set row
      const bool row_ok = r < nloc;
      const int64_t i = sc.row0 + r;
      const float ni = row_ok ? norms[i] : 0.f;
      const float rsi = (fp16 && row_ok) ? rscale[i] : 1.f;
      const RowK rk = make_rowk(kp, rsi, ni);
      const int64_t mypos = (row_ok && kp.kind == 2 && pos && i >= b0 && i < b0 + npos) ? pos[i - b0] - sbase : -1;
      double acc[KMAX];
#pragma unroll
      for (int c = 0; c < KMAX; ++c) acc[c] = 0.0;
      for (int tn = tn0; tn < tn1; ++tn, ++it) {
        const int64_t pbase = (int64_t)tn * 256 + half * 128;
        stage_column_constants(cn, snorms, fp16 ? srscale : nullptr, pbase, n, kp.kind == 2, lane);
        mbar_wait(s.tfull, (uint32_t)(it & 1));
        tc_fence_after();
        const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = half * 128 + c * 32;
          float v[32], w[32];
          tmem_ld2_32(tq + (uint32_t)col, tq + (uint32_t)(256 + col), v, w);
          if (c == 3) {  // all of the tile is in registers: TMEM back to the MMA warp now
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(s.tempty, 0);
          }
          const int64_t p0 = pbase + c * 32;
          if (p0 >= n) continue;
          kappa_chunk(v, w, cn + c * 32, cn + 128 + c * 32, kp, rk);
          if (mypos >= p0 && mypos < p0 + 32) {  // kappa(x_i, x_i) = 1 exactly (A1)
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (p0 + q == mypos) v[q] = 1.f;
          }
          if (p0 + 32 > n) {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (p0 + q >= n) v[q] = 0.f;
          }
          const int64_t p1 = p0 + 31 < n ? p0 + 31 : n - 1;
          int c0 = 0, c1 = 0;
          for (int cc = 1; cc < k; ++cc) {
            if (seg[cc] <= p0) c0 = cc;
            if (seg[cc] <= p1) c1 = cc;
          }
          if (c0 == c1) {
            float2 s2 = make_float2(v[0], v[1]);
#pragma unroll
            for (int q = 2; q < 32; q += 2) s2 = f2add(s2, make_float2(v[q], v[q + 1]));
            acc_add<KMAX>(acc, c0, (double)(s2.x + s2.y));
          } else {
            for (int cc = c0; cc <= c1; ++cc) {
              const int64_t lo = seg[cc] - p0, hi = seg[cc + 1] - p0;
              float sum = 0.f;
#pragma unroll
              for (int q = 0; q < 32; ++q) sum += (q >= lo && q < hi) ? v[q] : 0.f;
              acc_add<KMAX>(acc, cc, (double)sum);
            }
          }
        }
      }
      if (row_ok && tn1 > tn0) {
        double *dst = Spart + ((int64_t)(2 * sp + half) * rows_pad + r) * kstride + c0;
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
          if (c < k) dst[c] = acc[c];
      } else if (row_ok) {
        double *dst = Spart + ((int64_t)(2 * sp + half) * rows_pad + r) * kstride + c0;
        for (int c = 0; c < k; ++c) dst[c] = 0.0;
      }
    }
  }
  t2_teardown(s, warp, tmem_base);
}

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

template <int KMAX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1)
    tc2_stream_sym_kernel(const __grid_constant__ CUtensorMap t_hi, const __grid_constant__ CUtensorMap t_lo,
                          uint32_t idesc, int nkb, int64_t n, const float *__restrict__ snorms,
                          const float *__restrict__ srscale, const int32_t *__restrict__ seg_g, int k,
                          KappaParams kp, T2SymSched sc, double fx_scale, long long *__restrict__ Sfix) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *extra;
  const T2Smem s = t2_carve(smem_raw, (uint32_t)T2_STREAM_EXTRA, &extra);
  float *colc = reinterpret_cast<float *>(extra);
  int32_t *seg = reinterpret_cast<int32_t *>(extra + TC_EPI_WARPS * TC_COLC_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const bool fp16 = srscale != nullptr;
  for (int c = threadIdx.x; c <= k; c += blockDim.x) seg[c] = seg_g[c];
  t2_setup(s, warp);
  const uint32_t tmem_base = *s.tmem_slot;

  if (warp == 0) {
    if (lane == 0) t2_producer(sc, s, &t_hi, &t_lo, &t_hi, &t_lo, nkb, cr, 1);
  } else if (warp == 1) {
    if (lane == 0 && cr == 0) t2_mma(sc, s, nkb, idesc, tmem_base);
  } else {
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int half = e >> 2;
    float *cn = colc + e * 256;
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
      // labels of the warp's 32 rows (sorted: a contiguous run of segments r0 .. r1)
      const int64_t plast = rw + 31 < n ? rw + 31 : n - 1;
      int r0 = 0, r1 = 0;
      for (int cc = 1; cc < k; ++cc) {
        if (seg[cc] <= rw) r0 = cc;
        if (seg[cc] <= plast) r1 = cc;
      }
      int mylab = r0;
      for (int cc = r0 + 1; cc <= r1; ++cc)
        if (seg[cc] <= p) mylab = cc;
      double acc[KMAX];
#pragma unroll
      for (int c = 0; c < KMAX; ++c) acc[c] = 0.0;
      for (int tn = tn0; tn < tn1; ++tn, ++it) {
        const int64_t pbase = (int64_t)tn * 256 + half * 128;
        const bool diag = tn == tm;
        stage_column_constants(cn, snorms, fp16 ? srscale : nullptr, pbase, n, kp.kind == 2, lane);
        mbar_wait(s.tfull, (uint32_t)(it & 1));
        tc_fence_after();
        const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16);
        // chunk by chunk (main + correction summed in registers); TMEM goes back to the MMA
        // warp as soon as the last chunk is in registers, before its kappa / sums (single-
        // buffered TMEM: this shortens the serial drain; a one-chunk-ahead prefetch measured
        // slower, its third buffer spills)
        float m[32], r[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int colc = half * 128 + c * 32;
          tmem_ld32_nowait(tq + (uint32_t)colc, m);
          tmem_ld32_nowait(tq + (uint32_t)(256 + colc), r);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            const float2 t = f2add(make_float2(m[q], m[q + 1]), make_float2(r[q], r[q + 1]));
            m[q] = t.x;
            m[q + 1] = t.y;
          }
          if (c == 3) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(s.tempty, 0);
          }
          float(&v)[32] = m;
          const int64_t p0 = pbase + c * 32;
          if (p0 >= n || rw >= n) continue;
          kappa_chunk_sum(v, cn + c * 32, cn + 128 + c * 32, kp, rk);
          if (diag && kp.kind == 2 && p >= p0 && p < p0 + 32) {  // kappa(x_p, x_p) = 1 exactly (A1)
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (p0 + q == p) v[q] = 1.f;
          }
          if (p0 + 32 > n) {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (p0 + q >= n) v[q] = 0.f;
          }
          if (!row_ok) {
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = 0.f;
          }
          // row part: the chunk's columns by their segments
          const int64_t p1 = p0 + 31 < n ? p0 + 31 : n - 1;
          int c0 = 0, c1 = 0;
          for (int cc = 1; cc < k; ++cc) {
            if (seg[cc] <= p0) c0 = cc;
            if (seg[cc] <= p1) c1 = cc;
          }
          if (c0 == c1) {
            float2 s2 = make_float2(v[0], v[1]);
#pragma unroll
            for (int q = 2; q < 32; q += 2) s2 = f2add(s2, make_float2(v[q], v[q + 1]));
            acc_add<KMAX>(acc, c0, (double)(s2.x + s2.y));
          } else {
            for (int cc = c0; cc <= c1; ++cc) {
              const int64_t lo = seg[cc] - p0, hi = seg[cc + 1] - p0;
              float sum = 0.f;
#pragma unroll
              for (int q = 0; q < 32; ++q) sum += (q >= lo && q < hi) ? v[q] : 0.f;
              acc_add<KMAX>(acc, cc, (double)sum);
            }
          }
          if (diag) continue;
          // column part: column p0 + lane gets the sum over the warp's rows of each label
          if (r0 == r1) {  // one label (almost always): the butterfly may consume v
            const float cs = lane_column_sum(v, lane);
            if (p0 + lane < n) red_add_s64(Sfix + (p0 + lane) * k + r0, __double2ll_rn((double)cs * fx_scale));
          } else {  // the warp straddles a segment boundary: one masked pass per label
            for (int cc = r0; cc <= r1; ++cc) {
              float t[32];
              const bool mine = mylab == cc;
#pragma unroll
              for (int q = 0; q < 32; ++q) t[q] = mine ? v[q] : 0.f;
              const float cs = lane_column_sum(t, lane);
              if (p0 + lane < n)
                red_add_s64(Sfix + (p0 + lane) * k + cc, __double2ll_rn((double)cs * fx_scale));
            }
          }
        }
      }
      if (row_ok) {
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
          if (c < k) red_add_s64(Sfix + p * k + c, __double2ll_rn(acc[c] * fx_scale));
      }
    }
  }
  t2_teardown(s, warp, tmem_base);
}

// ---------------------------------------------------------------- host launchers
// Materialised: same contract as tc_gemm_launch (gemm_tc.cuh), on CTA pairs.
inline int tc2_gemm_launch(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16,
                           const float *rscale, int64_t rows, int64_t dp, int64_t n, int64_t i0, int64_t m,
                           int64_t j0, int64_t ncov, const float *norms, const KappaParams &kp, void *out,
                           int64_t ldo, cudaStream_t st, int64_t *launches, float oscale = 0.f,
                           void *out_lo = nullptr) {
  // oscale > 0: out is fp16 and receives hi = RN(K * oscale); with out_lo also lo = RN(K * oscale - hi)
  if (g.hi != Xhi || g.lo != Xlo || g.fp16 != fp16)
    if (tc_make_maps(g, Xhi, Xlo, fp16, rows, dp)) return 1;
  if ((ldo & (oscale > 0.f ? 7 : 3)) || (reinterpret_cast<uintptr_t>(out) & 15)) {
    tc_err_slot() = "tcgen05 GEMM output needs 16-byte alignment and 16-byte aligned rows";
    return 1;
  }
  if (out_lo) {
    if (tc_make_out_map(g, out_lo, m, ncov, ldo, true)) return 1;
    g.map_out2 = g.map_out;
  }
  if (tc_make_out_map(g, out, m, ncov, ldo, oscale > 0.f)) return 1;
  if (!out_lo) g.map_out2 = g.map_out;
  if (ensure_smem_attr((const void *)tc2_gemm_kernel<T2GemmSched>, T2_GEMM_SMEM) != cudaSuccess) {
    tc_err_slot() = "cudaFuncSetAttribute(tc2_gemm_kernel) failed";
    return 1;
  }
  if (!g.num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  T2GemmSched sc;
  sc.tiles_m = (int)((m + T2_BM - 1) / T2_BM);
  sc.tiles_n = (int)((ncov + 255) / 256);
  sc.nitems = (int64_t)sc.tiles_m * sc.tiles_n;
  sc.i0 = i0;
  sc.j0 = j0;
  sc.m = m;
  sc.ncov = ncov;
  const int64_t clusters = sc.nitems < g.num_sms / 2 ? sc.nitems : g.num_sms / 2;
  tc2_gemm_kernel<T2GemmSched><<<(unsigned)(2 * clusters), T2_THREADS, T2_GEMM_SMEM, st>>>(
      g.map_hi, g.map_lo, g.map_out, g.map_out2, nullptr, t2_idesc(fp16), (int)(dp / TC_BK), n, norms,
      fp16 ? rscale : nullptr, kp, sc, oscale, out_lo ? 2 : 1);
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// Several output regions (the f1 band pieces) in ONE launch: the per-band launches left each
// piece's last wave of CTA pairs partly idle. regs_dev: nreg regions (device), omaps: nreg * planes
// output maps (device, 64-B aligned; fp32 maps when oscale == 0). nitems = total pair tiles.
inline int tc2_gemm_launch_multi(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16,
                                 const float *rscale, int64_t rows, int64_t dp, int64_t n, const T2Region *regs_dev,
                                 int nreg, int64_t nitems, const CUtensorMap *omaps, const float *norms,
                                 const KappaParams &kp, float oscale, int planes, cudaStream_t st, int64_t *launches) {
  if (nitems <= 0) return 0;
  if (g.hi != Xhi || g.lo != Xlo || g.fp16 != fp16)
    if (tc_make_maps(g, Xhi, Xlo, fp16, rows, dp)) return 1;
  if (ensure_smem_attr((const void *)tc2_gemm_kernel<T2MultiSched>, T2_GEMM_SMEM) != cudaSuccess) {
    tc_err_slot() = "cudaFuncSetAttribute(tc2_gemm_kernel multi) failed";
    return 1;
  }
  if (!g.num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  T2MultiSched sc;
  sc.nitems = nitems;
  sc.nreg = nreg;
  sc.reg = regs_dev;
  const int64_t clusters = nitems < g.num_sms / 2 ? nitems : g.num_sms / 2;
  tc2_gemm_kernel<T2MultiSched><<<(unsigned)(2 * clusters), T2_THREADS, T2_GEMM_SMEM, st>>>(
      g.map_hi, g.map_lo, g.map_hi, g.map_hi, omaps, t2_idesc(fp16), (int)(dp / TC_BK), n, norms,
      fp16 ? rscale : nullptr, kp, sc, oscale, planes);
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

template <int KMAX>
inline int t2s_launch_k(unsigned grid, cudaStream_t st, const TcStream &g, uint32_t idesc, int nkb,
                        int64_t n, int64_t b0, int64_t nloc, int64_t rows_pad, const float *norms,
                        const float *rscale, const float *snorms, const float *srscale, const int32_t *pos,
                        int64_t npos, const int32_t *seg, int k, const KappaParams &kp, const T2StreamSched &sc,
                        double *Spart, int kstride, int c0) {
  if (ensure_smem_attr((const void *)tc2_stream_kernel<KMAX>, T2_STREAM_SMEM) != cudaSuccess) {
    tc_err_slot() = "cudaFuncSetAttribute(tc2_stream_kernel) failed";
    return 1;
  }
  tc2_stream_kernel<KMAX><<<grid, T2_THREADS, T2_STREAM_SMEM, st>>>(g.a_hi, g.a_lo, g.b_hi, g.b_lo, idesc, nkb, n,
                                                                    b0, nloc, rows_pad, norms, rscale, snorms,
                                                                    srscale, pos, npos, seg, k, kp, sc, Spart,
                                                                    kstride, c0);
  return 0;
}

// Streaming on CTA pairs. A: rows_a rows (Xhi/Xlo, norms, rscale), output rows [row0, row0 + nloc).
// B: the label-sorted operand (Shi/Slo, snorms, srscale; rows_b rows from its base) holding the
// clusters [c0, c0 + k) in n rows; seg = the cluster starts of those clusters (seg[0] = the
// sorted row of B's base). pos (may be NULL): sorted position of A row i for b0 <= i < b0 + npos
// (the Gaussian diagonal). Spart: [2 * nsplit][rows_pad][kstride], columns c0 .. c0 + k - 1.
inline int tc2_stream_launch(TcStream &g, const uint16_t *Xhi, const uint16_t *Xlo, const uint16_t *Shi,
                             const uint16_t *Slo, bool fp16, int64_t rows_a, int64_t rows_b, int64_t dp, int64_t n,
                             int64_t b0, int64_t row0, int64_t nloc, int64_t rows_pad, const float *norms,
                             const float *rscale, const float *snorms, const float *srscale, const int32_t *pos,
                             int64_t npos, const int32_t *seg, int k, const KappaParams &kp, int nsplit,
                             double *Spart, int kstride, int c0, cudaStream_t st, int64_t *launches) {
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
  if (nloc <= 0) return 0;
  T2StreamSched sc;
  sc.tiles_m = (int)((nloc + T2_BM - 1) / T2_BM);
  sc.tiles_n = (int)((n + 255) / 256);
  sc.nsplit = nsplit;
  sc.tps = (sc.tiles_n + nsplit - 1) / nsplit;
  sc.nitems = (int64_t)sc.tiles_m * nsplit;
  sc.row0 = row0;
  sc.hint = 1;         // L2 evict_last on the operand loads
  sc.split_major = 0;  // tile-major: measured faster at n = 1M, equal at 200k
  const int64_t clusters = sc.nitems < g.num_sms / 2 ? sc.nitems : g.num_sms / 2;
  const unsigned grid = (unsigned)(2 * clusters);
  const uint32_t idesc = t2_idesc(fp16);
  const int nkb = (int)(dp / TC_BK);
  const float *rs = fp16 ? rscale : nullptr;
  int rc;
  if (k > 16) {
    tc_err_slot() = "tc2_stream_launch: at most 16 clusters per launch";
    return 1;
  }
  if (k <= 4)
    rc = t2s_launch_k<4>(grid, st, g, idesc, nkb, n, b0, nloc, rows_pad, norms, rs, snorms, srscale, pos, npos,
                         seg, k, kp, sc, Spart, kstride, c0);
  else if (k <= 8)
    rc = t2s_launch_k<8>(grid, st, g, idesc, nkb, n, b0, nloc, rows_pad, norms, rs, snorms, srscale, pos, npos,
                         seg, k, kp, sc, Spart, kstride, c0);
  else
    rc = t2s_launch_k<16>(grid, st, g, idesc, nkb, n, b0, nloc, rows_pad, norms, rs, snorms, srscale, pos,
                          npos, seg, k, kp, sc, Spart, kstride, c0);
  if (rc) return rc;
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// f1 streaming launcher: A = B = the sorted operand (Shi/Slo, rows rows). units: device array
// of nunits int4 (tm, tn0, ntn, 0). Sfix (n x k int64) must be zeroed by the caller.
template <int KMAX>
inline int t2sym_launch_k(unsigned grid, cudaStream_t st, const TcStream &g, uint32_t idesc, int nkb,
                          int64_t n, const float *snorms, const float *rs, const int32_t *seg, int k,
                          const KappaParams &kp, const T2SymSched &sc, double fx_scale, long long *Sfix) {
  if (ensure_smem_attr((const void *)tc2_stream_sym_kernel<KMAX>, T2_STREAM_SMEM) != cudaSuccess) {
    tc_err_slot() = "cudaFuncSetAttribute(tc2_stream_sym_kernel) failed";
    return 1;
  }
  tc2_stream_sym_kernel<KMAX><<<grid, T2_THREADS, T2_STREAM_SMEM, st>>>(g.a_hi, g.a_lo, idesc, nkb, n, snorms, rs,
                                                                        seg, k, kp, sc, fx_scale, Sfix);
  return 0;
}

inline int tc2_stream_sym_launch(TcStream &g, const uint16_t *Shi, const uint16_t *Slo, bool fp16, int64_t rows,
                                 int64_t dp, int64_t n, const float *snorms, const float *srscale,
                                 const int32_t *seg, int k, const KappaParams &kp, const int4 *units,
                                 int64_t nunits, double fx_scale, long long *Sfix, cudaStream_t st,
                                 int64_t *launches) {
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
  if (k > 16) {
    tc_err_slot() = "tc2_stream_sym_launch: k <= 16";
    return 1;
  }
  T2SymSched sc;
  sc.units = units;
  sc.nitems = nunits;
  const int64_t clusters = nunits < g.num_sms / 2 ? nunits : g.num_sms / 2;
  const unsigned grid = (unsigned)(2 * clusters);
  const uint32_t idesc = t2_idesc(fp16);
  const int nkb = (int)(dp / TC_BK);
  const float *rs = fp16 ? srscale : nullptr;
  int rc;
  if (k <= 4) rc = t2sym_launch_k<4>(grid, st, g, idesc, nkb, n, snorms, rs, seg, k, kp, sc, fx_scale, Sfix);
  else if (k <= 8) rc = t2sym_launch_k<8>(grid, st, g, idesc, nkb, n, snorms, rs, seg, k, kp, sc, fx_scale, Sfix);
  else if (k <= 12)
    rc = t2sym_launch_k<12>(grid, st, g, idesc, nkb, n, snorms, rs, seg, k, kp, sc, fx_scale, Sfix);
  else rc = t2sym_launch_k<16>(grid, st, g, idesc, nkb, n, snorms, rs, seg, k, kp, sc, fx_scale, Sfix);
  if (rc) return rc;
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tc_err_slot() = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}


}  // namespace kkm
