// chain.cuh -- the chained fp16x3 mainloop shared by every tensor-core kernel of the a1 step
// (ssym.cuh: streaming f1; tc3.cuh: materialised GEMM, self dots, full streaming).
//
// CTA pairs (cta_group::2, M = 256 x N = 256 tiles; the tc2.cuh producer and UMMA helpers), TMEM
// holding TWO fp32 accumulators (columns [0, 256) and [256, 512)), and every tile computed as
// chains: the tile's nkb K-blocks of 64 are cut into nch = ceil(nkb / CH_CKB) balanced chains (chain
// ci covers K-blocks [ci nkb / nch, (ci + 1) nkb / nch)); the launch's chain c goes to buffer c & 1
// with all three fp16x3 MMAs of a k-step (hi*lo, lo*hi, hi*hi) into the one accumulator, and the epilogue drains each chain into fp32 registers (RN
// adds) while the tensor core fills the other buffer. Two effects (DESIGN A9, §5.1):
//   precision: the tensor core truncates every accumulation relative to the running fp32 sum; a
//     chain restarts that sum from zero, so the one-signed error of b = x.y is bounded by the
//     chain length (~6 CH_CKB truncation units of |b|) instead of growing with d/16
//     (tools/bias_model.py); and every kernel -- including the self dots that serve as the
//     Gaussian norms -- accumulates with the same chain boundaries, so like terms cancel;
//   speed: TMEM is double-buffered, no drain is serial with the MMAs.
// Epilogue layout: 16 warps = 4 TMEM lane quarters x 4 column quarters of 64; thread = row.
#pragma once
#include <type_traits>

#include "tc2.cuh"

namespace kkm {

constexpr int CH_EPI_WARPS = 16;
constexpr int CH_THREADS = (2 + CH_EPI_WARPS) * 32;
constexpr int CH_COLS = 64;  // columns per epilogue warp
constexpr int CH_CKB = 4;    // K-blocks of 64 per accumulation chain (at most): nch = ceil(nkb / CH_CKB)

inline int ch_chains(int nkb, int ckb_max) { return (nkb + ckb_max - 1) / ckb_max; }
constexpr size_t CH_COLC_BYTES = 2 * CH_COLS * 4;  // per warp: norms + rscale of its 64 columns

// Per-column constants of columns [j, j + 64) into cn[0..64) (norms) / cn[64..128) (rscale).
__device__ __forceinline__ void ch_stage_columns(float *cn, const float *__restrict__ norms,
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
  reinterpret_cast<float2 *>(cn + CH_COLS)[lane] = rv;
  __syncwarp();
}

// fp32 -> int64 fixed point: v * 2^s is exact in fp32 (a power-of-two scale), then one rounding to
// an integer at resolution 2^-s (n max K 2^s < 2^61) -- no fp64 arithmetic in the epilogue.
__device__ __forceinline__ long long ch_fix(float v, float fx) { return __float2ll_rn(v * fx); }

// Arrival on the leader CTA's TMEM-empty barrier without release semantics: the TMEM reads are
// complete (tcgen05.wait::ld) and ordered by tcgen05.fence::before_thread_sync; a release arrive
// would also wait for this warp's outstanding red.global of the previous tile (ERRBAR).
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

// kappa_chunk_sum (tc2.cuh) specialised on the kernel kind at compile time (fewer live registers).
template <int KIND>
__device__ __forceinline__ void ch_kappa(float (&v)[32], const float *cnj, const float *crs, const KappaParams &kp,
                                         const RowK &rk) {
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    const float4 rj = reinterpret_cast<const float4 *>(crs)[q4];
    float2 t01 = f2mul(make_float2(v[4 * q4], v[4 * q4 + 1]), make_float2(rj.x, rj.y));
    float2 t23 = f2mul(make_float2(v[4 * q4 + 2], v[4 * q4 + 3]), make_float2(rj.z, rj.w));
    if (KIND == 3) {  // (gamma b + c)^2 (the paper's benchmark kernel)
      const float2 b01 = f2fma(rk.g, t01, rk.c), b23 = f2fma(rk.g, t23, rk.c);
      t01 = f2mul(b01, b01);
      t23 = f2mul(b23, b23);
    } else if (KIND == 1) {  // (gamma b + c)^degree
      const float2 b01 = f2fma(rk.g, t01, rk.c), b23 = f2fma(rk.g, t23, rk.c);
      t01 = b01;
      t23 = b23;
      for (int e = 1; e < kp.degree; ++e) {
        t01 = f2mul(t01, b01);
        t23 = f2mul(t23, b23);
      }
    } else if (KIND == 2) {  // exp(-gamma max(0, (ni - b) + (nj - b)))
      // r^2 = (n_i - b) + (n_j - b): for near points (b ~ n_i ~ n_j, the pairs that decide E) both
      // differences are exact in fp32 (Sterbenz) and r^2 keeps its relative accuracy, where
      // n_i + n_j - 2b loses ~ulp(n_i + n_j) to the cancellation (A1, A23)
      const float4 nj = reinterpret_cast<const float4 *>(cnj)[q4];
      const float2 a01 = f2fma(rk.g, t01, rk.c), a23 = f2fma(rk.g, t23, rk.c);  // n_i - b
      const float2 c01 = f2fma(rk.g, t01, make_float2(nj.x, nj.y)), c23 = f2fma(rk.g, t23, make_float2(nj.z, nj.w));
      float2 r01 = f2add(a01, c01), r23 = f2add(a23, c23);
      r01 = f2mul(make_float2(fmaxf(r01.x, 0.f), fmaxf(r01.y, 0.f)), make_float2(rk.scale, rk.scale));
      r23 = f2mul(make_float2(fmaxf(r23.x, 0.f), fmaxf(r23.y, 0.f)), make_float2(rk.scale, rk.scale));
      t01 = make_float2(ex2_approx(r01.x), ex2_approx(r01.y));
      t23 = make_float2(ex2_approx(r23.x), ex2_approx(r23.y));
    } else {  // linear
      t01 = f2mul(t01, rk.g);
      t23 = f2mul(t23, rk.g);
    }
    v[4 * q4] = t01.x;
    v[4 * q4 + 1] = t01.y;
    v[4 * q4 + 2] = t23.x;
    v[4 * q4 + 3] = t23.y;
  }
}

// ---------------------------------------------------------------- chained accumulation
struct ChSmem {
  uint8_t *stages;
  uint64_t *full, *empty, *cfull, *cempty;
  uint32_t *tmem_slot;
};

__device__ __forceinline__ ChSmem ch_carve(uint8_t *smem_raw, uint32_t extra, uint8_t **extra_ptr) {
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  ChSmem s;
  s.stages = smem_raw + pad;
  *extra_ptr = s.stages + T2_STAGES * T2_STAGE_BYTES;
  s.full = reinterpret_cast<uint64_t *>(*extra_ptr + extra);
  s.empty = s.full + T2_STAGES;
  s.cfull = s.empty + T2_STAGES;
  s.cempty = s.cfull + 2;
  s.tmem_slot = reinterpret_cast<uint32_t *>(s.cempty + 2);
  return s;
}

__device__ __forceinline__ void ch_setup(const ChSmem &s, int warp, uint32_t cempty_count) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < T2_STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s.cfull[b], 1);
      mbar_init(&s.cempty[b], cempty_count);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s.tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
}

// MMA issuer body of one work item u (warp 1 lane 0 of the leader CTA): every tile as nch chains.
template <class Sched>
__device__ __forceinline__ void ch_mma_item(const Sched &sc, const ChSmem &s, int64_t u, int nkb, int nch,
                                            uint32_t idesc, uint32_t tmem_base, int &stage, uint32_t &phase,
                                            int64_t &chain) {
  int ra, rb0, ntn;
  sc.item(u, ra, rb0, ntn);
  for (int t = 0; t < ntn; ++t) {
    uint32_t d = tmem_base;
    int ci = 0, lo = 0, hi = nkb / nch;  // chain ci covers K-blocks [lo, hi) = [ci nkb / nch, (ci+1) nkb / nch)
    for (int kb = 0; kb < nkb; ++kb) {
      const bool first = kb == lo;
      if (first) {
        const int b = (int)(chain & 1);
        mbar_wait(&s.cempty[b], ((uint32_t)(chain >> 1) & 1u) ^ 1u);
        tc_fence_after();
        d = tmem_base + (uint32_t)b * 256u;
      }
      mbar_wait(&s.full[stage], phase);
      tc_fence_after();
      const uint32_t st = smem_u32(s.stages + stage * T2_STAGE_BYTES);
      const uint32_t a_hi = st, a_lo = st + T2_HALF_BYTES;
      const uint32_t b_hi = st + 2 * T2_HALF_BYTES, b_lo = st + 3 * T2_HALF_BYTES;
#pragma unroll
      for (int k = 0; k < TC_BK / 16; ++k) {
        const uint32_t ko = (uint32_t)k * 32u;
        umma2_f16(d, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_lo + ko), idesc, (first && k == 0) ? 0u : 1u);
        umma2_f16(d, umma_desc_sw128(a_lo + ko), umma_desc_sw128(b_hi + ko), idesc, 1u);
        umma2_f16(d, umma_desc_sw128(a_hi + ko), umma_desc_sw128(b_hi + ko), idesc, 1u);
      }
      umma2_commit_both(&s.empty[stage]);
      if (++stage == T2_STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if (kb == hi - 1) {
        ++ci;
        lo = hi;
        hi = (int)((int64_t)(ci + 1) * nkb / nch);
        umma2_commit_both(&s.cfull[chain & 1]);
        ++chain;
      }
    }
  }
}

// MMA issuer, static schedule (pair cl takes items cl, cl + ncl, ...).
template <class Sched>
__device__ __forceinline__ void ch_mma(const Sched &sc, const ChSmem &s, int nkb, int nch, uint32_t idesc,
                                       uint32_t tmem_base) {
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  int stage = 0;
  uint32_t phase = 0;
  int64_t chain = 0;
  for (int64_t u = cl; u < sc.nitems; u += ncl) ch_mma_item(sc, s, u, nkb, nch, idesc, tmem_base, stage, phase, chain);
}

__device__ __forceinline__ void ch_wait(const ChSmem &s, int64_t chain) {
  mbar_wait_backoff(&s.cfull[chain & 1], (uint32_t)(chain >> 1) & 1u);
  tc_fence_after();
}
__device__ __forceinline__ void ch_release(const ChSmem &s, int64_t chain, int lane) {
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive_cluster_relaxed(&s.cempty[chain & 1], 0);
}
// v += the 32 TMEM columns at taddr (fp32 RN), in two 16-column loads (fewer live registers)
__device__ __forceinline__ void ch_ld_add(uint32_t taddr, float (&v)[32]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float w[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=f"(w[0]), "=f"(w[1]), "=f"(w[2]), "=f"(w[3]), "=f"(w[4]), "=f"(w[5]), "=f"(w[6]), "=f"(w[7]),
          "=f"(w[8]), "=f"(w[9]), "=f"(w[10]), "=f"(w[11]), "=f"(w[12]), "=f"(w[13]), "=f"(w[14]), "=f"(w[15])
        : "r"(taddr + (uint32_t)(16 * h)));
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 16; q += 2) {
      const float2 t = f2add(make_float2(v[16 * h + q], v[16 * h + q + 1]), make_float2(w[q], w[q + 1]));
      v[16 * h + q] = t.x;
      v[16 * h + q + 1] = t.y;
    }
  }
}

// Epilogue side: drains the nch chains of one tile into va / vb (this warp's 64
// columns, fp32 RN sums); `chain` counts the launch's chains (the buffer / phase of each).
__device__ __forceinline__ void ch_drain(const ChSmem &s, uint32_t tq, int nch, int64_t &chain,
                                                float (&va)[32], float (&vb)[32], int lane) {
  ch_wait(s, chain);
  {
    const uint32_t ta = tq + (uint32_t)(chain & 1) * 256u;
    tmem_ld32_nowait(ta, va);
    tmem_ld32_nowait(ta + 32u, vb);
    tmem_wait_ld();
  }
  ch_release(s, chain, lane);
  ++chain;
#pragma unroll 1
  for (int ch = 1; ch < nch; ++ch, ++chain) {
    ch_wait(s, chain);
    const uint32_t ta = tq + (uint32_t)(chain & 1) * 256u;
    ch_ld_add(ta, va);
    ch_ld_add(ta + 32u, vb);
    ch_release(s, chain, lane);
  }
}


// ---------------------------------------------------------------- dynamic unit schedule
// The CTA pairs of a persistent chained kernel take work units from ONE global counter instead of
// a static round robin (pair p: units p, p + 74, ...), so the units in flight stay consecutive in
// the host's unit order however the pairs' speeds drift over a long launch.
constexpr int CH_RING = 8;  // unit-index slots in flight per pair
constexpr size_t CH_RING_BYTES = 2 * CH_RING * 8 + CH_RING * 4;
// arrivals that free a ring slot (on the leader CTA): per CTA its 16 epilogue warps + the MMA
// issuer (leader) / the producer (peer CTA)
constexpr uint32_t CH_RING_CONSUMERS = 2 * (CH_EPI_WARPS + 1);


__device__ __forceinline__ void st_cluster_s32(int32_t *p, uint32_t cta, int32_t v) {
  asm volatile("{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\tst.shared::cluster.s32 [ra], %2;\n\t}" ::"r"(
                   smem_u32(p)),
               "r"(cta), "r"(v)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_release(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t *bar, uint32_t parity) {
  uint32_t ns = 32;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
  }
}

// The pair's unit source. Static: pair cl takes units cl, cl + ncl, ... Dynamic: position i of the
// ring (slot i % CH_RING) carries the i-th unit the pair fetched from the global counter work[0]
// (-1: none left); the leader producer fetches (one ahead) and publishes, the other roles read.
// work[1] counts the pairs that saw the end; the last one resets both counters for the next launch.
struct ChRing {
  int32_t *slot;
  uint64_t *full, *empty;  // full: 1 arrival (the leader producer), in both CTAs; empty: leader CTA only
  bool dyn;
  int64_t nitems;
  int32_t *work;
  __device__ __forceinline__ int64_t static_unit(int64_t i) const {
    const int64_t u = (int64_t)(blockIdx.x >> 1) + i * (int64_t)(gridDim.x >> 1);
    return u < nitems ? u : -1;
  }
  // leader producer: publish the pair's next unit (nxt: the prefetched counter value)
  __device__ __forceinline__ int64_t publish(int64_t i, int &nxt) const {
    if (!dyn) return static_unit(i);
    const int sl = (int)(i % CH_RING);
    mbar_wait_acq_cluster(&empty[sl], (uint32_t)((i / CH_RING) & 1) ^ 1u);
    int u = nxt < nitems ? nxt : -1;
    if (u >= 0) {
      nxt = atomicAdd(work, 1);
    } else if (atomicAdd(work + 1, 1) == (int)(gridDim.x >> 1) - 1) {
      work[0] = 0;
      work[1] = 0;
    }
    slot[sl] = u;
    st_cluster_s32(&slot[sl], 1, u);
    mbar_arrive(&full[sl]);
    mbar_arrive_cluster_release(&full[sl], 1);
    return u;
  }
  // other roles: the unit at ring position i; `arrive`: this thread frees the slot for its warp
  __device__ __forceinline__ int64_t take(int64_t i, bool arrive) const {
    if (!dyn) return static_unit(i);
    const int sl = (int)(i % CH_RING);
    mbar_wait_acq_cluster(&full[sl], (uint32_t)((i / CH_RING) & 1));
    const int u = *reinterpret_cast<volatile int32_t *>(&slot[sl]);
    __syncwarp(__activemask());
    if (arrive) mbar_arrive_cluster_release(&empty[sl], 0);
    return u;
  }
};


// The ring in `bytes` (CH_RING_BYTES of shared memory, 8-byte aligned).
__device__ __forceinline__ ChRing ch_ring_carve(uint8_t *bytes, bool dyn, int64_t nitems, int32_t *work) {
  ChRing r;
  r.full = reinterpret_cast<uint64_t *>(bytes);
  r.empty = r.full + CH_RING;
  r.slot = reinterpret_cast<int32_t *>(r.empty + CH_RING);
  r.dyn = dyn;
  r.nitems = nitems;
  r.work = work;
  return r;
}
// (thread 0, before ch_setup: its fence and cluster barrier publish the init)
__device__ __forceinline__ void ch_ring_init(const ChRing &r) {
  if (threadIdx.x == 0)
    for (int i = 0; i < CH_RING; ++i) {
      mbar_init(&r.full[i], 1);
      mbar_init(&r.empty[i], CH_RING_CONSUMERS);
    }
}

// Warp 0 lane 0 (both CTAs) of a chained kernel on the dynamic schedule: the leader's producer
// fetches and publishes the units (ChRing::publish), the peer's takes them; both load their halves.
template <class Sched>
__device__ __forceinline__ void ch_ring_producer(const Sched &sc, const ChRing &ring, const ChSmem &s, uint32_t cr,
                                                 const CUtensorMap *a_hi, const CUtensorMap *a_lo,
                                                 const CUtensorMap *b_hi, const CUtensorMap *b_lo, int nkb) {
  T2Smem ts;  // the producer only uses the stage ring
  ts.stages = s.stages;
  ts.full = s.full;
  ts.empty = s.empty;
  const T2Policy pol(sc.hint);
  int stage = 0;
  uint32_t phase = 0;
  int nxt = (ring.dyn && cr == 0) ? atomicAdd(ring.work, 1) : 0;
  for (int64_t i = 0;; ++i) {
    const int64_t u = cr == 0 ? ring.publish(i, nxt) : ring.take(i, true);
    if (u < 0) break;
    t2_produce_item(sc, ts, u, a_hi, a_lo, b_hi, b_lo, nkb, cr, pol, stage, phase);
  }
}

// Warp 1 lane 0 of the leader CTA on the dynamic schedule: the MMA issuer.
template <class Sched>
__device__ __forceinline__ void ch_ring_mma(const Sched &sc, const ChRing &ring, const ChSmem &s, int nkb, int nch,
                                            uint32_t idesc, uint32_t tmem_base) {
  int stage = 0;
  uint32_t phase = 0;
  int64_t chain = 0;
  for (int64_t i = 0;; ++i) {
    const int64_t u = ring.take(i, true);
    if (u < 0) break;
    ch_mma_item(sc, s, u, nkb, nch, idesc, tmem_base, stage, phase, chain);
  }
}

// Warps 0 (TMA producer, both CTAs) and 1 (MMA issuer, leader CTA) of a chained kernel.
template <class Sched>
__device__ __forceinline__ void ch_producer_mma(const Sched &sc, const ChSmem &s, int warp, int lane, uint32_t cr,
                                                const CUtensorMap *a_hi, const CUtensorMap *a_lo,
                                                const CUtensorMap *b_hi, const CUtensorMap *b_lo, int nkb, int nch,
                                                uint32_t idesc, uint32_t tmem_base, int hint = 1) {
  if (warp == 0) {
    if (lane == 0) {
      T2Smem ts;  // the producer only uses the stage ring
      ts.stages = s.stages;
      ts.full = s.full;
      ts.empty = s.empty;
      t2_producer(sc, ts, a_hi, a_lo, b_hi, b_lo, nkb, cr, hint);
    }
  } else if (lane == 0 && cr == 0) {
    ch_mma(sc, s, nkb, nch, idesc, tmem_base);
  }
}

// Both CTAs done with TMEM and with each other's smem, then the allocating warp frees TMEM.
__device__ __forceinline__ void ch_teardown(int warp, uint32_t tmem_base) {
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// Row part of a chunk: columns p0 .. p0 + 31 of a label-sorted set of n points with segments
// seg[0 .. k) (cluster c = sorted positions [seg[c], seg[c + 1])); this thread's row accumulates
// one running int64 fixed-point sum `run` of segment `cur`, flushed to Srow[cur] (red.add) when
// the segment changes. cseg: the warp's segment pointer (columns only move forward). x: kappa
// values with invalid columns / rows already zeroed.
__device__ __forceinline__ void ch_row_part(const float (&x)[32], int64_t p0, int64_t n, const int32_t *seg, int k,
                                            int &cseg, int &cur, long long &run, bool row_ok,
                                            long long *__restrict__ Srow, float fx) {
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
      if (cur >= 0 && row_ok) red_add_s64(Srow + cur, run);
      run = 0;
      cur = c0;
    }
    run += ch_fix(s2.x + s2.y, fx);
  } else {
    for (int cc = c0; cc <= c1; ++cc) {
      const int64_t lo = seg[cc] - p0, hi = (cc + 1 < k ? (int64_t)seg[cc + 1] : n) - p0;
      float sum = 0.f;
#pragma unroll
      for (int q = 0; q < 32; ++q) sum += (q >= lo && q < hi) ? x[q] : 0.f;
      if (cc != cur) {
        if (cur >= 0 && row_ok) red_add_s64(Srow + cur, run);
        run = 0;
        cur = cc;
      }
      run += ch_fix(sum, fx);
    }
  }
}

// Last segment c in [0, k) with seg[c] <= p (seg[0] = 0 <= p).
__device__ __forceinline__ int ch_segment_of(const int32_t *seg, int k, int64_t p) {
  int lo = 0, hi = k - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid] <= p) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// KIND of a KappaParams: 0 linear, 1 polynomial, 2 Gaussian, 3 polynomial of degree 2.
inline int ch_kind(const KappaParams &kp) { return kp.kind == 2 ? 2 : kp.kind == 1 ? (kp.degree == 2 ? 3 : 1) : 0; }

// fn(std::integral_constant<int, KIND>) for the kernel's KIND (compile-time specialised epilogues).
template <class F>
inline int ch_dispatch_kind(const KappaParams &kp, F &&fn) {
  switch (ch_kind(kp)) {
    case 2: return fn(std::integral_constant<int, 2>{});
    case 3: return fn(std::integral_constant<int, 3>{});
    case 1: return fn(std::integral_constant<int, 1>{});
    default: return fn(std::integral_constant<int, 0>{});
  }
}

}  // namespace kkm
