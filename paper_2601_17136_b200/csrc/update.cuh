// update.cuh -- a3 and a4 of the iteration.
//   finalize:    E(i,c) = S(i,c) / |L_c| (Eq. e with Eq. v), z(i) = E(i, cl(i)) (Eq. z),
//                per-block fp64 partials of sum_{i in L_c} z(i) and of sum_i (K_ii - z_i)
//   cnorm_local: fixed-order sum of the block partials -> this rank's (k+1) partials
//   cnorm_final: fixed-order sum over ranks -> c(c) = ||mu_c||^2 (Eq. c; +inf if empty,
//                reading A7) and J = tr K - sum_c |L_c| c(c) (reading A8); also zeroes
//                the next iteration's size histogram and change counter
//   assign:      D(i,c) = -2E(i,c) + c(c) (Eq. d), lowest-index argmin (A6), new sizes
//                (exact int histogram) and the number of changed labels
// All reductions are fixed-order, so results are bitwise reproducible run to run.
#pragma once
#include "common.cuh"

namespace kkm {

constexpr int FIN_THREADS = 128;

// finalize's block size: the largest power of two <= FIN_THREADS with (k + 1) * threads doubles in
// the default 48 KB; from k = 192 on 32 threads and more than 48 KB (opted in by kkm_init).
inline int fin_threads(int k) {
  int fth = FIN_THREADS;
  while (fth > 32 && (size_t)(k + 1) * fth * 8 > 48 * 1024) fth >>= 1;
  return fth;
}
inline size_t fin_smem_bytes(int k) { return (size_t)(k + 1) * fin_threads(k) * 8; }

// grid: nblocks; block b handles rows [b * rows_per_block, ...). blockDim.x: a power of two
// <= FIN_THREADS; dynamic smem: (k + 1) * blockDim.x doubles.
// Sfix (optional): read S as int64 fixed point, Sfix[c * rows_pad + i] * inv (the 16-bit band
// path, spmm_tc.cuh) instead of the fp64 partials. fin (optional): the last block to finish also
// does cnorm_local + cnorm_final for a single "rank" (one rank, or the replicated a3 of §6) -- the
// same fixed-order sums, so the results are bitwise those of the separate kernels.
struct A3Fused {
  unsigned *counter;       // zero between launches (the last block resets it)
  const int32_t *sizes;
  double *cnorm, *J_out;
  int32_t *sizes_next;
  unsigned long long *changed_out;
};

__device__ __forceinline__ void cnorm_reduce_last(const double *__restrict__ blockpart, int nblocks, int k,
                                                  const A3Fused &f) {
  // = cnorm_local_kernel (one warp per c, lanes over blocks, fixed shuffle tree) + cnorm_final_kernel
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = threadIdx.x >> 5; c <= k; c += nw) {
    double sum = 0.0;
    int b = lane;
    for (; b + 32 * 7 < nblocks; b += 32 * 8) {  // 8 L2 loads in flight, added in the same order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(blockpart + (int64_t)(b + 32 * u) * (k + 1) + c);
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; b < nblocks; b += 32) sum += __ldcg(blockpart + (int64_t)b * (k + 1) + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      const double s = 0.0 + sum;  // (cnorm_final: the sum over one rank)
      if (c < k) {
        const int32_t sz = f.sizes[c];
        f.cnorm[c] = sz > 0 ? s / (double)sz : __longlong_as_double(0x7ff0000000000000LL);  // +inf
        if (f.sizes_next) f.sizes_next[c] = 0;
      } else if (f.J_out) {
        *f.J_out = s;
      }
    }
  }
  if (threadIdx.x == 0 && f.changed_out) *f.changed_out = 0ull;
}

__global__ void __launch_bounds__(128) finalize_kernel(
    const double *__restrict__ Spart, int nsplit, int64_t nrows, int64_t rows_pad, int k,
    const int32_t *__restrict__ sizes, const int32_t *__restrict__ cl_local,
    const double *__restrict__ diag, int64_t rows_per_block, double *__restrict__ E,
    double *__restrict__ blockpart, const long long *__restrict__ Sfix = nullptr, double inv = 1.0,
    A3Fused fin = A3Fused{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr}) {
  extern __shared__ double sacc[];  // [(k + 1)][blockDim.x]
  __shared__ unsigned s_last;
  const int T = blockDim.x;
  const int t = threadIdx.x;
  for (int c = 0; c <= k; ++c) sacc[c * T + t] = 0.0;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = rb + rows_per_block < nrows ? rb + rows_per_block : nrows;
  for (int64_t i = rb + t; i < re; i += T) {
    const int li = cl_local[i];
    double zi = 0.0;
    if (Sfix && k <= 16) {  // all k loads in flight first (the caller guarantees k <= 16 here)
      long long sv[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) sv[c] = c < k ? Sfix[(int64_t)c * rows_pad + i] : 0ll;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < k) {
          const double s = 0.0 + (double)sv[c] * inv;
          const int32_t sz = sizes[c];
          const double e = sz > 0 ? s / (double)sz : 0.0;
          E[i * k + c] = e;
          if (c == li) zi = e;
        }
    } else {
      for (int c = 0; c < k; ++c) {
        double s = 0.0;
        if (Sfix) {
          s += (double)Sfix[(int64_t)c * rows_pad + i] * inv;
        } else {
          for (int p = 0; p < nsplit; ++p) s += Spart[((int64_t)p * rows_pad + i) * k + c];
        }
        const int32_t sz = sizes[c];
        const double e = sz > 0 ? s / (double)sz : 0.0;
        E[i * k + c] = e;
        if (c == li) zi = e;
      }
    }
    sacc[li * T + t] += zi;
    sacc[k * T + t] += diag[i] - zi;
  }
  __syncthreads();
  // fixed tree over the T threads: levels w >= 32 in shared memory, the last five levels as warp
  // shuffles (lane t adds lane t + w: the same pairs, so the same bits as the all-smem tree)
  for (int w = T / 2; w >= 32; w >>= 1) {
    if (t < w)
      for (int c = 0; c <= k; ++c) sacc[c * T + t] += sacc[c * T + t + w];
    __syncthreads();
  }
  {
    const int lane = t & 31, nw = T >> 5;
    for (int c = t >> 5; c <= k; c += nw) {
      double v = sacc[c * T + lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) blockpart[(int64_t)blockIdx.x * (k + 1) + c] = v;
    }
  }
  if (!fin.counter) return;
  __threadfence();
  __syncthreads();
  if (t == 0) {
    s_last = atomicAdd(fin.counter, 1u) == gridDim.x - 1;
    if (s_last) {
      *fin.counter = 0u;
      __threadfence();
    }
  }
  __syncthreads();
  if (s_last) cnorm_reduce_last(blockpart, gridDim.x, k, fin);
}

// out[c] = sum_b blockpart[b][c]: one warp per c, lane l sums b = l, l + 32, ... in order,
// then a fixed shuffle tree (deterministic, independent of timing).
__global__ void cnorm_local_kernel(const double *__restrict__ blockpart, int nblocks, int k,
                                   double *__restrict__ out) {
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = threadIdx.x >> 5; c <= k; c += nw) {
    double s = 0.0;
    for (int b = lane; b < nblocks; b += 32) s += blockpart[(int64_t)b * (k + 1) + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
  }
}

// rankpart: [nranks][k + 1]. Writes cnorm[k], J_out[0]; zeroes sizes_next[k], changed_out[0].
__global__ void cnorm_final_kernel(const double *__restrict__ rankpart, int nranks, int k,
                                   const int32_t *__restrict__ sizes, double *__restrict__ cnorm,
                                   double *__restrict__ J_out, int32_t *__restrict__ sizes_next,
                                   unsigned long long *__restrict__ changed_out) {
  for (int c = threadIdx.x; c <= k; c += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += rankpart[(int64_t)r * (k + 1) + c];
    if (c < k) {
      const int32_t sz = sizes[c];
      cnorm[c] = sz > 0 ? s / (double)sz : __longlong_as_double(0x7ff0000000000000LL);  // +inf
      if (sizes_next) sizes_next[c] = 0;
    } else if (J_out) {
      *J_out = s;  // sum_i (K_ii - z_i) = tr K - sum_c |L_c| c(c)
    }
  }
  if (threadIdx.x == 0 && changed_out) *changed_out = 0ull;
}

// One thread per local row. new_labels / old labels are the rank's slice.
__global__ void assign_kernel(const double *__restrict__ E, int64_t nrows, int k,
                              const double *__restrict__ cnorm, const double *__restrict__ diag,
                              const int32_t *__restrict__ cl_old, int32_t *__restrict__ cl_new,
                              int32_t *__restrict__ sizes_next,
                              unsigned long long *__restrict__ changed_out,
                              double *__restrict__ Dfull) {
  extern __shared__ int32_t hist[];
  for (int c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned changed = 0;
  if (i < nrows) {
    int best = 0;
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    for (int c = 0; c < k; ++c) {
      const double cn = cnorm[c];
      const double dsh = isinf(cn) ? cn : fma(-2.0, E[i * k + c], cn);
      if (Dfull) Dfull[i * k + c] = diag[i] + dsh;
      if (dsh < bd) {
        bd = dsh;
        best = c;
      }
    }
    cl_new[i] = best;
    changed = (best != cl_old[i]);
    atomicAdd(&hist[best], 1);
  }
  const unsigned wc = __reduce_add_sync(0xffffffffu, changed);
  if ((threadIdx.x & 31) == 0 && wc) atomicAdd(changed_out, (unsigned long long)wc);
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    if (hist[c]) atomicAdd(&sizes_next[c], hist[c]);
}

// Out-of-sample assignment (kkm_predict): one thread per new point y.
// E(y, c) = S(y, c) / |L_c| from the streaming partials, D(y, c) = K(y, y) - 2 E(y, c) + c(c)
// (Eq. d), lowest-index argmin on -2E + c exactly as assign_kernel (A6, A7).
__global__ void predict_kernel(const double *__restrict__ Spart, int nsplit, int64_t m, int64_t rows_pad, int k,
                               const int32_t *__restrict__ sizes, const double *__restrict__ cnorm,
                               const double *__restrict__ diag, int32_t *__restrict__ labels,
                               double *__restrict__ Dfull) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int best = 0;
  double bd = __longlong_as_double(0x7ff0000000000000LL);
  for (int c = 0; c < k; ++c) {
    double s = 0.0;
    for (int p = 0; p < nsplit; ++p) s += Spart[((int64_t)p * rows_pad + i) * k + c];
    const int32_t sz = sizes[c];
    const double e = sz > 0 ? s / (double)sz : 0.0;
    const double cn = cnorm[c];
    const double dsh = isinf(cn) ? cn : fma(-2.0, e, cn);
    if (Dfull) Dfull[i * k + c] = diag[i] + dsh;
    if (dsh < bd) {
      bd = dsh;
      best = c;
    }
  }
  labels[i] = best;
}

}  // namespace kkm

namespace kkm {

// ---- f3: incremental S (kkm_params.incremental)
// S1[i][c] = sum_s S[(s * rows_pad + i) * k + c] (fixed order) for the own rows i < nrows.
__global__ void sinc_set_kernel(const double *__restrict__ S, int nsplit, int64_t rows_pad, int64_t nrows, int k,
                                double *__restrict__ S1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows * k) return;
  const int64_t i = t / k;
  const int c = (int)(t % k);
  double s = 0.0;
  for (int p = 0; p < nsplit; ++p) s += S[((int64_t)p * rows_pad + i) * k + c];
  S1[t] = s;
}

// S1[i][c] += sign * sum_s Sd[s][i][c] (fixed order) for the own rows i < nrows.
__global__ void sinc_add_kernel(const double *__restrict__ Sd, int nsplit, int64_t rows_pad, int64_t nrows, int k,
                                double sign, double *__restrict__ S1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows * k) return;
  const int64_t i = t / k;
  const int c = (int)(t % k);
  double s = 0.0;
  for (int p = 0; p < nsplit; ++p) s += Sd[((int64_t)p * rows_pad + i) * k + c];
  S1[t] += sign * s;
}

// Sort key of the moved points: key[i] = new (or old) label if cl_old[i] != cl_new[i], else k
// (the bucket after the last cluster: not moved); -1 beyond n.
__global__ void moved_key_kernel(const int32_t *__restrict__ cl_old, const int32_t *__restrict__ cl_new, int64_t n,
                                 int64_t len, int k, int use_new, int32_t *__restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  int32_t v = -1;
  if (i < n) v = cl_old[i] != cl_new[i] ? (use_new ? cl_new[i] : cl_old[i]) : k;
  key[i] = v;
}

// ---- a3 + a4 in ONE grid-wide launch over the int64 fixed-point S (the 16-bit band / f1 paths on
// one rank or replicated, k <= UG_MAX_K): a cooperative launch (all blocks co-resident) with a grid
// barrier. Phase 1: z_i = E(i, cl_i) = (S(i, cl_i) 2^-s) / |L_cl_i| (Eq. z) -- ONE S value per row
// -- and per-cluster sums of z plus sum_i (K_ii - z_i), reduced per warp by a 31-shuffle
// reduce-scatter butterfly (lane l ends with cluster l's sum) and per block over its warps in
// order, into blockpart. Grid barrier. Every block sums blockpart over the blocks in the same
// fixed order, so every block holds the same c and J (Eqs. c, A8) -- no second launch. Phase 2:
// per row all k S values, E = S 2^-s / |L_c| (bitwise the value finalize stores), D = -2E + c, the
// lowest-index argmin (A6), new labels, the exact integer size histogram and the changed count.
// The E rows are stored (debug reads); the full distances are formed on demand (dfull_kernel).
//
// LSA = true (several ranks on one NVLink domain): the a2 all-reduce of S is fused in
// and the update is DISTRIBUTED instead of replicated. Every rank's S lives in an NCCL symmetric
// window mapped by all ranks (peer pointers, load/store over NVLink); a rank handles only its own
// 1D block of rows: S(i, c) = the sum of the P ranks' S(i, c) read in rank order (exact integers),
// its per-cluster partials go to every rank's table (peer stores), and after a cross-rank barrier
// every rank sums the P partials in rank order (the same c and J everywhere); the new labels, the
// size histogram and the changed count are stored / added into every rank's copies. Three
// cross-rank arrivals per launch (S complete; partials published; labels landed), each one
// red.release.sys per peer on the peers' flag words and an acquire spin on the own one.
constexpr int UG_THREADS = 256;
constexpr int UG_MAX_K = 64;
constexpr int LSA_MAX_RANKS = 8;

struct LsaArgs {
  uint8_t *base[LSA_MAX_RANKS];  // every rank's window, as mapped in this process (base[rank]: own)
  int nranks, rank;
  int64_t row0;                  // this rank's rows [row0, row0 + nrows)
  size_t off_S, off_lab_next, off_sizes_next, off_changed, off_rankpart, off_flag;
  unsigned target;               // arrivals the first cross-rank wait needs (then + nranks, + 2 nranks)
  long long *Sred;               // [k][rows_pad] (own rows used): the ranks' S summed (phase 0)
};

__device__ __forceinline__ void grid_barrier(unsigned *bar) {  // bar[0]: arrivals, bar[1]: generation
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = *reinterpret_cast<volatile unsigned *>(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned *>(bar) = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      uint32_t ns = 32;
      while (*reinterpret_cast<volatile unsigned *>(bar + 1) == gen) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Cross-rank arrival (block 0, after a system-scope fence: its own and -- through the preceding
// grid barrier -- the grid's peer stores are visible first) and wait (every block, or only block
// 0 with all_wait = false) until the own flag reaches `target`. A rank that never arrives is
// bounded by ~600 s of %globaltimer: the own flag page's word 16 is set (the host reports
// KKM_ENCCL) and the kernel finishes on whatever it reads.
__device__ __forceinline__ void lsa_arrive_wait(const LsaArgs &L, unsigned target, bool all_wait) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();
      for (int p = 0; p < L.nranks; ++p)
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(L.base[p] + L.off_flag) : "memory");
    }
    if (all_wait || blockIdx.x == 0) {
      const unsigned *flag = reinterpret_cast<const unsigned *>(L.base[L.rank] + L.off_flag);
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (uint32_t ns = 32;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if ((int)(v - target) >= 0) break;
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 600ull * 1000000000ull) {
          atomicExch(reinterpret_cast<unsigned *>(L.base[L.rank] + L.off_flag) + 16, 1u);
          break;
        }
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
    }
  }
  __syncthreads();
}

// S(i, c): this rank's (LSA = false) or the ranks' sum of the own rows (phase 0's local copy).
template <bool LSA>
__device__ __forceinline__ long long s_load(const long long *__restrict__ Sfix, const LsaArgs &L, int64_t idx) {
  return LSA ? __ldcg(L.Sred + idx) : Sfix[idx];
}

// Phase 0 of the distributed update: Sred[c][i] = sum over the ranks (rank order; exact integers)
// of their S[c][i] for the own rows i, every c -- the reduce-scatter of S done by the kernel with
// all P (P - 1 of them remote, over NVLink) loads of two elements in flight per thread.
__device__ __forceinline__ void lsa_reduce_own(const LsaArgs &L, int64_t rows_pad, int64_t nrows, int k) {
  constexpr int U = 4;  // elements per thread and pass: U x P loads in flight
  const int64_t total = nrows * k, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += U * stride) {
    int64_t x[U];
    long long v[U][LSA_MAX_RANKS];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      x[u] = e < total ? (e / nrows) * rows_pad + L.row0 + e % nrows : -1;
    }
#pragma unroll
    for (int p = 0; p < LSA_MAX_RANKS; ++p)
      if (p < L.nranks) {
        const long long *S = reinterpret_cast<const long long *>(L.base[p] + L.off_S);
#pragma unroll
        for (int u = 0; u < U; ++u) v[u][p] = x[u] >= 0 ? __ldcv(S + x[u]) : 0ll;
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long sum = 0;
#pragma unroll
      for (int p = 0; p < LSA_MAX_RANKS; ++p)
        if (p < L.nranks) sum += v[u][p];
      if (x[u] >= 0) L.Sred[x[u]] = sum;
    }
  }
}

#ifdef KKM_EXP_LSA_STAMPS  // (A/B experiment builds only: block 0's phase timestamps into the flag page)
#define LSA_STAMP(j)                                                                                      \
  if (LSA && blockIdx.x == 0 && threadIdx.x == 0) {                                                      \
    unsigned long long ts_;                                                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_));                                              \
    reinterpret_cast<unsigned long long *>(L.base[L.rank] + L.off_flag)[32 + (j)] = ts_;                 \
  }
#else
#define LSA_STAMP(j)
#endif

template <bool LSA>
__global__ void __launch_bounds__(UG_THREADS) update_grid_kernel(
    const long long *__restrict__ Sfix, int64_t rows_pad, int64_t nrows, int k, double inv,
    const int32_t *__restrict__ sizes, const int32_t *__restrict__ cl, const double *__restrict__ diag,
    double *__restrict__ E, double *__restrict__ blockpart, unsigned *__restrict__ bar, double *__restrict__ cnorm_out,
    double *__restrict__ J_out, int32_t *__restrict__ cl_new, int32_t *__restrict__ sizes_next,
    unsigned long long *__restrict__ changed_out, LsaArgs L) {
  __shared__ double wpart[UG_THREADS / 32][UG_MAX_K + 1];
  __shared__ double cn[UG_MAX_K];
  __shared__ int hist[UG_MAX_K];
  __shared__ unsigned long long nchg;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = UG_THREADS / 32;
  const int64_t stride = (int64_t)gridDim.x * UG_THREADS;
  const int64_t r0 = LSA ? L.row0 : 0;  // rows r0 + [0, nrows)
  if (blockIdx.x == 0) {  // zeroed before the barrier (LSA: before this rank's second arrival), accumulated after
    for (int c = t; c < k; c += UG_THREADS) sizes_next[c] = 0;
    if (t == 0) *changed_out = 0ull;
  }
  LSA_STAMP(0)
  if (LSA) {
    lsa_arrive_wait(L, L.target, true);  // every rank's S is complete
    LSA_STAMP(1)
    lsa_reduce_own(L, rows_pad, nrows, k);
    __threadfence();
    grid_barrier(bar);
  }
  LSA_STAMP(9)
  // ---- phase 1: per-cluster sums of z and sum (K_ii - z_i)
  double acc0 = 0.0, acc1 = 0.0, accJ = 0.0;  // lane l: clusters l and l + 32
  for (int64_t base = (int64_t)blockIdx.x * UG_THREADS + (t & ~31); base < nrows; base += stride) {
    const int64_t i = r0 + base + lane;
    int li = -1;
    double zi = 0.0, ji = 0.0;
    if (base + lane < nrows) {
      li = cl[i];
      const int32_t sz = sizes[li];
      const double sv = 0.0 + (double)s_load<LSA>(Sfix, L, (int64_t)li * rows_pad + i) * inv;
      zi = sz > 0 ? sv / (double)sz : 0.0;
      ji = diag[i] - zi;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h * 32 >= k) break;
      double v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = (li == h * 32 + q) ? zi : 0.0;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {  // reduce-scatter butterfly: lane l keeps the sum of v[l]
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int q = 0; q < o; ++q) {
          const double send = up ? v[q] : v[q + o];
          const double keep = up ? v[q + o] : v[q];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (h == 0) acc0 += v[0];
      else acc1 += v[0];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ji += __shfl_xor_sync(0xffffffffu, ji, o);
    accJ += ji;
  }
  if (lane < k) wpart[w][lane] = acc0;
  if (lane + 32 < k) wpart[w][lane + 32] = acc1;
  if (lane == 0) wpart[w][k] = accJ;
  __syncthreads();
  for (int c = t; c <= k; c += UG_THREADS) {
    double sum = 0.0;
    for (int q = 0; q < nw; ++q) sum += wpart[q][c];
    blockpart[(int64_t)blockIdx.x * (k + 1) + c] = sum;
  }
  LSA_STAMP(2)
  grid_barrier(bar);
  LSA_STAMP(3)
  // ---- the grid's (k + 1) sums, by every block in the same fixed order
  for (int c = w; c <= k; c += nw) {
    double sum = 0.0;
    int b = lane;
    for (; b + 32 * 7 < (int)gridDim.x; b += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(blockpart + (int64_t)(b + 32 * u) * (k + 1) + c);
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; b < (int)gridDim.x; b += 32) sum += __ldcg(blockpart + (int64_t)b * (k + 1) + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      if (LSA) {  // this rank's partial -> every rank's table (block 0), then summed over the ranks below
        if (blockIdx.x == 0)
          for (int p = 0; p < L.nranks; ++p)
            reinterpret_cast<double *>(L.base[p] + L.off_rankpart)[L.rank * (k + 1) + c] = sum;
      } else if (c < k) {
        const int32_t sz = sizes[c];
        const double v = sz > 0 ? sum / (double)sz : __longlong_as_double(0x7ff0000000000000LL);  // +inf (A7)
        cn[c] = v;
        if (blockIdx.x == 0) cnorm_out[c] = v;
      } else if (blockIdx.x == 0) {
        *J_out = sum;  // sum_i (K_ii - z_i) = tr K - sum_c |L_c| c(c) (A8)
      }
    }
  }
  if (LSA) {
    LSA_STAMP(4)
    lsa_arrive_wait(L, L.target + L.nranks, true);  // every rank's partials published
    LSA_STAMP(5)
    const double *rp = reinterpret_cast<const double *>(L.base[L.rank] + L.off_rankpart);
    for (int c = t; c <= k; c += UG_THREADS) {
      double sum = 0.0;
      for (int p = 0; p < L.nranks; ++p) sum += __ldcv(rp + p * (k + 1) + c);
      if (c < k) {
        const int32_t sz = sizes[c];
        const double v = sz > 0 ? sum / (double)sz : __longlong_as_double(0x7ff0000000000000LL);
        cn[c] = v;
        if (blockIdx.x == 0) cnorm_out[c] = v;
      } else if (blockIdx.x == 0) {
        *J_out = sum;
      }
    }
  }
  for (int c = t; c < k; c += UG_THREADS) hist[c] = 0;
  if (t == 0) nchg = 0ull;
  __syncthreads();
  // ---- phase 2: E, D, argmin, sizes, changed
  unsigned changed = 0;
  for (int64_t li0 = (int64_t)blockIdx.x * UG_THREADS + t; li0 < nrows; li0 += stride) {
    const int64_t i = r0 + li0;
    int best = 0;
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    for (int c0 = 0; c0 < k; c0 += 16) {
      long long sv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) sv[q] = c0 + q < k ? s_load<LSA>(Sfix, L, (int64_t)(c0 + q) * rows_pad + i) : 0ll;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int c = c0 + q;
        if (c < k) {
          const double s = 0.0 + (double)sv[q] * inv;
          const int32_t sz = sizes[c];
          const double e = sz > 0 ? s / (double)sz : 0.0;
          if (E) E[i * k + c] = e;
          const double cv = cn[c];
          const double dsh = isinf(cv) ? cv : fma(-2.0, e, cv);
          if (dsh < bd) {
            bd = dsh;
            best = c;
          }
        }
      }
    }
    if (LSA) {
      for (int p = 0; p < L.nranks; ++p) reinterpret_cast<int32_t *>(L.base[p] + L.off_lab_next)[i] = best;
    } else {
      cl_new[i] = best;
    }
    changed += best != cl[i];
    atomicAdd(&hist[best], 1);
  }
  const unsigned wc = __reduce_add_sync(0xffffffffu, changed);
  if (lane == 0 && wc) atomicAdd(&nchg, (unsigned long long)wc);
  __syncthreads();
  if (LSA) {
    for (int c = t; c < k; c += UG_THREADS)
      if (hist[c])
        for (int p = 0; p < L.nranks; ++p)
          atomicAdd(reinterpret_cast<int32_t *>(L.base[p] + L.off_sizes_next) + c, hist[c]);
    if (t == 0 && nchg)
      for (int p = 0; p < L.nranks; ++p)
        atomicAdd(reinterpret_cast<unsigned long long *>(L.base[p] + L.off_changed), nchg);
    LSA_STAMP(6)
    __threadfence_system();
    grid_barrier(bar);  // every block's peer stores issued and fenced
    LSA_STAMP(7)
    lsa_arrive_wait(L, L.target + 2 * L.nranks, false);  // block 0: every rank's labels landed here
    LSA_STAMP(8)
  } else {
    for (int c = t; c < k; c += UG_THREADS)
      if (hist[c]) atomicAdd(&sizes_next[c], hist[c]);
    if (t == 0 && nchg) atomicAdd(changed_out, nchg);
  }
}

// Dfull(i, c) = K_ii + D(i, c) from the stored E and c (debug reads; the same expression as assign).
__global__ void dfull_kernel(const double *__restrict__ E, int64_t nrows, int k, const double *__restrict__ cnorm,
                             const double *__restrict__ diag, double *__restrict__ Dfull) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows * k) return;
  const int64_t i = t / k;
  const int c = (int)(t % k);
  const double cn = cnorm[c];
  Dfull[t] = diag[i] + (isinf(cn) ? cn : fma(-2.0, E[t], cn));
}

}  // namespace kkm

namespace kkm {

// ---- a3 + a4 in one CTA (single rank, n <= FUSED_MAX_ROWS, k <= 16): the launch-latency bound
// regime (config 1). Same arithmetic as finalize / cnorm_* / assign (fixed-order sums: thread
// partials over rows t, t + T, ..., then a fixed tree; exact integer histogram), one launch
// instead of four. Writes E, cnorm, *J_out; with do_assign also Dfull, the new labels,
// sizes_next (stored, not accumulated) and *changed_out.
constexpr int FUSED_THREADS = 512;
constexpr int64_t FUSED_MAX_ROWS = 32768;

__global__ void __launch_bounds__(FUSED_THREADS) fused_update_kernel(
    const double *__restrict__ S, int nsplit, int64_t n, int64_t rows_pad, int k, const int32_t *__restrict__ sizes,
    const int32_t *__restrict__ cl, const double *__restrict__ diag, double *__restrict__ E,
    double *__restrict__ cnorm, double *__restrict__ J_out, int do_assign, int32_t *__restrict__ cl_new,
    int32_t *__restrict__ sizes_next, unsigned long long *__restrict__ changed_out, double *__restrict__ Dfull) {
  extern __shared__ double sacc[];  // [(k + 1)][T], then cn[k]
  __shared__ int hist[16];
  __shared__ unsigned long long nchg;
  const int T = blockDim.x, t = threadIdx.x;
  double *cn = sacc + (size_t)(k + 1) * T;
  for (int c = 0; c <= k; ++c) sacc[c * T + t] = 0.0;
  if (t < 16) hist[t] = 0;
  if (t == 0) nchg = 0ull;
  for (int64_t i = t; i < n; i += T) {
    const int li = cl[i];
    double zi = 0.0;
    for (int c = 0; c < k; ++c) {
      double s = 0.0;
      for (int p = 0; p < nsplit; ++p) s += S[((int64_t)p * rows_pad + i) * k + c];
      const int32_t sz = sizes[c];
      const double e = sz > 0 ? s / (double)sz : 0.0;
      E[i * k + c] = e;
      if (c == li) zi = e;
    }
    sacc[li * T + t] += zi;
    sacc[k * T + t] += diag[i] - zi;
  }
  __syncthreads();
  for (int w = T / 2; w >= 32; w >>= 1) {  // the same fixed tree as finalize (last five levels shuffled)
    if (t < w)
      for (int c = 0; c <= k; ++c) sacc[c * T + t] += sacc[c * T + t + w];
    __syncthreads();
  }
  for (int c = t >> 5; c <= k; c += T >> 5) {
    double v = sacc[c * T + (t & 31)];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) sacc[c * T] = v;
  }
  __syncthreads();
  if (t < k) {
    const int32_t sz = sizes[t];
    const double v = sz > 0 ? sacc[t * T] / (double)sz : __longlong_as_double(0x7ff0000000000000LL);
    cnorm[t] = v;
    cn[t] = v;
  }
  if (t == 0) *J_out = sacc[k * T];
  __syncthreads();
  if (!do_assign) return;
  unsigned changed = 0;
  for (int64_t i = t; i < n; i += T) {
    int best = 0;
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    for (int c = 0; c < k; ++c) {
      const double cv = cn[c];
      const double dsh = isinf(cv) ? cv : fma(-2.0, E[i * k + c], cv);
      if (Dfull) Dfull[i * k + c] = diag[i] + dsh;
      if (dsh < bd) {
        bd = dsh;
        best = c;
      }
    }
    cl_new[i] = best;
    changed += best != cl[i];
    atomicAdd(&hist[best], 1);
  }
  const unsigned wc = __reduce_add_sync(0xffffffffu, changed);
  if ((t & 31) == 0 && wc) atomicAdd(&nchg, (unsigned long long)wc);
  __syncthreads();
  if (t < k) sizes_next[t] = hist[t];
  if (t == 0) *changed_out = nchg;
}

}  // namespace kkm
