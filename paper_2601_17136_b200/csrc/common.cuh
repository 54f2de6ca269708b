// common.cuh -- device helpers shared by the kkm kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

namespace kkm {

constexpr int KKM_MAX_K = 900;  // finalize keeps (k + 1) x 32 doubles per block in smem (<= 227 KB)

// Opts kernel `fn` in to `bytes` of dynamic shared memory on the CURRENT device. The attribute
// belongs to a (function, device) pair, so the cache is keyed by both (a second handle on another
// device sets it again) and guarded by a mutex (handles may live on different host threads).
inline cudaError_t ensure_smem_attr(const void *fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(fn, dev);
  const auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}

// Kernel-function parameters as the device sees them (fp32 epilogue math).
struct KappaParams {
  int kind;            // KKM_KERNEL_*
  int degree;          // poly degree
  float gamma;         // poly gamma
  float coef0;         // poly offset
  float neg_gamma_log2e;  // Gaussian: -gamma * log2(e), so K = 2^(neg_gamma_log2e * r2)
};

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// kappa applied to b = x_i . x_j (Eqs. b, k; Gaussian by reading A1 with
// r^2 = (||x_i||^2 - b) + (||x_j||^2 - b) clamped at 0, reading A23; on the diagonal (same
// point, `same`) r^2 = 0 exactly so K_ii = 1 as the definition gives).
__device__ __forceinline__ float kappa_epilogue(const KappaParams &kp, float b, float ni, float nj,
                                                bool same = false) {
  if (kp.kind == 0) return b;
  if (kp.kind == 1) {
    float base = fmaf(kp.gamma, b, kp.coef0);
    float r = base;
    for (int e = 1; e < kp.degree; ++e) r *= base;
    return r;
  }
  float r2 = same ? 0.0f : fmaxf((ni - b) + (nj - b), 0.0f);  // exact differences for near points
  return ex2_approx(kp.neg_gamma_log2e * r2);
}


// d += a * b elementwise on float pairs: one FFMA2 (sm_100).
__device__ __forceinline__ void ffma2(float2 &d, float ax, float ay, float bx, float by) {
  unsigned long long dd = pack2(d.x, d.y);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(pack2(ax, ay)), "l"(pack2(bx, by)));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(dd));
}

__device__ __forceinline__ float mask_eq(int a, int b) { return a == b ? 1.0f : 0.0f; }

// Packed fp32 pair arithmetic (sm_100 add/mul/fma.rn.f32x2): one instruction for two lanes
// of work; operands are register pairs (x, y).
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pack2(a.x, a.y)), "l"(pack2(b.x, b.y)));
  float2 o;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pack2(a.x, a.y)), "l"(pack2(b.x, b.y)));
  float2 o;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pack2(a.x, a.y)), "l"(pack2(b.x, b.y)),
      "l"(pack2(c.x, c.y)));
  float2 o;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- mbarrier / bulk-copy PTX wrappers (Hopper+ async proxy) ----------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: a thread whose phase is not complete is suspended until the
// phase completes (or ~1 ms passes) instead of re-issuing the test -- waiting warps stop taking
// issue slots (and power) from the warps that work (ncu: the spin loops were ~35 % of the
// streaming kernel's executed instructions).
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef KKM_NO_WAIT_HINT
  while (!mbar_try_wait(bar, parity)) {
  }
#else
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
#endif
}
// Wait with exponential nanosleep backoff (32 ns .. 512 ns) between tests, for waits that are long
// and not latency-critical (epilogue warps waiting for a chain of ~4 us, the TMA producer waiting for
// a free stage): a spinning warp re-issues its test every few cycles and burns issue slots and power
// (ncu at n = 1M: the epilogue's spin loops were over half of the kernel's executed instructions).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
  uint32_t ns = 32;
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
  }
}

// L2 eviction-priority policies for .L2::cache_hint operands.
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
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

// 1-D bulk copy global -> shared, completing `bytes` on `bar` (cp.async.bulk, TMA engine).
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace kkm
