// gemm_tc.cuh -- shared tcgen05 / TMA building blocks of the tensor-core kernels in tc2.cuh:
// operand split reading A9 (bf16x3 or fp16x3: b = hi*hi + (hi*lo + lo*hi), 3 MMAs with fp32 TMEM
// accumulation, product error ~2^-16..2^-22 relative instead of bf16's 2^-8), the UMMA smem
// descriptor (128-byte swizzle, K-major), TMEM loads, L2 cache policies, TMA stores and the
// host-side operand tensor-map encoder (the kernels: tc3.cuh, ssym.cuh on chain.cuh).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace kkm {

constexpr int TC_BK = 64;  // K block = one 128-byte swizzle atom of 16-bit operands


// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
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


__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int c0, int c1, const void *smem_src,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src)), "l"(pol)
      : "memory");
}

// ---------------------------------------------------------------- host side
struct TcGemm {
  const void *hi = nullptr, *lo = nullptr;  // operands the tensor maps describe
  bool fp16 = false;
  CUtensorMap map_hi, map_lo;
  CUtensorMap map_out, map_out2;              // re-encoded per launch (cheap, host only)
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

// Resolves the driver's cuTensorMapEncodeTiled once; 0 on success.
inline int tc_encode_ready() {
  PFN_cuTensorMapEncodeTiled_v12000 &encode = tc_encode_fn();
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode) {
      encode = nullptr;
      tc_err_slot() = "cuTensorMapEncodeTiled unavailable";
      return 1;
    }
  }
  return 0;
}

inline int tc_make_maps(TcGemm &g, const uint16_t *Xhi, const uint16_t *Xlo, bool fp16, int64_t rows,
                        int64_t dp) {
  if (tc_encode_ready()) return 1;
  PFN_cuTensorMapEncodeTiled_v12000 &encode = tc_encode_fn();
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


}  // namespace kkm
