// stream.cuh -- host side of the fused streaming a1+a2 (K never stored; the kernels are
// tc3_stream_kernel in tc3.cuh and ssym_kernel in ssym.cuh): operand tensor maps of the A set and
// of the label-sorted B set (sort.cuh), and the choice of column splits per row tile.
#pragma once
#include "gemm_tc.cuh"

namespace kkm {

// ---------------------------------------------------------------- host side
struct TcStream {
  const void *ahi = nullptr, *alo = nullptr, *bhi = nullptr, *blo = nullptr;
  bool fp16 = false;
  int64_t arows = 0, brows = 0;
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
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

// Splits of the sorted column range: enough work units for a full last wave. Callers pass half
// the rows and the CTA-pair count, so 128-row tiles here are the kernel's 256-row pair tiles.
inline int ts_choose_splits(int64_t nloc, int64_t n, int num_sms) {
  const int64_t tiles_m = (nloc + 127) / 128;
  const int64_t tiles_n = (n + 255) / 256;
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
