// stream.cuh -- host side of the fused streaming a1+a2 (K never stored; the kernels are
// tc3_stream_kernel in tc3.cuh and ssym_kernel in ssym.cuh): operand tensor maps of the A set and
// of the label-sorted B set (sort.cuh).
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
  int32_t *work = nullptr;  // tc3_stream_kernel's dynamic unit counters (allocated at first launch)
  TcStream() = default;
  TcStream(const TcStream &) = delete;
  TcStream &operator=(const TcStream &) = delete;
  ~TcStream() {
    if (work) cudaFree(work);
  }
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

}  // namespace kkm
