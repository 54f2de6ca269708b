// gemm_tc.cuh -- a1 on the 5th-generation tensor cores (placeholder until the
// tcgen05 kernel lands; KKM_PREC_BF16X3 reports failure).
#pragma once
#include "common.cuh"

namespace kkm {

struct TcGemm {
  int dummy = 0;
};

inline const char *tc_gemm_error() { return "tcgen05 GEMM not built yet"; }

inline int tc_gemm_launch(TcGemm &, const __nv_bfloat16 *, const __nv_bfloat16 *, int64_t, int64_t,
                          int64_t, int64_t, int64_t, int64_t, int64_t, const float *,
                          const KappaParams &, float *, int64_t, cudaStream_t, int64_t *) {
  return 1;
}
constexpr int TC_BK = 64;

}  // namespace kkm
