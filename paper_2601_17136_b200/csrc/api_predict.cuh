// api_predict.cuh -- kkm_predict internals (f4: out-of-sample assignment): scratch layout and the
// pass over Y (split operands, self dots, the streaming kernel against X sorted by label, argmin).
#pragma once

namespace {

// Layout of kkm_predict's scratch: Y operands, sort scratch, sorted X (materialised handles
// only: streaming handles lend their own), the partials and the outputs.
struct PredictPlan {
  int64_t mpad;
  int nblk;
  bool own_sorted;
  size_t oYf, oYhi, oYlo, oYn, oYr, oYd, oSp, oSx, oFx, oLab, oD, oPerm, oPos, oSeg, oBc, oBo, oShi, oSlo, oSn, oSr,
      total;
};

PredictPlan predict_plan(const kkm_ctx *h, int64_t m) {
  const Plan &P = h->P;
  PredictPlan q;
  q.mpad = round_up(std::max<int64_t>(m, 1), 256);
  q.nblk = (int)ceil_div(P.n, SORT_BLOCK);
  q.own_sorted = P.materialize;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const int k = P.k;
  q.oYf = take((size_t)q.mpad * P.ldf * 4);
  q.oYhi = take((size_t)q.mpad * P.dp * 2);
  q.oYlo = take((size_t)q.mpad * P.dp * 2);
  q.oYn = take((size_t)q.mpad * 4);
  q.oYr = take((size_t)q.mpad * 4);
  q.oYd = take((size_t)q.mpad * 8);
  q.oSp = take((size_t)q.mpad * k * 8);
  q.oSx = take((size_t)q.mpad * k * 8);
  q.oFx = take(16);
  q.oLab = take((size_t)q.mpad * 4);
  q.oD = take((size_t)q.mpad * k * 8);
  q.oPerm = take((size_t)P.lablen * 4);
  q.oPos = take((size_t)P.lablen * 4);
  q.oSeg = take((size_t)(k + 1) * 4);
  q.oBc = take((size_t)q.nblk * k * 4);
  q.oBo = take((size_t)q.nblk * k * 4);
  q.oShi = q.own_sorted ? take((size_t)P.npad * P.dp * 2) : 0;
  q.oSlo = q.own_sorted ? take((size_t)P.npad * P.dp * 2) : 0;
  q.oSn = q.own_sorted ? take((size_t)P.npad * 4) : 0;
  q.oSr = q.own_sorted ? take((size_t)P.npad * 4) : 0;
  q.total = off;
  return q;
}

int predict_run(kkm_ctx *h, const PredictPlan &q, uint8_t *t, const float *Y, int64_t m, int64_t ldy,
                int32_t *labels_out, double *D_out) {
  const Plan &P = h->P;
  const int k = P.k;
  float *Yf = (float *)(t + q.oYf), *yn = (float *)(t + q.oYn), *yr = (float *)(t + q.oYr);
  uint16_t *Yhi = (uint16_t *)(t + q.oYhi), *Ylo = (uint16_t *)(t + q.oYlo);
  double *yd = (double *)(t + q.oYd), *Sp = (double *)(t + q.oSp), *Dy = D_out ? (double *)(t + q.oD) : nullptr;
  int32_t *ylab = (int32_t *)(t + q.oLab);
  const bool own = q.own_sorted;
  SortedSet B{own ? (uint16_t *)(t + q.oShi) : h->Shi, own ? (uint16_t *)(t + q.oSlo) : h->Slo,
              own ? (float *)(t + q.oSn) : h->snorms, own ? (float *)(t + q.oSr) : h->srscale,
              (int32_t *)(t + q.oPerm), (int32_t *)(t + q.oPos), (int32_t *)(t + q.oSeg), (int32_t *)(t + q.oBc),
              (int32_t *)(t + q.oBo)};
  // a5 for the new points: split operands, norms, kappa(y, y) (prep_rows and diag read only
  // rows < m and columns < d of Yf, and write the split's pad rows/columns as zeros)
  CK(cudaMemcpy2DAsync(Yf, P.ldf * 4, Y, ldy * 4, P.d * 4, m, cudaMemcpyDefault, h->st));
  if (h->p.kind == KKM_KERNEL_GAUSSIAN) {  // the training points were centered (kkm_init)
    center_rows_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, h->st>>>(Yf, P.ldf, m, P.d, h->mean);
    CKL();
  }
  prep_rows_kernel<<<(unsigned)ceil_div(q.mpad, 8), 256, 0, h->st>>>(Yf, P.ldf, m, q.mpad, P.d, yn, Yhi, Ylo, P.dp,
                                                                     P.fp16 ? 2 : 1, yr);
  CKL();
  if (h->p.kind == KKM_KERNEL_GAUSSIAN) {  // the tensor core's own y . y, as the training norms (kkm_init)
    TcGemm gy;
    if (tc3_self_dots(gy, Yhi, Ylo, P.fp16, yr, q.mpad, P.dp, m, yn, h->st, &h->launches, h->chain_kb)) {
      h->poisoned = true;
      return fail(KKM_ECUDA, "tensor-core self dots failed: %s", tc_gemm_error());
    }
  }
  diag_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, h->st>>>(Yf, P.ldf, P.d, 0, m, h->p.kind, h->p.gamma, h->p.coef0,
                                                            h->p.degree, yd);
  CKL();
  // B = all n training points sorted by their current labels; A = Y
  CKR(sort_gather(h, h->lab[h->cur], 0, P.n, P.npad, B));
  TcStream &ts = h->ts_predict;
  const StreamA A{Yhi, Ylo, yn, yr, q.mpad, 0, m, q.mpad};
  // fixed-point scale of the streaming sums: n max|K(y, x)| 2^s < 2^61, |K(y, x)| <= max(K(y, y), K(x, x))
  double kmax = 1.0;
  if (h->p.kind != KKM_KERNEL_GAUSSIAN) {
    float *fm = (float *)(t + q.oFx);
    max_norm_kernel<<<1, 1024, 0, h->st>>>(h->norms, P.n, fm);
    CKL();
    max_norm_kernel<<<1, 1024, 0, h->st>>>(yn, m, fm + 1);
    CKL();
    float mx[2] = {0.f, 0.f};
    CK(cudaMemcpyAsync(mx, fm, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const double nm = std::max((double)mx[0], (double)mx[1]);
    kmax = h->p.kind == KKM_KERNEL_LINEAR ? std::max(1e-30, nm)
                                          : std::pow(h->p.gamma * nm + std::fabs(h->p.coef0), (double)h->p.degree);
  }
  const double fx = std::ldexp(1.0, (int)std::floor(61.0 - std::log2(std::max(1e-300, (double)P.n * kmax * 1.0001))));
  CKR(stream_pass(h, ts, A, B, P.npad, P.n, 0, nullptr, 0, fx, (long long *)(t + q.oSx), Sp));
  predict_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, h->st>>>(Sp, 1, m, q.mpad, k, h->sizes[h->cur],
                                                                h->cnorm2, yd, ylab, Dy);
  CKL();
  CKR(copy_any(h, labels_out, ylab, (size_t)m * 4));
  if (D_out) CKR(copy_any(h, D_out, Dy, (size_t)m * k * 8));
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

}  // namespace
