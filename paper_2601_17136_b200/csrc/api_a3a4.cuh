// api_a3a4.cuh -- a3 (z, c, J: Eqs. z, c P:134-158) and a4 (D, argmin, sizes: Eq. d)
// launches of kkm_api.cu with their exchange steps, the a1 GEMM launcher and the f3 delta update.
#pragma once

namespace {

// a3: E, z, c (cnorm) and J for the labels entering the iteration -> E_out, cnorm_out,
// J_out. sizes_next / changed_out (may be NULL) are zeroed for the following assign.
int run_cnorm(kkm_ctx *h, const double *S, int nsplit, int64_t rows_pad, double *E_out, double *cnorm_out,
              double *J_out, int32_t *sizes_next, unsigned long long *changed_out) {
  const Plan &P = h->P;
  const int32_t *labels = h->lab[h->cur];
  const int32_t *sizes = h->sizes[h->cur];
  const int k1 = P.k + 1;
  const int nr = P.repl ? 1 : P.nranks, r = P.repl ? 0 : P.rank;  // replicated a3: one "rank"
  if (P.a3fix && P.a_n > 0) {  // int64 S in, c and J from the last block (same sums as below)
    const int fth = fin_threads(P.k);
    finalize_kernel<<<P.nfin, fth, (size_t)k1 * fth * 8, h->st>>>(
        nullptr, 1, P.a_n, P.npad, P.k, sizes, labels + P.a_row0, h->diag, P.rows_per_block, E_out, h->blockpart,
        h->tSfix, h->tfx_inv, A3Fused{h->a3ctr, sizes, cnorm_out, J_out, sizes_next, changed_out});
    CKL();
    return KKM_OK;
  }
  if (P.a_n > 0) {
    const int fth = fin_threads(P.k);
    finalize_kernel<<<P.nfin, fth, (size_t)k1 * fth * 8, h->st>>>(
        S, nsplit, P.a_n, rows_pad, P.k, sizes, labels + P.a_row0, h->diag, P.rows_per_block,
        E_out, h->blockpart);
    CKL();
  }
  cnorm_local_kernel<<<1, 32 * std::min(32, k1), 0, h->st>>>(h->blockpart, P.a_n > 0 ? P.nfin : 0, P.k,
                                           h->rankpart + (int64_t)r * k1);
  CKL();
  if (nr > 1)
    CKN(ncclAllGather(h->rankpart + (int64_t)r * k1, h->rankpart, k1, ncclDouble, h->comm, h->st));
  cnorm_final_kernel<<<1, 128, 0, h->st>>>(h->rankpart, nr, P.k, sizes, cnorm_out, J_out,
                                           sizes_next, changed_out);
  CKL();
  return KKM_OK;
}

// a3 + a4 in one cooperative launch (update_grid_kernel): the int64 S of the one-rank / replicated
// f1 paths, k <= UG_MAX_K, no peer exchange. New labels into lab[cur^1], sizes into sizes[cur^1].
// With the NVLink peer-memory window (h->lsa, in the fit loop) the launch is the distributed
// variant: own rows only, S summed over the ranks while read, labels / sizes / changed stored into
// every rank's copies, three cross-rank arrivals.
bool use_update_grid(const kkm_ctx *h) { return h->ug_grid > 0; }
int run_update_grid(kkm_ctx *h, double *J_out, unsigned long long *changed_out) {
  const Plan &P = h->P;
  const int nx = h->cur ^ 1;
  const long long *Sfix = h->tSfix;
  int64_t rows_pad = P.npad, nrows = P.a_n;
  int k = P.k;
  double inv = h->tfx_inv;
  const int32_t *sizes = h->sizes[h->cur], *cl = h->lab[h->cur] + P.a_row0;
  const double *diag = h->diag;
  double *E = h->E, *bp = h->blockpart, *cn = h->cnorm;
  unsigned *bar = h->a3ctr;
  int32_t *cl_new = h->lab[nx] + P.a_row0, *sz_next = h->sizes[nx];
  const bool lsa = h->lsa && h->ls_fused_next;
  LsaArgs L = h->lsargs;
  if (lsa) {
    nrows = P.nloc;
    L.row0 = P.row0;
    L.off_S = (size_t)h->ls_par * h->ls_sb;
    L.off_lab_next = h->ls_off_lab + (size_t)nx * h->ls_lb;
    L.off_sizes_next = h->ls_off_sizes + (size_t)nx * 4096;
    L.off_changed = (size_t)((uint8_t *)changed_out - h->lsbuf);
    L.target = (h->ls_epoch + 1) * (unsigned)P.nranks;
    L.Sred = (long long *)(h->ws + P.o_tSfix);  // (the workspace S is free: S lives in the window)
    h->ls_epoch += 3;
  }
  void *args[] = {&Sfix, &rows_pad, &nrows, &k, &inv, &sizes, &cl, &diag, &E, &bp, &bar, &cn, &J_out, &cl_new,
                  &sz_next, &changed_out, &L};
  // (the distributed variant takes every co-resident block: its phase 0 is a latency-bound
  // NVLink read of P copies, more threads = more loads in flight)
  const int64_t need = lsa ? (int64_t)h->ug_grid : std::max<int64_t>(1, ceil_div(nrows, UG_THREADS));
  const unsigned grid = (unsigned)std::min<int64_t>({need, (int64_t)h->ug_grid, (int64_t)P.nfin});
  if (lsa) CK(cudaLaunchCooperativeKernel((const void *)update_grid_kernel<true>, grid, UG_THREADS, args, 0, h->st));
  else CK(cudaLaunchCooperativeKernel((const void *)update_grid_kernel<false>, grid, UG_THREADS, args, 0, h->st));
  return KKM_OK;
}

// a4 + the V update: new labels into lab[cur^1], sizes into sizes[cur^1], allgather.
int run_assign(kkm_ctx *h, unsigned long long *changed_out) {
  const Plan &P = h->P;
  const int nx = h->cur ^ 1;
  if (P.a_n > 0) {
    const int th = 256;
    assign_kernel<<<(unsigned)ceil_div(P.a_n, th), th, (size_t)P.k * 4, h->st>>>(
        h->E, P.a_n, P.k, h->cnorm, h->diag, h->lab[h->cur] + P.a_row0, h->lab[nx] + P.a_row0,
        h->sizes[nx], changed_out, nullptr);  // (Dfull: formed on demand by kkm_debug_read)
    CKL();
  }
  if (P.nranks > 1 && !P.repl) {  // the changed count is global too: every rank takes the same control path
    CKN(ncclGroupStart());
    CKN(ncclAllGather(h->lab[nx] + P.row0, h->lab[nx], P.B, ncclInt32, h->comm, h->st));
    CKN(ncclAllReduce(h->sizes[nx], h->sizes[nx], P.k, ncclInt32, ncclSum, h->comm, h->st));
    CKN(ncclAllReduce(changed_out, changed_out, 1, ncclUint64, ncclSum, h->comm, h->st));
    CKN(ncclGroupEnd());
  }
  return KKM_OK;
}

// oscale > 0: out is fp16 and receives K * oscale (tensor-core precisions only)
int launch_gemm(kkm_ctx *h, int64_t i0, int64_t m, int64_t j0, int64_t ncov, void *out, int64_t ldo,
                float oscale = 0.f, void *out_lo = nullptr) {
  const Plan &P = h->P;
  if (m <= 0 || ncov <= 0) return KKM_OK;
  if (P.tc) {
    int rc = tc3_gemm_launch(h->tc, h->Xhi, h->Xlo, P.fp16, h->rscale, P.npad, P.dp, P.n, i0, m, j0, ncov, h->norms,
                             h->kp, out, ldo, h->st, &h->launches, oscale, out_lo, h->chain_kb);
    if (rc) {
      h->poisoned = true;
      return fail(KKM_ECUDA, "tcgen05 GEMM launch failed: %s", tc_gemm_error());
    }
    return KKM_OK;
  }
  dim3 grid((unsigned)ceil_div(ncov, SG_BN), (unsigned)ceil_div(m, SG_BM));
  gemm_simt_kernel<<<grid, 256, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, i0, m, j0, ncov, h->norms,
                                             h->kp, (float *)out, ldo);
  CKL();
  return KKM_OK;
}

// f3: S of the own rows for the labels lab[cur ^ 1] from S (Sinc) of lab[cur]: the points
// that moved, sorted by new label, added; sorted by old label, subtracted (the fused
// streaming kernel, A = own rows, B = the moved points). m = number of moved points.
int delta_update(kkm_ctx *h, int64_t m) {
  const Plan &P = h->P;
  const int k = P.k;
  const int32_t *cl_old = h->lab[h->cur], *cl_new = h->lab[h->cur ^ 1];
  const int nblk = (int)ceil_div(P.n, SORT_BLOCK);
  const int64_t mpad = round_up(m, 256);
  const StreamA A{h->Xhi, h->Xlo, h->norms, h->rscale, P.npad, P.row0, P.nloc, P.B};
  for (int pass = 0; pass < 2; ++pass) {  // 0: + new labels, 1: - old labels
    moved_key_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(cl_old, cl_new, P.n, P.lablen, k,
                                                                           pass == 0, h->dkey);
    CKL();
    const SortedSet &D = h->dset;
    sort_count_kernel<<<nblk, 256, (size_t)(k + 1) * 4, h->st>>>(h->dkey, P.n, k + 1, D.bcount);
    CKL();
    sort_scan_kernel<<<k + 2, 1024, 1024 * 4, h->st>>>(D.bcount, nblk, k + 1, D.boff, D.seg);
    CKL();
    sort_scatter_kernel<<<nblk, 256, (size_t)9 * (k + 1) * 4, h->st>>>(h->dkey, P.n, k + 1, D.boff, D.perm, D.pos);
    CKL();
    gather_rows_kernel<<<(unsigned)ceil_div(mpad, 8), 256, 0, h->st>>>(h->Xhi, h->Xlo, h->norms, h->rscale, D.perm, 0,
                                                                       m, mpad, P.dp, D.hi, D.lo, D.norms, D.rscale);
    CKL();
    // B = the m moved points (clusters 0..k-1 of the k+1 buckets); pos: sorted position of
    // each point (>= m for the points that did not move) for the Gaussian diagonal
    CKR(stream_pass(h, h->ts_delta, A, D, mpad, m, 0, D.pos, P.n, h->fx_scale, h->Sdx, h->Sd));
    sinc_add_kernel<<<(unsigned)ceil_div(P.nloc * k, 256), 256, 0, h->st>>>(h->Sd, 1, P.B, P.nloc, k,
                                                                            pass == 0 ? 1.0 : -1.0, h->Sinc);
    CKL();
  }
  return KKM_OK;
}

struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace
