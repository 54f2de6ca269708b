// api_a2.cuh -- a2 (E = K V^T, Eq. e) launches of kkm_api.cu: the materialised SpMMs (full K
// rows, f1 fp32 bands, f1 16-bit bands on the tensor cores), the streaming passes (full and upper
// triangle) and the 1.5D column-split reduce-scatter.
#pragma once

namespace {

template <int KP>
int launch_spmm_kp(kkm_ctx *h, const int32_t *labels, int c0) {
  const Plan &P = h->P;
  CK(ensure_smem_attr((const void *)spmm_onehot_kernel<KP>, spmm_smem_bytes<KP>()));
  const int64_t items = ceil_div(P.nA, SpRows<KP>::R) * P.nsplit;
  const int grid = (int)std::min<int64_t>(items, h->num_sms);
  spmm_onehot_kernel<KP><<<grid, SpRows<KP>::THREADS, spmm_smem_bytes<KP>(), h->st>>>(
      h->K, P.ldk, P.nA, labels, P.k, c0, P.nsplit, P.chunks_per_split, P.nApad, h->Spart);
  CKL();
  return KKM_OK;
}

// Sorts the points [b0, b0 + nB) of the handle's X by label (stable counting sort) and gathers
// their split operands, norms and scales in that order into o (rows [nB, rows) zeroed).
int sort_gather(kkm_ctx *h, const int32_t *labB, int64_t b0, int64_t nB, int64_t rows, const SortedSet &o) {
  const Plan &P = h->P;
  const int k = P.k;
  const int nblk = (int)ceil_div(std::max<int64_t>(nB, 1), SORT_BLOCK);
  sort_count_kernel<<<nblk, 256, (size_t)k * 4, h->st>>>(labB, nB, k, o.bcount);
  CKL();
  sort_scan_kernel<<<k + 1, 1024, 1024 * 4, h->st>>>(o.bcount, nblk, k, o.boff, o.seg);
  CKL();
  sort_scatter_kernel<<<nblk, 256, (size_t)9 * k * 4, h->st>>>(labB, nB, k, o.boff, o.perm, o.pos);
  CKL();
  gather_rows_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, h->st>>>(h->Xhi, h->Xlo, h->norms, h->rscale, o.perm, b0,
                                                                     nB, rows, P.dp, o.hi, o.lo, o.norms, o.rscale);
  CKL();
  return KKM_OK;
}

// The streaming kernel's A operand: rows [row0, row0 + nA) of a split operand with arows rows.
struct StreamA {
  const uint16_t *hi, *lo;
  const float *norms, *rscale;
  int64_t arows, row0, nA, rows_pad;
};

// One fused a1+a2 pass: S[rows_pad][k] (fp64) = the sums over the sorted set B (nB points, brows
// rows, k segments) of kappa(a_i, b_p) by cluster -- accumulated by tc3_stream_kernel in int64 fixed
// point (Sx, exact integer sums in any order, any k in one launch) and converted once. pos (NULL if
// A and B are disjoint): sorted position of A row i for b0 <= i < b0 + npos (the Gaussian
// diagonal). fx = 2^s with nB max|K| 2^s < 2^61.
int stream_pass(kkm_ctx *h, TcStream &ts, const StreamA &A, const SortedSet &B, int64_t brows, int64_t nB,
                int64_t b0, const int32_t *pos, int64_t npos, double fx, long long *Sx, double *S) {
  const Plan &P = h->P;
  const int k = P.k;
  if (A.nA == 0) return KKM_OK;
  CK(cudaMemsetAsync(Sx, 0, (size_t)A.rows_pad * k * 8, h->st));
  if (tc3_stream_launch(ts, A.hi, A.lo, B.hi, B.lo, P.fp16, A.arows, brows, P.dp, nB, b0, A.row0, A.nA, A.norms,
                        A.rscale, B.norms, B.rscale, pos, npos, B.seg, k, h->kp, fx, Sx, h->st, &h->launches,
                        h->chain_kb)) {
    h->poisoned = true;
    return fail(KKM_ECUDA, "streaming kernel launch failed: %s", tc_gemm_error());
  }
  fx_to_double_kernel<<<(unsigned)ceil_div(A.rows_pad * k, 256), 256, 0, h->st>>>(Sx, A.rows_pad * k, 1.0 / fx, S);
  CKL();
  return KKM_OK;
}

// Streaming a1+a2 of the clustering loop: sort the B set by label, then the fused kernel writes
// the S partials (Spart) of the A set's rows.
int launch_stream(kkm_ctx *h, const int32_t *labels) {
  const Plan &P = h->P;
  const SortedSet B{h->Shi, h->Slo, h->snorms, h->srscale, h->perm, h->pos, h->seg, h->bcount, h->boff};
  CKR(sort_gather(h, labels + P.b0, P.b0, P.nB, P.npad, B));
  const StreamA A{h->Xhi, h->Xlo, h->norms, h->rscale, P.npad, P.a0, P.nA, P.nApad};
  a2_mark(h);
  const int rc = stream_pass(h, h->ts, A, B, P.npad, P.nB, P.b0, h->pos, P.nB, h->fx_scale,
                            (long long *)(h->ws + P.o_Sx), h->Spart);
  a2_mark(h);
  return rc;
}

// a2 on the materialised K tile (A set rows x B set columns).
int launch_spmm_mat_body(kkm_ctx *h, const int32_t *labels);
int launch_spmm_mat(kkm_ctx *h, const int32_t *labels) {
  a2_mark(h);
  const int rc = launch_spmm_mat_body(h, labels);
  a2_mark(h);
  return rc;
}

int launch_spmm_mat_body(kkm_ctx *h, const int32_t *labels) {
  const Plan &P = h->P;
  if (P.nA == 0) return KKM_OK;
  if (P.spmm_v2) {
    const int64_t ngroups = P.ldk / 32;
    group_code_kernel<<<(unsigned)ceil_div(ngroups, 8), 256, 0, h->st>>>(labels + P.b0, P.nB, P.ldk, h->codes);
    CKL();
    CK(ensure_smem_attr((const void *)spmm_group_kernel, sg_smem_bytes(SG_MAX_K)));
    const int64_t items = ceil_div(P.nA, SG_ROWS) * P.nsplit;
    const int grid = (int)std::min<int64_t>(items, h->num_sms);
    spmm_group_kernel<<<grid, SG_THREADS, sg_smem_bytes(P.k), h->st>>>(h->K, P.ldk, P.nA, h->codes, P.k, P.nsplit,
                                                                     P.chunks_per_split, P.nApad, h->Spart);
    CKL();
    return KKM_OK;
  }
  if (P.pr > 1) {  // the B set's labels, -1 padded to the tile pitch
    copy_labels_kernel<<<(unsigned)ceil_div(P.ldk, 256), 256, 0, h->st>>>(labels + P.b0, P.nB, P.ldk, h->labB);
    CKL();
    labels = h->labB;
  }
  if (P.k > SP_KPMAX) {
    for (int c0 = 0; c0 < P.k; c0 += SP_KPMAX) CKR(launch_spmm_kp<SP_KPMAX>(h, labels, c0));
    return KKM_OK;
  }
  const int kp = (P.k + 1) / 2 * 2;
  switch (kp) {
    case 2: return launch_spmm_kp<2>(h, labels, 0);
    case 4: return launch_spmm_kp<4>(h, labels, 0);
    case 6: return launch_spmm_kp<6>(h, labels, 0);
    case 8: return launch_spmm_kp<8>(h, labels, 0);
    case 10: return launch_spmm_kp<10>(h, labels, 0);
    case 12: return launch_spmm_kp<12>(h, labels, 0);
    case 14: return launch_spmm_kp<14>(h, labels, 0);
    default: return launch_spmm_kp<16>(h, labels, 0);
  }
}

template <int KP>
int launch_spmm_sym_kp(kkm_ctx *h, const int32_t *labels) {
  const Plan &P = h->P;
  CK(ensure_smem_attr((const void *)spmm_sym_kernel<KP>, spmm_sym_smem_bytes()));
  if (P.sym_items == 0) {
    a2_mark(h);
    a2_mark(h);
    return KKM_OK;
  }
  const int grid = (int)std::min<int64_t>(P.sym_items, h->num_sms);
  a2_mark(h);
  spmm_sym_kernel<KP><<<grid, SYM_THREADS, spmm_sym_smem_bytes(), h->st>>>(
      h->K, h->bands, (int)P.bands.size(), P.sym_items, labels, h->perm_b, h->groups, P.sym_gmax, P.k, P.nApad,
      h->Spart, h->colpart, h->work);
  a2_mark(h);
  CKL();
  return KKM_OK;
}

// f1: a2 over the symmetric band storage -> the rank's contributions to S of all rows (Sfin),
// reduce-scattered over the ranks for P > 1 (each rank then holds S of its own 1D block).
int launch_spmm_sym(kkm_ctx *h, const int32_t *labels, const double **s_out) {
  const Plan &P = h->P;
  const int k = P.k;
  if (P.kh) {  // f4: 16-bit bands, a2 on the tensor cores (spmm_tc.cuh), S in int64 fixed point
    const bool nl32 = P.tnl == 32;
    if (nl32) CK(ensure_smem_attr((const void *)spmm_tc_kernel<32>, TsCfg<32>::SMEM));
    else CK(ensure_smem_attr((const void *)spmm_tc_kernel<16>, TsCfg<16>::SMEM));
    long long *Sx = h->tSfix;
    if (h->lsa) {  // alternate parities of the symmetric window: a peer may still read the
      h->ls_par ^= 1;     // other one (its reads end before it reaches the next cross-rank barrier)
      Sx = (long long *)(h->lsbuf + (size_t)h->ls_par * h->ls_sb);
      h->tSfix = Sx;
    }
    CK(cudaMemsetAsync(Sx, 0, (size_t)P.npad * k * 8, h->st));
    a2_mark(h);
    if (!P.tunits.empty()) {
      const int grid = (int)std::min<int64_t>((int64_t)P.tunits.size(), h->num_sms);
      float *cpart = nl32 ? (float *)(h->ws + P.o_tcolpart) : nullptr;
      if (nl32)
        spmm_tc_kernel<32><<<grid, TS_THREADS, TsCfg<32>::SMEM, h->st>>>(
            h->tmaps, h->tbands, h->tunits, (int)P.tunits.size(), labels, P.n, k, P.npad, h->tfxm, Sx, h->work,
            P.kplanes, cpart);
      else
        spmm_tc_kernel<16><<<grid, TS_THREADS, TsCfg<16>::SMEM, h->st>>>(
            h->tmaps, h->tbands, h->tunits, (int)P.tunits.size(), labels, P.n, k, P.npad, h->tfxm, Sx, h->work,
            P.kplanes, cpart);
      CKL();
      if (nl32 && !P.tslabs.empty()) {  // the column parts, summed over this rank's slabs
        ts_colpart_reduce_kernel<<<dim3((unsigned)ceil_div(P.n, 4 * 256), (unsigned)k), 256, 0, h->st>>>(
            cpart, (const TsSlab *)(h->ws + P.o_tslabs), (int)P.tslabs.size(), P.n, k, P.npad, h->tfxm, Sx);
        CKL();
      }
    }
    a2_mark(h);
    if (h->lsa && h->ls_fused_next) {  // update_grid_kernel<true> sums the ranks' S itself
      *s_out = nullptr;
      return KKM_OK;
    }
    const unsigned gr = (unsigned)ceil_div(P.npad * k, 256);
    if (P.repl)  // S of all points on every rank (exact int64 sum)
      CKN(ncclAllReduce(h->tSfix, h->tSfix, (size_t)P.npad * k, ncclInt64, ncclSum, h->comm, h->st));
    if (P.a3fix) {  // run_cnorm's finalize reads tSfix directly
      *s_out = nullptr;
      return KKM_OK;
    }
    if (P.nranks == 1 || P.repl) {
      ts_fix_out_kernel<<<gr, 256, 0, h->st>>>(h->tSfix, P.n, P.npad, k, h->tfx_inv, nullptr, h->Sfin);
      CKL();
      *s_out = h->Sfin;
      return KKM_OK;
    }
    // exact: the int64 sums of the ranks' contributions, any order gives the same bits
    ts_fix_out_kernel<<<gr, 256, 0, h->st>>>(h->tSfix, P.n, P.npad, k, 1.0, h->tSint, nullptr);
    CKL();
    CKN(ncclReduceScatter(h->tSint, h->tSmine, (size_t)P.B * k, ncclInt64, ncclSum, h->comm, h->st));
    fx_to_double_kernel<<<(unsigned)ceil_div(P.B * k, 256), 256, 0, h->st>>>(h->tSmine, P.B * k, h->tfx_inv,
                                                                           h->Smine);
    *s_out = h->Smine;
    return KKM_OK;
  }
  band_sort_kernel<<<P.T, SYM_TB, (size_t)(32 * k + 2 * (k + 1)) * 4, h->st>>>(
      labels, P.n, k, sym_rows(k), P.sym_gmax, h->perm_b, h->groups, h->ngroups, h->gfirst);
  CKL();
  int rc;
  switch ((k + 1) / 2 * 2) {
    case 2: rc = launch_spmm_sym_kp<2>(h, labels); break;
    case 4: rc = launch_spmm_sym_kp<4>(h, labels); break;
    case 6: rc = launch_spmm_sym_kp<6>(h, labels); break;
    case 8: rc = launch_spmm_sym_kp<8>(h, labels); break;
    case 10: rc = launch_spmm_sym_kp<10>(h, labels); break;
    case 12: rc = launch_spmm_sym_kp<12>(h, labels); break;
    case 14: rc = launch_spmm_sym_kp<14>(h, labels); break;
    default: rc = launch_spmm_sym_kp<16>(h, labels); break;
  }
  CKR(rc);
  int64_t wmax = 0;
  for (const SymBand &b : P.bands) wmax = std::max<int64_t>(wmax, b.ldb - SYM_TB);
  if (wmax > 0 && !P.bands.empty()) {
    sym_colsum_kernel<<<dim3((unsigned)ceil_div(wmax, 4 * 128), (unsigned)P.bands.size(), (unsigned)k), 128, 0,
                        h->st>>>(
        h->colpart, h->bands, h->gfirst, k, h->colsum);
    CKL();
  }
  sym_reduce_kernel<<<dim3((unsigned)ceil_div(P.npad, 256), (unsigned)k), 256, 0, h->st>>>(
      h->Spart, h->colsum, h->bands, h->band_desc, P.n, P.npad, k, h->Sfin);
  CKL();
  if (P.repl) CKN(ncclAllReduce(h->Sfin, h->Sfin, (size_t)P.npad * k, ncclDouble, ncclSum, h->comm, h->st));
  if (P.nranks == 1 || P.repl) {
    *s_out = h->Sfin;
    return KKM_OK;
  }
  CKN(ncclReduceScatter(h->Sfin, h->Smine, (size_t)P.B * k, ncclDouble, ncclSum, h->comm, h->st));
  *s_out = h->Smine;
  return KKM_OK;
}

// f1 streaming a1+a2: sort all points by label, the upper-triangle kernel accumulates S of
// the sorted points in int64 fixed point; back to original order (exact), reduce-scattered
// in int64 for P > 1 (exact: any reduction order gives the same bits), then fp64.
int launch_stream_sym(kkm_ctx *h, const int32_t *labels, const double **s_out) {
  const Plan &P = h->P;
  const int k = P.k;
  const SortedSet B{h->Shi, h->Slo, h->snorms, h->srscale, h->perm, h->pos, h->seg, h->bcount, h->boff};
  CKR(sort_gather(h, labels, 0, P.n, P.npad, B));
  CK(cudaMemsetAsync(h->Sfix, 0, (size_t)P.npad * k * 8, h->st));
  a2_mark(h);
  int rc = ssym_launch(h->ts, h->Shi, h->Slo, P.fp16, P.npad, P.dp, P.n, h->snorms, h->srscale, h->seg, k, h->kp,
                       h->units, (int64_t)P.units.size(), h->work + 2, h->fx_scale, h->Sfix, h->st, &h->launches, h->chain_kb);
  a2_mark(h);
  if (rc) {
    h->poisoned = true;
    return fail(KKM_ECUDA, "symmetric streaming kernel launch failed: %s", tc_gemm_error());
  }
  const unsigned g = (unsigned)ceil_div(P.npad * k, 256);
  double *Sd = h->Spart;  // P.nsplit = 1: [npad][k] fp64
  if (P.repl)  // the sorted order is the same on every rank (same labels, stable sort): sum in place
    CKN(ncclAllReduce(h->Sfix, h->Sfix, (size_t)P.npad * k, ncclInt64, ncclSum, h->comm, h->st));
  if (P.nranks == 1 || P.repl) {
    fx_unpermute_kernel<<<g, 256, 0, h->st>>>(h->Sfix, h->pos, P.n, P.npad, k, h->fx_inv, nullptr, Sd);
    CKL();
    *s_out = Sd;
    return KKM_OK;
  }
  fx_unpermute_kernel<<<g, 256, 0, h->st>>>(h->Sfix, h->pos, P.n, P.npad, k, h->fx_inv, h->Sorig, nullptr);
  CKL();
  CKN(ncclReduceScatter(h->Sorig, h->Sfmine, (size_t)P.B * k, ncclInt64, ncclSum, h->comm, h->st));
  fx_to_double_kernel<<<(unsigned)ceil_div(P.B * k, 256), 256, 0, h->st>>>(h->Sfmine, P.B * k, h->fx_inv, h->Smine);
  CKL();
  *s_out = h->Smine;
  return KKM_OK;
}

// The 1.5D column-split reduce-scatter over the pr ranks of process column j,
// as point-to-point exchanges on the world communicator (no split communicator: its creation cost
// ~3 s of init and a first-use spike): rank (i, j) sends piece i' of its Scol to rank (i', j), receives
// piece i from every other rank of the column, and sums the pr pieces in rank order (fixed order,
// so the result is bitwise the same on every run). Collective over the column.
int column_reduce_scatter(kkm_ctx *h) {
  const Plan &P = h->P;
  const size_t bk = (size_t)P.B * P.k;
  double *rbuf = (double *)(h->ws + P.o_Srecv);
  CKN(ncclGroupStart());
  for (int ip = 0; ip < P.pr; ++ip) {
    if (ip == P.gi) continue;
    const int peer = ip + P.gj * P.pr;
    CKN(ncclSend(h->Scol + ip * bk, bk, ncclDouble, peer, h->comm, h->st));
    CKN(ncclRecv(rbuf + ip * bk, bk, ncclDouble, peer, h->comm, h->st));
  }
  CKN(ncclGroupEnd());
  column_sum_kernel<<<(unsigned)ceil_div((int64_t)bk, 256), 256, 0, h->st>>>(h->Scol, rbuf, P.pr, P.gi, (int64_t)bk,
                                                                           h->Smine);
  CKL();
  return KKM_OK;
}

// a2 + the 1.5D column-split reduce-scatter: afterwards the S partials of this rank's own 1D
// block are in s_out[nsplit_out][B][k] (the 1D case reduces nothing: s_out = Spart).
int launch_spmm(kkm_ctx *h, const int32_t *labels, const double **s_out, int *nsplit_out) {
  const Plan &P = h->P;
  if (P.sym) {
    *nsplit_out = 1;
    return launch_spmm_sym(h, labels, s_out);
  }
  if (P.ssym) {
    *nsplit_out = 1;
    return launch_stream_sym(h, labels, s_out);
  }
  CKR(P.materialize ? launch_spmm_mat(h, labels) : launch_stream(h, labels));
  if (P.pr == 1) {
    *s_out = h->Spart;
    *nsplit_out = P.nsplit;
    return KKM_OK;
  }
  split_sum_kernel<<<(unsigned)ceil_div(P.nApad * P.k, 256), 256, 0, h->st>>>(h->Spart, P.nsplit, P.nA,
                                                                              P.nApad, P.k, h->Scol);
  CKL();
  // P(i, j) keeps piece i of column block j = its own 1D block (column-major ranks)
  CKR(column_reduce_scatter(h));
  *s_out = h->Smine;
  *nsplit_out = 1;
  return KKM_OK;
}

}  // namespace
