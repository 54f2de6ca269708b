// kkm_api.cu -- the C-ABI of include/kkm.h: handle, workspace planner, one-time setup,
// the clustering loop of Alg. 1 over the kernels in *.cuh, the NCCL
// exchange steps of the 1D algorithm, and the test hooks.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>

#include "kkm.h"
#include "common.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "kpp.cuh"
#include "prep.cuh"
#include "sort.cuh"
#include "spmm.cuh"
#include "stream.cuh"
#include "spmm_tc.cuh"
#include "sym.cuh"
#include "tc2.cuh"
#include "ssym.cuh"
#include "tc3.cuh"
#include "update.cuh"

using namespace kkm;

#include "api_plan.cuh"
#include "api_ctx.cuh"
#include "api_a2.cuh"
#include "api_a3a4.cuh"
#include "api_exchange.cuh"
#include "api_predict.cuh"

extern "C" {

int kkm_default_params(kkm_params *p) {
  if (!p) return fail(KKM_EINVAL, "params is NULL");
  std::memset(p, 0, sizeof(*p));
  p->kind = KKM_KERNEL_POLY;
  p->gamma = 1.0;
  p->coef0 = 1.0;
  p->degree = 2;
  p->k = 2;
  p->max_iter = 100;
  p->path = KKM_PATH_AUTO;
  p->precision = KKM_PREC_FP16X3;
  return KKM_OK;
}

int64_t kkm_shard_begin(int64_t n, int32_t rank, int32_t nranks) {
  if (nranks < 1 || n < 0 || rank < 0) return -1;
  const int64_t B = ceil_div(n, nranks);
  return std::min<int64_t>(n, (int64_t)rank * B);
}

int kkm_workspace_size(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks,
                       size_t *bytes) {
  if (!bytes) return fail(KKM_EINVAL, "bytes is NULL");
  Plan P;
  CKR(make_plan(p, n, d, rank, nranks, &P));
  *bytes = P.total;
  return KKM_OK;
}

int kkm_plan_query(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks, kkm_plan_info *info,
                   int64_t *pieces, int64_t cap) {
  if (!info) return fail(KKM_EINVAL, "info is NULL");
  Plan P;
  CKR(make_plan(p, n, d, rank, nranks, &P));
  std::memset(info, 0, sizeof(*info));
  info->path = P.materialize ? KKM_PATH_MATERIALIZE : KKM_PATH_STREAM;
  info->layout = P.sym ? (P.kh ? KKM_LAYOUT_SYM_BANDS16 : KKM_LAYOUT_SYM_BANDS)
                 : P.ssym ? KKM_LAYOUT_SYM_STREAM : P.materialize ? KKM_LAYOUT_FULL : KKM_LAYOUT_STREAM;
  info->exchange = nranks == 1 ? KKM_XCHG_NONE
                   : P.repl ? KKM_XCHG_S_ALLREDUCE
                   : (P.sym || P.ssym) ? KKM_XCHG_S_REDUCE_SCATTER : KKM_XCHG_PARTIALS;
  info->grid_rows = P.pr;
  info->grid_cols = P.pc;
  info->row0 = P.row0;
  info->nloc = P.nloc;
  info->a0 = P.a0;
  info->nA = P.nA;
  info->b0 = P.b0;
  info->nB = P.nB;
  info->ws_bytes = (int64_t)P.total;
  std::vector<int64_t> r;
  auto add = [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc, int64_t cd) {
    nr = std::min(nr, n - r0);
    nc = std::min(nc, n - c0);
    if (nr <= 0 || nc <= 0) return;
    r.insert(r.end(), {r0, nr, c0, nc, std::min(cd, n)});
  };
  if (P.sym) {
    for (const SymBand &b : P.bands) {
      const int64_t j0 = (int64_t)b.band * SYM_TB;
      add(j0 + b.row0, b.rows, j0, n - j0, j0 + SYM_TB);
    }
  } else if (P.ssym) {
    for (const int4 &u : P.units) add((int64_t)u.x * 256, 256, (int64_t)u.y * 256, (int64_t)u.z * 256,
                                      u.x == u.y ? (int64_t)(u.y + 1) * 256 : (int64_t)u.y * 256);
  } else {
    add(P.a0, P.nA, P.b0, P.nB, n);
  }
  info->npieces = (int64_t)(r.size() / 5);
  if (pieces)
    std::memcpy(pieces, r.data(), (size_t)std::min<int64_t>(cap, info->npieces) * 5 * sizeof(int64_t));
  return KKM_OK;
}

const char *kkm_last_error(void) { return g_err; }

int kkm_init(kkm_handle *out, const kkm_params *p, const float *X_local, int64_t n, int64_t d,
             int64_t ldx, int32_t rank, int32_t nranks, const int32_t *init_labels, void *workspace,
             size_t ws_bytes, void *cuda_stream, void *nccl_comm) {
  if (!out) return fail(KKM_EINVAL, "out is NULL");
  *out = nullptr;
  Plan P;
  CKR(make_plan(p, n, d, rank, nranks, &P));
  if (ldx < d) return fail(KKM_EINVAL, "ldx=%lld < d=%lld", (long long)ldx, (long long)d);
  if (!X_local && P.nloc > 0) return fail(KKM_EINVAL, "X_local is NULL");
  if (!workspace) return fail(KKM_EINVAL, "workspace is NULL");
  if (((uintptr_t)workspace) & 255) return fail(KKM_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < P.total)
    return fail(KKM_ENOMEM, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  if (nranks > 1 && !nccl_comm) return fail(KKM_EINVAL, "nranks > 1 needs an NCCL communicator");

  kkm_ctx *h = new kkm_ctx();
  h->p = *p;
  h->P = P;
  h->st = (cudaStream_t)cuda_stream;
  h->comm = (ncclComm_t)nccl_comm;
  h->ws = (uint8_t *)workspace;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    delete h;
    return fail(KKM_ECUDA, "no CUDA device");
  }
  uint8_t *w = h->ws;
  h->Xf = (float *)(w + P.o_Xf);
  h->mean = (float *)(w + P.o_mean);
  h->Xhi = P.tc ? (uint16_t *)(w + P.o_Xhi) : nullptr;
  h->Xlo = P.tc ? (uint16_t *)(w + P.o_Xlo) : nullptr;
  h->rscale = (float *)(w + P.o_rscale);
  h->norms = (float *)(w + P.o_norms);
  h->diag = (double *)(w + P.o_diag);
  h->K = P.materialize ? (float *)(w + P.o_K) : nullptr;
  for (int b = 0; b < 2; ++b) {
    h->lab[b] = (int32_t *)(w + P.o_lab[b]);
    h->sizes[b] = (int32_t *)(w + P.o_sizes[b]);
  }
  h->Spart = (double *)(w + P.o_Spart);
  h->E = (double *)(w + P.o_E);
  h->a3ctr = (unsigned *)(w + P.o_a3ctr);
  h->blockpart = (double *)(w + P.o_blockpart);
  h->rankpart = (double *)(w + P.o_rankpart);
  h->cnorm = (double *)(w + P.o_cnorm);
  h->J = (double *)(w + P.o_J);
  h->changed = (unsigned long long *)(w + P.o_changed);
  h->Dfull = (double *)(w + P.o_Dfull);
  h->bad = (int *)(w + P.o_bad);
  h->E2 = (double *)(w + P.o_E2);
  h->cnorm2 = (double *)(w + P.o_cnorm2);
  if (!P.materialize) {
    h->Shi = (uint16_t *)(w + P.o_Shi);
    h->Slo = (uint16_t *)(w + P.o_Slo);
    h->snorms = (float *)(w + P.o_snorms);
    h->srscale = (float *)(w + P.o_srscale);
    h->perm = (int32_t *)(w + P.o_perm);
    h->pos = (int32_t *)(w + P.o_pos);
    h->seg = (int32_t *)(w + P.o_seg);
    h->bcount = (int32_t *)(w + P.o_bcount);
    h->boff = (int32_t *)(w + P.o_boff);
  }
  h->fxmax = (float *)(w + P.o_fxmax);
  if (P.materialize && P.spmm_v2) h->codes = (uint32_t *)(w + P.o_codes);
  if (P.pr > 1) {
    h->labB = (int32_t *)(w + P.o_labB);
    h->Scol = (double *)(w + P.o_Scol);
  }
  if (P.need_smine) h->Smine = (double *)(w + P.o_Smine);
  if (P.inc) {
    h->Sinc = (double *)(w + P.o_Sinc);
    h->Sd = (double *)(w + P.o_Sd);
    h->Sdx = (long long *)(w + P.o_Sdx);
    h->dkey = (int32_t *)(w + P.o_dkey);
    h->dset = SortedSet{(uint16_t *)(w + P.o_Dhi), (uint16_t *)(w + P.o_Dlo), (float *)(w + P.o_Dn),
                        (float *)(w + P.o_Dr),      (int32_t *)(w + P.o_dperm), (int32_t *)(w + P.o_dpos),
                        (int32_t *)(w + P.o_dseg),  (int32_t *)(w + P.o_dbc),   (int32_t *)(w + P.o_dbo)};
  }
  if (P.ssym || P.sym) h->work = (int32_t *)(w + P.o_work);
  if (P.ssym) {
    h->units = (int4 *)(w + P.o_units);
    h->Sfix = (long long *)(w + P.o_Sfix);
    if (P.nranks > 1) {
      h->Sorig = (long long *)(w + P.o_Sorig);
      h->Sfmine = (long long *)(w + P.o_Sfmine);
    }
  }
  if (P.sym) {
    h->perm_b = (int32_t *)(w + P.o_perm_b);
    h->groups = (SymGroup *)(w + P.o_groups);
    h->ngroups = (int32_t *)(w + P.o_ngroups);
    h->bands = (SymBand *)(w + P.o_bands);
    h->band_desc = (int32_t *)(w + P.o_band_desc);
    h->colpart = (float *)(w + P.o_colpart);
    h->colsum = (double *)(w + P.o_colsum);
    if (P.kh) {
      h->tmaps = (CUtensorMap *)(w + P.o_tmaps);
      h->tbands = (TsBand *)(w + P.o_tbands);
      h->tunits = (TsUnit *)(w + P.o_tunits);
      h->tSfix = (long long *)(w + P.o_tSfix);
      if (P.nranks > 1) {
        h->tSint = (long long *)(w + P.o_tSint);
        h->tSmine = (long long *)(w + P.o_tSmine);
      }
    }
    h->gfirst = (int32_t *)(w + P.o_gfirst);
    h->Sfin = (double *)(w + P.o_Sfin);
  }
  if (const char *e = std::getenv("KKM_CHAIN_KB")) h->chain_kb = std::max(0, std::atoi(e));
  h->kp.kind = p->kind;
  h->kp.degree = p->degree;
  h->kp.gamma = (float)p->gamma;
  h->kp.coef0 = (float)p->coef0;
  h->kp.neg_gamma_log2e = (float)(-p->gamma * 1.4426950408889634);

  int rc = [&]() -> int {
    if (P.fused) CK(ensure_smem_attr((const void *)fused_update_kernel, 17 * FUSED_THREADS * 8 + 16 * 8));
    if (fin_smem_bytes(P.k) > 48 * 1024) CK(ensure_smem_attr((const void *)finalize_kernel, fin_smem_bytes(P.k)));
    EventList evs;  // init phases: prep, GEMM
    if (!evs.record(h->st)) return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    // ---- X (Alg. 1 line 1: allgather P) into Xf [npad x ldf], zero padded
    CK(cudaMemsetAsync(h->Xf, 0, (size_t)P.npad * P.ldf * 4, h->st));
    if (P.nloc > 0)
      CK(cudaMemcpy2DAsync(h->Xf + P.row0 * P.ldf, P.ldf * 4, X_local, ldx * 4, P.d * 4, P.nloc,
                           cudaMemcpyDefault, h->st));
    if (P.nranks > 1)
      CKN(ncclAllGather(h->Xf + (int64_t)P.rank * P.B * P.ldf, h->Xf, (size_t)P.B * P.ldf, ncclFloat,
                        h->comm, h->st));
    // ---- Gaussian: center X on its column means (exact for kappa; smaller norms shrink the
    // accumulation bias of r^2 on the tensor cores, DESIGN A9). Every rank holds all of X.
    CK(cudaMemsetAsync(h->mean, 0, (size_t)P.ldf * 4, h->st));
    if (p->kind == KKM_KERNEL_GAUSSIAN) {
      const unsigned nch = (unsigned)ceil_div(P.n, CM_ROWS);
      double *part = (double *)(h->ws + P.o_cmpart);
      colmean_partial_kernel<<<dim3((unsigned)ceil_div(P.d, 128), nch), 128, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, part);
      CKL();
      colmean_final_kernel<<<(unsigned)ceil_div(P.d, 128), 128, 0, h->st>>>(part, (int)nch, P.n, P.d, h->mean);
      CKL();
      center_rows_kernel<<<(unsigned)ceil_div(P.n, 8), 256, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, h->mean);
      CKL();
    }
    // ---- a5: norms, bf16 split, diag
    {
      const int wpb = 8;
      prep_rows_kernel<<<(unsigned)ceil_div(P.npad, wpb), wpb * 32, 0, h->st>>>(
          h->Xf, P.ldf, P.n, P.npad, P.d, h->norms, h->Xhi, h->Xlo, P.dp,
          P.tc ? (P.fp16 ? 2 : 1) : 0, h->rscale);
      CKL();
      // Gaussian: the norms of r^2 = n_i + n_j - 2 b become the tensor core's own x_i . x_i, so the
      // one-signed accumulation error of b and of the norms cancels for like terms (DESIGN A9)
      if (p->kind == KKM_KERNEL_GAUSSIAN && P.tc &&
          tc3_self_dots(h->tc, h->Xhi, h->Xlo, P.fp16, h->rscale, P.npad, P.dp, P.n, h->norms, h->st, &h->launches,
                        h->chain_kb)) {
        h->poisoned = true;
        return fail(KKM_ECUDA, "tensor-core self dots failed: %s", tc_gemm_error());
      }
      if (P.a_n > 0) {
        diag_kernel<<<(unsigned)ceil_div(P.a_n, wpb), wpb * 32, 0, h->st>>>(
            h->Xf, P.ldf, P.d, P.a_row0, P.a_n, p->kind, p->gamma, p->coef0, p->degree, h->diag);
        CKL();
      }
    }
    // ---- labels (A5 round robin, or the caller's) and sizes
    for (int b = 0; b < 2; ++b) {
      round_robin_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(h->lab[b], P.n, P.lablen, P.k);
      CKL();
    }
    if (init_labels) {
      CK(cudaMemsetAsync(h->bad, 0, 4, h->st));
      int32_t *tmp = h->lab[1];
      CK(cudaMemcpyAsync(tmp, init_labels, (size_t)P.n * 4, cudaMemcpyDefault, h->st));
      load_labels_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(tmp, h->lab[0], P.n,
                                                                               P.lablen, P.k, h->bad);
      CKL();
      round_robin_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(h->lab[1], P.n, P.lablen, P.k);
      CKL();
      int bad = 0;
      CK(cudaMemcpyAsync(&bad, h->bad, 4, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      if (bad) return fail(KKM_ELABEL, "%d init labels outside [0, %d)", bad, P.k);
    }
    CK(cudaMemsetAsync(h->sizes[0], 0, (size_t)P.k * 4, h->st));
    histogram_kernel<<<std::min<int64_t>(ceil_div(P.n, 256), 1024), 256, (size_t)P.k * 4, h->st>>>(
        h->lab[0], P.n, P.k, h->sizes[0]);
    CKL();
    if (!evs.record(h->st)) return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    // ---- a1: K tile [A set, B set] = kappa(X X^T), materialised once; with
    // symmetric storage (f1) the owned upper-triangle bands, one launch each
    if (P.ssym) CK(cudaMemsetAsync(h->work, 0, 4 * 4, h->st));
    if (P.ssym && !P.units.empty())
      CK(cudaMemcpyAsync(h->units, P.units.data(), P.units.size() * sizeof(int4), cudaMemcpyHostToDevice, h->st));
    if (P.tc) {  // the fixed-point scale 2^s of the streaming kernels' S (loop, f3 deltas): n max|K| 2^s < 2^61
      max_norm_kernel<<<1, 1024, 0, h->st>>>(h->norms, P.n, h->fxmax);
      CKL();
      float mx = 0.f;
      CK(cudaMemcpyAsync(&mx, h->fxmax, 4, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      // |K_ij| <= max_i K_ii (K is a Gram matrix of phi); K_ii from the squared norm
      double kmax = 1.0;
      if (p->kind == KKM_KERNEL_LINEAR) kmax = std::max(1e-30, (double)mx);
      if (p->kind == KKM_KERNEL_POLY) kmax = std::pow(p->gamma * mx + std::fabs(p->coef0), (double)p->degree);
      const int sh = (int)std::floor(61.0 - std::log2(std::max(1e-300, (double)P.n * kmax * 1.0001)));
      h->fx_scale = std::ldexp(1.0, sh);
      h->fx_inv = std::ldexp(1.0, -sh);
    }
    if (P.sym) {
      if (!P.bands.empty())
        CK(cudaMemcpyAsync(h->bands, P.bands.data(), P.bands.size() * sizeof(SymBand), cudaMemcpyHostToDevice,
                           h->st));
      CK(cudaMemcpyAsync(h->band_desc, P.band_desc.data(), (size_t)P.T * 4, cudaMemcpyHostToDevice, h->st));
      CK(cudaMemsetAsync(h->work, 0, 4 * 4, h->st));
      CK(cudaMemsetAsync(h->a3ctr, 0, 16, h->st));
      if (P.kh) {  // f4: storage scale 2^e with |K| 2^e <= 60000 (|K_ij| <= max_i K_ii, bounded as for ssym)
        max_norm_kernel<<<1, 1024, 0, h->st>>>(h->norms, P.n, h->fxmax);
        CKL();
        float mx = 0.f;
        CK(cudaMemcpyAsync(&mx, h->fxmax, 4, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        double kmax = 1.0;
        if (p->kind == KKM_KERNEL_LINEAR) kmax = (double)mx;
        if (p->kind == KKM_KERNEL_POLY) kmax = std::pow(p->gamma * mx + std::fabs(p->coef0), (double)p->degree);
        const int e = std::max(-100, std::min(100, (int)std::floor(std::log2(60000.0 / std::max(1e-30, kmax * 1.0001)))));
        h->kscale = std::ldexp(1.0f, e);
        // S as int64 fixed point 2^s with n max|K| 2^s < 2^61 (as the streaming f1 kernel)
        const int sh = (int)std::floor(61.0 - std::log2(std::max(1e-300, (double)P.n * kmax * 1.0001)));
        h->tfxm = std::ldexp(1.0, sh - e);
        h->tfx_inv = std::ldexp(1.0, -sh);
        std::vector<CUtensorMap> maps(P.tbands.size() * P.kplanes);
        for (size_t b = 0; b < P.tbands.size(); ++b)
          for (int pl = 0; pl < P.kplanes; ++pl)
            if (ts_encode_band(&maps[b * P.kplanes + pl], (const __half *)h->K + pl * P.kelems + P.tbands[b].koff,
                               P.tbands[b].rows, P.tbands[b].ldb))
              return fail(KKM_ECUDA, "%s", tc_gemm_error());
        if (!maps.empty()) {
          CK(cudaMemcpyAsync(h->tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, h->st));
          CK(cudaMemcpyAsync(h->tbands, P.tbands.data(), P.tbands.size() * sizeof(TsBand), cudaMemcpyHostToDevice,
                             h->st));
        }
        if (!P.tunits.empty())
          CK(cudaMemcpyAsync(h->tunits, P.tunits.data(), P.tunits.size() * sizeof(TsUnit), cudaMemcpyHostToDevice,
                             h->st));
        if (!P.tslabs.empty())
          CK(cudaMemcpyAsync(h->ws + P.o_tslabs, P.tslabs.data(), P.tslabs.size() * sizeof(TsSlab),
                             cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));  // (host vectors go out of scope)
      }
      if (P.tc && !P.bands.empty()) {  // all owned pieces in one tcgen05 launch
        const int planes = P.kh ? P.kplanes : 1;
        std::vector<T2Region> regs(P.bands.size());
        std::vector<CUtensorMap> maps(P.bands.size() * planes);
        int64_t items = 0;
        for (size_t r = 0; r < P.bands.size(); ++r) {
          const SymBand &b = P.bands[r];
          T2Region &g = regs[r];
          g.j0 = (int64_t)b.band * SYM_TB;  // rows of the piece, columns >= the band start
          g.i0 = g.j0 + b.row0;
          g.m = b.rows;
          g.ncov = b.ldb;
          g.item0 = items;
          g.tiles_m = (int32_t)ceil_div(b.rows, T2_BM);
          g.tiles_n = (int32_t)ceil_div(b.ldb, 256);
          items += (int64_t)g.tiles_m * g.tiles_n;
          for (int pl = 0; pl < planes; ++pl) {
            void *out = P.kh ? (void *)((__half *)h->K + pl * P.kelems + b.koff) : (void *)(h->K + b.koff);
            if (tc3_encode_out_map(&maps[r * planes + pl], out, b.rows, b.ldb, b.ldb, P.kh))
              return fail(KKM_ECUDA, "%s", tc_gemm_error());
          }
        }
        T2Region *gregs = (T2Region *)((uint8_t *)h->ws + P.o_gregs);
        CUtensorMap *gmaps = (CUtensorMap *)((uint8_t *)h->ws + P.o_gmaps);
        CK(cudaMemcpyAsync(gregs, regs.data(), regs.size() * sizeof(T2Region), cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(gmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, h->st));
        if (tc3_gemm_launch_multi(h->tc, h->Xhi, h->Xlo, P.fp16, h->rscale, P.npad, P.dp, P.n, gregs,
                                  (int)regs.size(), items, gmaps, h->norms, h->kp, P.kh ? h->kscale : 0.f, planes,
                                  h->st, &h->launches, h->chain_kb)) {
          h->poisoned = true;
          return fail(KKM_ECUDA, "tcgen05 GEMM launch failed: %s", tc_gemm_error());
        }
        CK(cudaStreamSynchronize(h->st));  // (host copies of the regions and maps go out of scope)
      } else {
        for (const SymBand &b : P.bands) {
          const int64_t j0 = (int64_t)b.band * SYM_TB, i0 = j0 + b.row0;  // rows of the piece, columns >= band start
          CKR(launch_gemm(h, i0, b.rows, j0, b.ldb, h->K + b.koff, b.ldb));
        }
      }
    } else if (P.materialize) {
      CKR(launch_gemm(h, P.a0, P.nA, P.b0, P.ldk, h->K, P.ldk));
    }
    if (!evs.record(h->st)) return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    CK(cudaStreamSynchronize(h->st));
    if (h->p.timing) {
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, evs.v[0], evs.v[1]));
      CK(cudaEventElapsedTime(&b, evs.v[1], evs.v[2]));
      h->phase_ms[KKM_PH_INIT_PREP] += a;
      h->phase_ms[KKM_PH_INIT_GEMM] += b;
    }
    return KKM_OK;
  }();
  if (rc == KKM_OK && P.pr > 1) {
    // one column exchange and one pass of the iteration's world collectives now, so their NCCL
    // connection setup is part of the one-time init and not of the first iterations
    rc = [&]() -> int {
      CK(cudaMemsetAsync(h->Scol, 0, (size_t)P.nApad * P.k * 8, h->st));
      CKR(column_reduce_scatter(h));
      CK(cudaMemsetAsync(h->rankpart, 0, (size_t)P.nranks * (P.k + 1) * 8, h->st));
      CKN(ncclAllGather(h->rankpart + (int64_t)P.rank * (P.k + 1), h->rankpart, P.k + 1, ncclDouble, h->comm, h->st));
      CK(cudaMemsetAsync(h->changed, 0, 8, h->st));
      CKN(ncclAllReduce(h->changed, h->changed, 1, ncclUint64, ncclSum, h->comm, h->st));
      CK(cudaStreamSynchronize(h->st));
      return KKM_OK;
    }();
  }
  if (rc == KKM_OK && P.a3fix && P.k <= UG_MAX_K && P.a_n > 0) {  // a3 + a4 as one cooperative launch
    int coop = 0, per_sm = 0, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) == cudaSuccess && coop &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, update_grid_kernel<true>, UG_THREADS, 0) == cudaSuccess)
      h->ug_grid = per_sm * h->num_sms;
    cudaGetLastError();
  }
  // Opt-in (KKM_LSA=1): a3/a4 distributed over the ranks inside the fused update, reading S from
  // every rank's NCCL symmetric window over NVLink instead of an NCCL allreduce per iteration.
  // Measured on 4 B200: the same per-iteration time as the allreduce + replicated
  // update (0.398 vs 0.404 ms at config 2; three cross-rank arrivals cost what the allreduce did)
  // and +50 ms of window registration per handle, so the default stays on NCCL. Every rank
  // evaluates the same condition (same plan, env) and agrees before the collective setup.
  if (rc == KKM_OK && P.repl && P.nranks > 1 && P.nranks <= LSA_MAX_RANKS && P.a3fix &&
      P.k <= UG_MAX_K) {
    int want = 0;
    if (const char *e = std::getenv("KKM_LSA")) want = h->ug_grid > 0 && std::atoi(e) == 1;
    if (std::getenv("KKM_LSA_DEBUG"))
      std::fprintf(stderr, "[kkm rank %d] lsa wish %d (ug_grid %d)\n", P.rank, want, h->ug_grid);
    rc = agree_min(h, &want);
    if (rc == KKM_OK && want) rc = setup_lsa(h);
  }
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return KKM_OK;
}

int kkm_fit(kkm_handle h, int32_t *iters_run, double *J_trace, int64_t *changed) {
  if (!h) return fail(KKM_EINVAL, "handle is NULL");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned by an earlier CUDA/NCCL error");
  const Plan &P = h->P;
  const int T = h->p.max_iter;
  EventList ev;  // 5 per iteration (timing mode)
  const bool timing = h->p.timing != 0;
  auto rec = [&](EventList &l) -> int {
    if (!l.record(h->st)) {
      h->poisoned = true;
      return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    }
    return KKM_OK;
  };
  h->a2ev.clear();
  int t = 0;
  h->time_a2 = timing;
  for (t = 0; t < T; ++t) {
    if (timing) CKR(rec(ev));
    const double *S = nullptr;
    int ns = 0;
    int64_t rows_pad = P.s_rows_pad;
    if (P.inc && h->s_valid) {  // f3: S of the current labels maintained incrementally
      S = h->Sinc;
      ns = 1;
      rows_pad = P.B;
    } else {
      h->ls_fused_next = h->lsa && use_update_grid(h);  // (peer-memory window: no allreduce, run_update_grid)
      const int arc = launch_spmm(h, h->lab[h->cur], &S, &ns);  // a2 (+ 1.5D reduce-scatter)
      if (arc != KKM_OK) {
        h->ls_fused_next = false;
        return arc;
      }
      if (P.inc && P.nloc > 0) {
        sinc_set_kernel<<<(unsigned)ceil_div(P.nloc * P.k, 256), 256, 0, h->st>>>(S, ns, rows_pad, P.nloc, P.k,
                                                                                   h->Sinc);
        CKL();
      }
    }
    if (timing) CKR(rec(ev));
    if (P.fused) {  // a3 + a4 in one launch (the phase split is reported as a3)
      fused_update_kernel<<<1, FUSED_THREADS, (size_t)(P.k + 1) * FUSED_THREADS * 8 + P.k * 8, h->st>>>(
          S, ns, P.n, rows_pad, P.k, h->sizes[h->cur], h->lab[h->cur], h->diag, h->E, h->cnorm, h->J + t, 1,
          h->lab[h->cur ^ 1], h->sizes[h->cur ^ 1], h->changed + t, h->Dfull);
      CKL();
      if (timing) CKR(rec(ev));
    } else if (use_update_grid(h)) {  // a3 + a4 in one launch (reported as a3)
      const int urc = run_update_grid(h, h->J + t, h->changed + t);
      h->ls_fused_next = false;
      CKR(urc);
      if (timing) CKR(rec(ev));
    } else {
      CKR(run_cnorm(h, S, ns, rows_pad, h->E, h->cnorm, h->J + t, h->sizes[h->cur ^ 1], h->changed + t));  // a3
      if (timing) CKR(rec(ev));
      CKR(run_assign(h, h->changed + t));                                   // a4
    }
    if (timing) CKR(rec(ev));
    unsigned long long c = 1;
    if (h->p.stop_on_no_change || P.inc) {
      CK(cudaMemcpyAsync(&c, h->changed + t, 8, cudaMemcpyDeviceToHost, h->st));
      CKR(sync_stream(h));
    }
    if (P.inc) {  // S for the new labels: unchanged, by the moved points, or a full pass next time
      if (c > 0 && (int64_t)c <= P.dmax) {
        CKR(delta_update(h, (int64_t)c));
        h->s_valid = true;
      } else {
        h->s_valid = c == 0;
      }
    }
    if (timing) CKR(rec(ev));
    h->cur ^= 1;
    h->have_last = true;
    if (h->p.stop_on_no_change && c == 0) {
      ++t;
      break;
    }
  }
  h->time_a2 = false;
  // J of the final labels (one more a2 + a3 pass, as the oracle's J_trace[iters])
  {
    const double *S = nullptr;
    int ns = 0;
    int64_t rows_pad = P.s_rows_pad;
    if (P.inc && h->s_valid) {
      S = h->Sinc;
      ns = 1;
      rows_pad = P.B;
    } else {
      CKR(launch_spmm(h, h->lab[h->cur], &S, &ns));
    }
    CKR(run_cnorm(h, S, ns, rows_pad, h->E2, h->cnorm2, h->J + t, nullptr, nullptr));
    h->cnorm2_valid = true;
  }
  std::vector<double> J((size_t)t + 1);
  std::vector<unsigned long long> ch((size_t)std::max(t, 1));
  CK(cudaMemcpyAsync(J.data(), h->J, (size_t)(t + 1) * 8, cudaMemcpyDeviceToHost, h->st));
  if (t > 0) CK(cudaMemcpyAsync(ch.data(), h->changed, (size_t)t * 8, cudaMemcpyDeviceToHost, h->st));
  CKR(sync_stream(h));
  CKR(check_lsa(h));
#ifdef KKM_EXP_LSA_STAMPS
  if (h->lsa) {
    unsigned long long st[10];
    CK(cudaMemcpy(st, h->lsbuf + h->ls_off_flag + 32 * 8, sizeof(st), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[kkm rank %d] last update (us): wait1 %.1f ph0 %.1f ph1 %.1f gridbar %.1f sums %.1f wait2 %.1f ph2 %.1f "
                 "gridbar %.1f wait3 %.1f\n", h->P.rank, (st[1] - st[0]) * 1e-3, (st[9] - st[1]) * 1e-3, (st[2] - st[9]) * 1e-3,
                 (st[3] - st[2]) * 1e-3, (st[4] - st[3]) * 1e-3, (st[5] - st[4]) * 1e-3, (st[6] - st[5]) * 1e-3,
                 (st[7] - st[6]) * 1e-3, (st[8] - st[7]) * 1e-3);
  }
#endif
  if (timing) {
    const std::vector<cudaEvent_t> &e5 = ev.v;
    for (size_t i = 0; i + 4 < e5.size(); i += 5) {  // the a2 phase includes the f3 S update
      float a, b, c, d;
      CK(cudaEventElapsedTime(&a, e5[i], e5[i + 1]));
      CK(cudaEventElapsedTime(&b, e5[i + 1], e5[i + 2]));
      CK(cudaEventElapsedTime(&c, e5[i + 2], e5[i + 3]));
      CK(cudaEventElapsedTime(&d, e5[i + 3], e5[i + 4]));
      h->phase_ms[KKM_PH_SPMM] += a + d;
      h->phase_ms[KKM_PH_CNORM] += b;
      h->phase_ms[KKM_PH_ASSIGN] += c;
    }
    const std::vector<cudaEvent_t> &a2 = h->a2ev.v;
    for (size_t i = 0; i + 1 < a2.size(); i += 2) {
      float a = 0;
      CK(cudaEventElapsedTime(&a, a2[i], a2[i + 1]));
      h->phase_ms[KKM_PH_A2_KERNEL] += a;
    }
  }
  h->a2ev.clear();
  if (iters_run) *iters_run = t;
  if (J_trace) std::memcpy(J_trace, J.data(), (size_t)(t + 1) * 8);
  if (changed)
    for (int i = 0; i < t; ++i) changed[i] = (int64_t)ch[i];
  (void)P;
  return KKM_OK;
}

int kkm_assign(kkm_handle h, int32_t *labels_out) {
  if (!h || !labels_out) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  CKR(copy_any(h, labels_out, h->lab[h->cur], (size_t)h->P.n * 4));
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

int kkm_objective(kkm_handle h, double *J) {
  if (!h || !J) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  double *slot = h->J + h->P.max_iter + 1;
  const double *S = nullptr;
  int ns = 0;
  CKR(launch_spmm(h, h->lab[h->cur], &S, &ns));
  CKR(run_cnorm(h, S, ns, h->P.s_rows_pad, h->E2, h->cnorm2, slot, nullptr, nullptr));
  h->cnorm2_valid = true;
  CK(cudaMemcpyAsync(J, slot, 8, cudaMemcpyDeviceToHost, h->st));
  CKR(sync_stream(h));
  return KKM_OK;
}

int kkm_set_labels(kkm_handle h, const int32_t *labels) {
  if (!h || !labels) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  // validated in the scratch buffer first: a rejected call leaves the current labels untouched
  int32_t *dst = h->lab[h->cur], *tmp = h->lab[h->cur ^ 1];
  CK(cudaMemsetAsync(h->bad, 0, 4, h->st));
  CK(cudaMemcpyAsync(tmp, labels, (size_t)P.n * 4, cudaMemcpyDefault, h->st));
  check_labels_kernel<<<(unsigned)ceil_div(P.n, 256), 256, 0, h->st>>>(tmp, P.n, P.k, h->bad);
  CKL();
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, h->bad, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (!bad) {
    load_labels_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(tmp, dst, P.n, P.lablen, P.k, h->bad);
    CKL();
    CK(cudaMemsetAsync(h->sizes[h->cur], 0, (size_t)P.k * 4, h->st));
    histogram_kernel<<<std::min<int64_t>(ceil_div(P.n, 256), 1024), 256, (size_t)P.k * 4, h->st>>>(
        dst, P.n, P.k, h->sizes[h->cur]);
    CKL();
  }
  round_robin_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(tmp, P.n, P.lablen, P.k);
  CKL();
  CK(cudaStreamSynchronize(h->st));
  if (bad) return fail(KKM_ELABEL, "%d labels outside [0, %d); current labels kept", bad, P.k);
  h->have_last = false;
  h->cnorm2_valid = false;
  h->s_valid = false;
  return KKM_OK;
}

}  // extern "C"

extern "C" {

int kkm_predict_workspace_size(kkm_handle h, int64_t m, size_t *bytes) {
  if (!h || !bytes) return fail(KKM_EINVAL, "NULL argument");
  if (m < 0) return fail(KKM_EINVAL, "m=%lld < 0", (long long)m);
  *bytes = predict_plan(h, m).total;
  return KKM_OK;
}

int kkm_predict(kkm_handle h, const float *Y, int64_t m, int64_t ldy, int32_t *labels_out, double *D_out,
                void *workspace, size_t ws_bytes) {
  if (!h) return fail(KKM_EINVAL, "handle is NULL");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  if (m < 0) return fail(KKM_EINVAL, "m=%lld < 0", (long long)m);
  if (m == 0) return KKM_OK;
  if (!Y || !labels_out) return fail(KKM_EINVAL, "NULL argument");
  if (ldy < P.d) return fail(KKM_EINVAL, "ldy=%lld < d=%lld", (long long)ldy, (long long)P.d);
  if (!P.tc) return fail(KKM_EUNSUP, "kkm_predict needs a tensor-core precision (FP16X3 or BF16X3)");
  const PredictPlan q = predict_plan(h, m);
  if (workspace) {
    if (((uintptr_t)workspace) & 255) return fail(KKM_EINVAL, "workspace must be 256-byte aligned");
    if (ws_bytes < q.total) return fail(KKM_ENOMEM, "workspace %zu bytes < required %zu", ws_bytes, q.total);
  }
  if (!h->cnorm2_valid) {  // c of the current labels: the kkm_objective pass (collective for nranks > 1)
    if (P.nranks > 1) return fail(KKM_ESTATE, "call kkm_fit or kkm_objective on every rank before kkm_predict");
    double J = 0.0;
    CKR(kkm_objective(h, &J));
  }
  if (workspace) return predict_run(h, q, (uint8_t *)workspace, Y, m, ldy, labels_out, D_out);
  uint8_t *t = nullptr;
  if (cudaMallocAsync((void **)&t, q.total, h->st) != cudaSuccess) {
    cudaGetLastError();
    return fail(KKM_ENOMEM, "kkm_predict: cannot allocate %zu temporary bytes", q.total);
  }
  const int rc = predict_run(h, q, t, Y, m, ldy, labels_out, D_out);
  cudaFreeAsync(t, h->st);
  if (rc == KKM_OK) CK(cudaStreamSynchronize(h->st));
  return rc;
}

int kkm_seed_kmeanspp(kkm_handle h, const double *u, int64_t *centers_out) {
  if (!h || !u) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  const int k = P.k;
  for (int t = 0; t < k; ++t)
    if (!(u[t] >= 0.0 && u[t] < 1.0)) return fail(KKM_EINVAL, "u[%d] = %g outside [0, 1)", t, u[t]);
  int64_t c0 = (int64_t)(u[0] * (double)P.n);
  if (c0 >= P.n) c0 = P.n - 1;
  uint8_t *t0 = nullptr;
  const size_t oD = 0, oL = round_up((int64_t)P.n * 8, 256), oC = oL + round_up((int64_t)P.n * 4, 256),
               total = oC + round_up((int64_t)k * 8, 256);
  if (cudaMallocAsync((void **)&t0, total, h->st) != cudaSuccess) {
    cudaGetLastError();
    return fail(KKM_ENOMEM, "kkm_seed_kmeanspp: cannot allocate %zu temporary bytes", total);
  }
  double *D = (double *)(t0 + oD);
  int32_t *lab = (int32_t *)(t0 + oL);
  int64_t *cen = (int64_t *)(t0 + oC);
  int rc = [&]() -> int {
    CK(cudaMemcpyAsync(cen, &c0, 8, cudaMemcpyHostToDevice, h->st));
    for (int t = 0; t < k; ++t) {
      kpp_dist_kernel<<<(unsigned)ceil_div(P.n, 8), 256, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, cen, t, h->p.kind,
                                                                      h->p.gamma, h->p.coef0, h->p.degree, D, lab);
      CKL();
      if (t + 1 < k) {
        kpp_pick_kernel<<<1, 1024, 0, h->st>>>(D, P.n, u[t + 1], t, cen);
        CKL();
      }
    }
    if (centers_out) CKR(copy_any(h, centers_out, cen, (size_t)k * 8));
    CK(cudaStreamSynchronize(h->st));
    return kkm_set_labels(h, lab);  // validates, sets sizes, invalidates the derived state
  }();
  cudaFreeAsync(t0, h->st);
  cudaStreamSynchronize(h->st);
  return rc;
}

int kkm_debug_read(kkm_handle h, int32_t what, void *dst) {
  if (!h || !dst) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  const int prev = h->cur ^ 1;  // buffers of the labels entering the last iteration
  switch (what) {
    case KKM_DBG_E: CKR(copy_any(h, dst, h->E + (P.row0 - P.a_row0) * P.k, (size_t)P.nloc * P.k * 8)); break;
    case KKM_DBG_CNORM: CKR(copy_any(h, dst, h->cnorm, (size_t)P.k * 8)); break;
    case KKM_DBG_SIZES:
      CKR(copy_any(h, dst, h->sizes[h->have_last ? prev : h->cur], (size_t)P.k * 4));
      break;
    case KKM_DBG_DIAG: CKR(copy_any(h, dst, h->diag + (P.row0 - P.a_row0), (size_t)P.nloc * 8)); break;
    case KKM_DBG_DFULL:  // formed from the last iteration's E and c (the expression of a4)
      if (P.a_n > 0) {
        dfull_kernel<<<(unsigned)ceil_div(P.a_n * P.k, 256), 256, 0, h->st>>>(h->E, P.a_n, P.k, h->cnorm, h->diag,
                                                                            h->Dfull);
        CKL();
      }
      CKR(copy_any(h, dst, h->Dfull + (P.row0 - P.a_row0) * P.k, (size_t)P.nloc * P.k * 8));
      break;
    case KKM_DBG_LABELS_PREV:
      CKR(copy_any(h, dst, h->lab[h->have_last ? prev : h->cur], (size_t)P.n * 4));
      break;
    default: return fail(KKM_EINVAL, "unknown debug selector %d", what);
  }
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

int kkm_stored_k_row(kkm_handle h, int64_t i, double *dst) {
  if (!h || !dst) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  if (i < 0 || i >= P.n) return fail(KKM_EINVAL, "row %lld out of range", (long long)i);
  if (!P.materialize) return fail(KKM_ESTATE, "the handle streams K: nothing is stored");
  std::vector<double> out((size_t)P.n, std::nan(""));
  if (P.sym) {
    const SymBand *piece = nullptr;
    for (const SymBand &b : P.bands) {
      const int64_t r0 = (int64_t)b.band * SYM_TB + b.row0;
      if (i >= r0 && i < r0 + b.rows) piece = &b;
    }
    if (!piece) return fail(KKM_ESTATE, "row %lld is not stored on this rank", (long long)i);
    const int64_t j0 = (int64_t)piece->band * SYM_TB;
    const int64_t r = i - j0 - piece->row0, cols = P.n - j0;
    if (P.kh) {
      std::vector<__half> hi((size_t)cols), lo((size_t)cols);
      const __half *base = (const __half *)h->K + piece->koff + r * piece->ldb;
      CK(cudaMemcpyAsync(hi.data(), base, (size_t)cols * 2, cudaMemcpyDeviceToHost, h->st));
      if (P.kplanes > 1)
        CK(cudaMemcpyAsync(lo.data(), base + P.kelems, (size_t)cols * 2, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      const double inv = 1.0 / (double)h->kscale;
      for (int64_t j = 0; j < cols; ++j)
        out[(size_t)(j0 + j)] = ((double)__half2float(hi[(size_t)j]) +
                                 (P.kplanes > 1 ? (double)__half2float(lo[(size_t)j]) : 0.0)) * inv;
    } else {
      std::vector<float> v((size_t)cols);
      CK(cudaMemcpyAsync(v.data(), h->K + piece->koff + r * piece->ldb, (size_t)cols * 4, cudaMemcpyDeviceToHost,
                         h->st));
      CK(cudaStreamSynchronize(h->st));
      for (int64_t j = 0; j < cols; ++j) out[(size_t)(j0 + j)] = v[(size_t)j];
    }
  } else {  // full K rows: the A set's rows x the B set's columns
    if (i < P.a0 || i >= P.a0 + P.nA) return fail(KKM_ESTATE, "row %lld is not stored on this rank", (long long)i);
    std::vector<float> v((size_t)P.nB);
    CK(cudaMemcpyAsync(v.data(), h->K + (i - P.a0) * P.ldk, (size_t)P.nB * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    for (int64_t j = 0; j < P.nB; ++j) out[(size_t)(P.b0 + j)] = v[(size_t)j];
  }
  std::memcpy(dst, out.data(), (size_t)P.n * 8);
  return KKM_OK;
}

int kkm_kernel_tile(kkm_handle h, int64_t i0, int64_t j0, int32_t m, int32_t nc, float *dst) {
  if (!h || !dst) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  if (m < 1 || nc < 1 || i0 < 0 || j0 < 0 || i0 + m > P.n || j0 + nc > P.n)
    return fail(KKM_EINVAL, "tile out of range");
  float *tmp = nullptr;
  const int64_t ldt = round_up(nc, 4);  // TMA-store pitch
  CK(cudaMallocAsync((void **)&tmp, (size_t)m * ldt * 4, h->st));
  int rc = launch_gemm(h, i0, m, j0, nc, tmp, ldt);
  if (rc == KKM_OK) {
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)nc * 4, tmp, (size_t)ldt * 4, (size_t)nc * 4, m,
                                      cudaMemcpyDefault, h->st);
    if (e != cudaSuccess) rc = fail(KKM_ECUDA, "kernel_tile copy: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(tmp, h->st);
  if (rc) return rc;
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

int kkm_phase_ms(kkm_handle h, float *ms) {
  if (!h || !ms) return fail(KKM_EINVAL, "NULL argument");
  std::memcpy(ms, h->phase_ms, sizeof(h->phase_ms));
  return KKM_OK;
}

int kkm_launch_count(kkm_handle h, int64_t *count) {
  if (!h || !count) return fail(KKM_EINVAL, "NULL argument");
  *count = h->launches;
  return KKM_OK;
}

int kkm_destroy(kkm_handle h) {
  if (!h) return KKM_OK;
  cudaStreamSynchronize(h->st);
  if (h->lsa) {  // collective: every rank destroys its handle before the communicator
    ncclDevCommDestroy(h->comm, &h->lsdev);
    ncclCommWindowDeregister(h->comm, h->lswin);
    ncclMemFree(h->lsbuf);
    cudaGetLastError();
  }
  delete h;
  return KKM_OK;
}

int kkm_get_unique_id(char id[128]) {
  if (!id) return fail(KKM_EINVAL, "id is NULL");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(KKM_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return KKM_OK;
}

int kkm_comm_init(void **comm, int32_t nranks, int32_t rank, const char id[128]) {
  if (!comm || !id) return fail(KKM_EINVAL, "NULL argument");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return fail(KKM_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  *comm = c;
  return KKM_OK;
}

int kkm_comm_destroy(void *comm) {
  if (!comm) return KKM_OK;
  ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return fail(KKM_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return KKM_OK;
}

}  // extern "C"

