// api_ctx.cuh -- the handle (kkm_ctx) of kkm_api.cu, the status macros and small helpers.
#pragma once

// CUDA events owned for one scope (destroyed on every exit path, errors included).
struct EventList {
  std::vector<cudaEvent_t> v;
  EventList() = default;
  EventList(const EventList &) = delete;
  EventList &operator=(const EventList &) = delete;
  ~EventList() { clear(); }
  void clear() {
    for (cudaEvent_t e : v) cudaEventDestroy(e);
    v.clear();
  }
  // creates and records one event; false if the runtime refused
  bool record(cudaStream_t st) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return false;
    v.push_back(e);
    return cudaEventRecord(e, st) == cudaSuccess;
  }
};

// Label-sorted copy of a point set (the B operand of the streaming kernel) and its sort.
struct SortedSet {
  uint16_t *hi, *lo;
  float *norms, *rscale;
  int32_t *perm, *pos, *seg, *bcount, *boff;
};

struct kkm_ctx {
  kkm_params p;
  Plan P;
  cudaStream_t st = nullptr;
  ncclComm_t comm = nullptr;
  int num_sms = 148;
  int ug_grid = 0;  // co-resident blocks of update_grid_kernel (0: not used by this plan)
  uint8_t *ws = nullptr;
  float *Xf = nullptr, *norms = nullptr, *K = nullptr;
  float *mean = nullptr;  // Gaussian: the column means X was centered on (0 otherwise)
  uint16_t *Xhi = nullptr, *Xlo = nullptr;  // bf16 or fp16 split of X (P.tc)
  float *rscale = nullptr;                   // 1 / s_i of the fp16 split
  double *diag, *Spart, *E, *blockpart, *rankpart, *cnorm, *J, *Dfull;
  double *E2, *cnorm2;  // E / c of the final-labels pass (kept apart from the last iteration's)
  // streaming path: cluster-sorted operands and the sort
  uint16_t *Shi = nullptr, *Slo = nullptr;
  float *snorms = nullptr, *srscale = nullptr;
  int32_t *perm = nullptr, *pos = nullptr, *seg = nullptr, *bcount = nullptr, *boff = nullptr;
  TcStream ts, ts_predict;  // tensor maps of the clustering loop / of kkm_predict
  // 1.5D: padded labels of the B set, column-block partials, own-block sums; column comm
  int32_t *labB = nullptr;
  double *Scol = nullptr, *Smine = nullptr;
  uint32_t *codes = nullptr;  // SpMM v2 per-iteration group codes
  // f1 symmetric storage
  int32_t *perm_b = nullptr, *ngroups = nullptr, *band_desc = nullptr, *gfirst = nullptr;
  SymGroup *groups = nullptr;
  SymBand *bands = nullptr;
  float *colpart = nullptr;
  double *colsum = nullptr, *Sfin = nullptr;
  int32_t *work = nullptr;  // item schedulers: [0, 2) spmm_tc, [2, 4) ssym (zero between launches)
  unsigned *a3ctr = nullptr;  // finalize's last-block counter (zero between launches)
  // Distributed a3/a4 over NVLink peer memory (16-bit bands, replicated plan, several ranks;
  // api_exchange.cuh setup_lsa): an NCCL symmetric window per rank [2 parities of k x npad int64 S |
  // 2 label buffers | 2 size histograms | changed counters | rank partials | flag page], mapped by
  // every rank; S is summed by the fused a3/a4 kernel while it reads it (no allreduce)
  bool lsa = false;
  uint8_t *lsbuf = nullptr;            // own window (ncclMemAlloc)
  ncclWindow_t lswin = nullptr;
  ncclDevComm lsdev{};
  LsaArgs lsargs{};                    // peer bases + section offsets (off_S etc. set per launch)
  size_t ls_sb = 0, ls_off_lab = 0, ls_lb = 0, ls_off_sizes = 0, ls_off_changed = 0, ls_off_rankpart = 0,
         ls_off_flag = 0;
  int ls_par = 0;                      // parity of the S buffer the latest a2 wrote
  bool ls_fused_next = false;          // the next a2's consumer sums S itself (no allreduce)
  uint32_t ls_epoch = 0;               // cross-rank arrivals per rank so far
  // f4 fp16 K storage
  CUtensorMap *tmaps = nullptr;
  TsBand *tbands = nullptr;
  TsUnit *tunits = nullptr;
  long long *tSfix = nullptr, *tSint = nullptr, *tSmine = nullptr;
  float kscale = 1.f;  // stored K = K * kscale (a power of two)
  double tfxm = 1.0, tfx_inv = 1.0;  // S fixed point: drained (scaled) sums x tfxm; back x tfx_inv
  // f1 streaming: units, int64 fixed-point S (sorted order), its original-order copy
  int4 *units = nullptr;
  long long *Sfix = nullptr, *Sorig = nullptr, *Sfmine = nullptr;
  float *fxmax = nullptr;
  double fx_scale = 1.0, fx_inv = 1.0;
  // f3 incremental S
  double *Sinc = nullptr, *Sd = nullptr;
  long long *Sdx = nullptr;
  int32_t *dkey = nullptr;
  SortedSet dset{};
  bool s_valid = false;  // Sinc holds S of the current labels
  TcStream ts_delta;
  int32_t *lab[2], *sizes[2];
  unsigned long long *changed;
  int *bad;
  int cur = 0;  // labels[cur] / sizes[cur] are the labels entering the next iteration
  bool poisoned = false;
  int chain_kb = 0;      // K-blocks per accumulation chain of every tensor-core kernel (0: CH_CKB; KKM_CHAIN_KB)
  bool have_last = false;
  bool cnorm2_valid = false;  // cnorm2 holds c of the current labels (after kkm_fit / kkm_objective)
  int64_t launches = 0;
  float phase_ms[KKM_NPHASES] = {0, 0, 0, 0, 0, 0};
  bool time_a2 = false;             // timing mode, inside the kkm_fit loop
  EventList a2ev;                   // (start, end) pairs around the dominant a2 kernel
  KappaParams kp;
  TcGemm tc;
};

namespace {

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      h->poisoned = true;                                                                \
      return fail(KKM_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    }                                                                                    \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    ++h->launches;                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess) {                                                             \
      h->poisoned = true;                                                                \
      return fail(KKM_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
    }                                                                                    \
  } while (0)

#define CKN(call)                                                                        \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      h->poisoned = true;                                                                \
      return fail(KKM_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call, ncclGetErrorString(r_)); \
    }                                                                                    \
  } while (0)

#define CKR(expr)        \
  do {                   \
    int rc_ = (expr);    \
    if (rc_) return rc_; \
  } while (0)

// Brackets the dominant a2 kernel launch(es) with CUDA events (timing mode, kkm_fit loop).
void a2_mark(kkm_ctx *h) {
  if (h->time_a2) h->a2ev.record(h->st);
}

// Waits for the handle's stream. With a communicator the wait polls the stream and NCCL's
// asynchronous error state instead of blocking: a failed or aborted peer turns into KKM_ENCCL (handle
// poisoned; the caller aborts the communicator) rather than a hang, and a collective that has not
// completed within KKM_NCCL_TIMEOUT_S seconds (default 1800) is reported the same way.
int sync_stream(kkm_ctx *h) {
  if (!h->comm) {
    CK(cudaStreamSynchronize(h->st));
    return KKM_OK;
  }
  double tmo = 1800.0;
  if (const char *e = std::getenv("KKM_NCCL_TIMEOUT_S")) tmo = std::max(1.0, std::atof(e));
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(h->st);
    if (q == cudaSuccess) return KKM_OK;
    if (q != cudaErrorNotReady) CK(q);
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(h->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
      h->poisoned = true;
      return fail(KKM_ENCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ar));
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > tmo) {
      h->poisoned = true;
      return fail(KKM_ENCCL, "collective did not complete within %.0f s (KKM_NCCL_TIMEOUT_S)", tmo);
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// Host or device pointer copy on the handle's stream.
int copy_any(kkm_ctx *h, void *dst, const void *src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->st));
  return KKM_OK;
}

}  // namespace
