// api_exchange.cuh -- multi-GPU setup of kkm_api.cu beyond NCCL: the rank agreement helper and the
// opt-in peer-memory exchange of S (IPC buffers, epoch flags, bounded waits).
#pragma once

// *v = the minimum of *v over all ranks (a collective on the handle's communicator).
static int agree_min(kkm_ctx *h, int *v) {
  int *d = nullptr;
  if (cudaMallocAsync((void **)&d, 4, h->st) != cudaSuccess) return fail(KKM_ECUDA, "cudaMallocAsync failed");
  int rc = [&]() -> int {
    CK(cudaMemcpyAsync(d, v, 4, cudaMemcpyHostToDevice, h->st));
    CKN(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, h->comm, h->st));
    CK(cudaMemcpyAsync(v, d, 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return KKM_OK;
  }();
  cudaFreeAsync(d, h->st);
  return rc;
}

namespace {
// Every rank's window base as mapped in this process (device-side NCCL accessor, read back once).
__global__ void lsa_bases_kernel(ncclWindow_t win, int nranks, uint8_t **out) {
  for (int p = 0; p < nranks; ++p) out[p] = (uint8_t *)ncclGetPeerPointer(win, 0, p);
}
}  // namespace

// NVLink peer-memory window for the distributed a3/a4 (16-bit bands, several ranks on one NVLink
// domain, §6): an NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister) per rank holding
// [2 parities of k x npad int64 S | 2 label buffers | 2 size histograms | the changed counters |
// the ranks' (k + 1) partials | a flag page], every rank's window mapped here (ncclGetPeerPointer;
// ncclDevCommCreate confirms all ranks share the load/store domain). The handle's labels, sizes
// and changed counters move into the window (current values copied). spmm_tc writes the rank's S
// into it; update_grid_kernel<true> reads the P copies of its own rows' S and stores the results
// into every rank's copies. All ranks agree on the outcome (allreduce min); any failure leaves
// every rank on the NCCL allreduce path. Collective; kkm_destroy undoes it (also collective).
static int setup_lsa(kkm_ctx *h) {
  const Plan &P = h->P;
  auto r4k = [](size_t b) { return (b + 4095) / 4096 * 4096; };
  const size_t sb = r4k((size_t)P.npad * P.k * 8), lb = r4k((size_t)P.lablen * 4);
  const size_t off_lab = 2 * sb, off_sizes = off_lab + 2 * lb, off_changed = off_sizes + 2 * 4096;
  const size_t off_rankpart = off_changed + r4k((size_t)(P.max_iter + 2) * 8);
  const size_t off_flag = off_rankpart + r4k((size_t)P.nranks * (P.k + 1) * 8);
  const size_t total = off_flag + 4096;
  void *buf = nullptr;
  int ok = ncclMemAlloc(&buf, total) == ncclSuccess ? 1 : 0;
  if (std::getenv("KKM_LSA_DEBUG"))
    std::fprintf(stderr, "[kkm rank %d] setup_lsa: ncclMemAlloc(%zu) ok %d\n", P.rank, total, ok);
  CKR(agree_min(h, &ok));
  if (!ok) {
    if (buf) ncclMemFree(buf);
    cudaGetLastError();
    return KKM_OK;
  }
  ncclWindow_t win = nullptr;
  CKN(ncclCommWindowRegister(h->comm, buf, total, &win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements reqs;
  std::memset(&reqs, 0, sizeof(reqs));
  ncclDevComm dev;
  std::memset(&dev, 0, sizeof(dev));
  const bool have_dev = ncclDevCommCreate(h->comm, &reqs, &dev) == ncclSuccess;
  ok = have_dev && dev.lsaSize == P.nranks && dev.nRanks == P.nranks;
  LsaArgs L{};
  if (ok) {
    uint8_t **d = nullptr;
    CK(cudaMallocAsync((void **)&d, sizeof(L.base), h->st));
    lsa_bases_kernel<<<1, 1, 0, h->st>>>(win, P.nranks, d);
    CKL();
    CK(cudaMemcpyAsync(L.base, d, (size_t)P.nranks * sizeof(uint8_t *), cudaMemcpyDeviceToHost, h->st));
    CK(cudaFreeAsync(d, h->st));
    CK(cudaStreamSynchronize(h->st));
    for (int p = 0; p < P.nranks; ++p) ok = ok && L.base[p] != nullptr;
    // (base[rank] is NCCL's flat-space alias of buf: the same pages under another address)
  }
  if (ok) {  // the current labels / sizes / changed into the window; flags and partials zeroed
    CK(cudaMemsetAsync(buf, 0, total, h->st));
    for (int b = 0; b < 2; ++b) {
      CK(cudaMemcpyAsync((uint8_t *)buf + off_lab + b * lb, h->lab[b], (size_t)P.lablen * 4, cudaMemcpyDeviceToDevice,
                         h->st));
      CK(cudaMemcpyAsync((uint8_t *)buf + off_sizes + b * 4096, h->sizes[b], (size_t)P.k * 4, cudaMemcpyDeviceToDevice,
                         h->st));
    }
    CK(cudaStreamSynchronize(h->st));
  }
  if (std::getenv("KKM_LSA_DEBUG"))
    std::fprintf(stderr, "[kkm rank %d] setup_lsa: devcomm %d lsaSize %d nRanks %d bases %p %p ok %d\n", P.rank,
                 (int)have_dev, dev.lsaSize, dev.nRanks, (void *)L.base[0], (void *)L.base[1], ok);
  CKR(agree_min(h, &ok));  // (also orders every rank's zeroing before any peer's first arrival)
  if (!ok) {
    if (have_dev) ncclDevCommDestroy(h->comm, &dev);
    ncclCommWindowDeregister(h->comm, win);
    ncclMemFree(buf);
    cudaGetLastError();
    return KKM_OK;
  }
  L.nranks = P.nranks;
  L.rank = P.rank;
  L.off_rankpart = off_rankpart;
  L.off_flag = off_flag;
  h->lsa = true;
  h->lsbuf = (uint8_t *)buf;
  h->lswin = win;
  h->lsdev = dev;
  h->lsargs = L;
  h->ls_sb = sb;
  h->ls_lb = lb;
  h->ls_off_lab = off_lab;
  h->ls_off_sizes = off_sizes;
  h->ls_off_changed = off_changed;
  h->ls_off_rankpart = off_rankpart;
  h->ls_off_flag = off_flag;
  h->ls_par = 0;
  h->ls_epoch = 0;
  for (int b = 0; b < 2; ++b) {
    h->lab[b] = (int32_t *)(h->lsbuf + off_lab + b * lb);
    h->sizes[b] = (int32_t *)(h->lsbuf + off_sizes + b * 4096);
  }
  h->changed = (unsigned long long *)(h->lsbuf + off_changed);
  return KKM_OK;
}

// After a synchronised fit on the peer-memory path: a cross-rank wait that ran out poisons the handle.
static int check_lsa(kkm_ctx *h) {
  if (!h->lsa) return KKM_OK;
  unsigned to = 0;
  CK(cudaMemcpy(&to, h->lsbuf + h->ls_off_flag + 64, 4, cudaMemcpyDeviceToHost));
  if (to) {
    h->poisoned = true;
    return fail(KKM_ENCCL, "peer-memory a3/a4: a peer did not arrive within 600 s");
  }
  return KKM_OK;
}
