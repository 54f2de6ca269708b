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

// After a synchronised a3 on the peer path: a finalize that gave up waiting for a peer poisons the
// handle (KKM_ENCCL: the exchange failed) instead of trapping the context.
static int check_p2p(kkm_ctx *h) {
  if (!h->p2p) return KKM_OK;
  int to = 0;
  CK(cudaMemcpy(&to, h->xbuf + h->xflag_off + 64, 4, cudaMemcpyDeviceToHost));
  if (to) {
    h->poisoned = true;
    return fail(KKM_ENCCL, "peer-memory S exchange: a peer's flag did not arrive within %.0f s",
                (double)h->p2p_timeout_ns * 1e-9);
  }
  return KKM_OK;
}

// Peer-memory exchange of S for the replicated a3 (16-bit bands, several ranks, §6): an own
// cudaMalloc'd buffer [2 epochs of k x npad int64 | epoch flag | peer table], its IPC handle
// allgathered over NCCL and the peers' buffers opened here. All ranks must agree: the outcome is
// allreduced (min) and any failure leaves every rank on the NCCL allreduce path. Collective.
static int setup_p2p(kkm_ctx *h) {
  const Plan &P = h->P;
  const size_t sbytes = (size_t)P.npad * P.k * 8;
  const size_t xbytes = 2 * sbytes + 256 + (size_t)P.nranks * 8;
  int ok = 1;
  char *dh = nullptr;
  std::vector<char> hs((size_t)64 * P.nranks);
  std::vector<const uint8_t *> bases((size_t)P.nranks, nullptr);
  if (cudaMalloc(&h->xbuf, xbytes) != cudaSuccess) {
    h->xbuf = nullptr;
    ok = 0;
  }
  if (ok && cudaMemset(h->xbuf, 0, xbytes) != cudaSuccess) ok = 0;
  cudaIpcMemHandle_t mine;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (ok && cudaIpcGetMemHandle(&mine, h->xbuf) != cudaSuccess) ok = 0;
  if (cudaMalloc(&dh, hs.size() + 8) != cudaSuccess) return fail(KKM_ECUDA, "cudaMalloc (IPC handles) failed");
  if (ok) CK(cudaMemcpy(dh + 64 * (size_t)P.rank, &mine, 64, cudaMemcpyHostToDevice));
  CKN(ncclAllGather(dh + 64 * (size_t)P.rank, dh, 64, ncclChar, h->comm, h->st));
  CK(cudaMemcpyAsync(hs.data(), dh, hs.size(), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (ok) {
    for (int r = 0; r < P.nranks; ++r) {
      if (r == P.rank) {
        bases[(size_t)r] = h->xbuf;
        continue;
      }
      cudaIpcMemHandle_t hr;
      std::memcpy(&hr, hs.data() + 64 * (size_t)r, 64);
      void *q = nullptr;
      if (cudaIpcOpenMemHandle(&q, hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      h->xpeers.push_back(q);
      bases[(size_t)r] = (const uint8_t *)q;
    }
  }
  // every rank on the same path
  int *dok = (int *)(dh + hs.size());
  CK(cudaMemcpy(dok, &ok, 4, cudaMemcpyHostToDevice));
  CKN(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, h->comm, h->st));
  CK(cudaMemcpyAsync(&ok, dok, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  cudaFree(dh);
  if (ok) {
    h->xtable = (const uint8_t **)(h->xbuf + 2 * sbytes + 256);
    h->xflag_off = 2 * sbytes;
    CK(cudaMemcpy((void *)h->xtable, bases.data(), (size_t)P.nranks * 8, cudaMemcpyHostToDevice));
    h->p2p = true;
    return KKM_OK;
  }
  for (void *q : h->xpeers) cudaIpcCloseMemHandle(q);
  h->xpeers.clear();
  if (h->xbuf) cudaFree(h->xbuf);
  h->xbuf = nullptr;
  cudaGetLastError();
  return KKM_OK;  // NCCL allreduce path
}

