/*
 * kkm.h -- C-ABI of the B200-native exact Kernel K-means hot path.
 *
 * Method: arXiv 2601.17136 ("PAPER.md"), §2.2. One clustering
 * iteration computes, for the current assignment cl(.) and its n x k
 * indicator V (Eq. v, V(c,j) = 1/|L_c| if cl(j) = c):
 *   (a1) K = kappa(P P^T)               Eqs. (b), (k)
 *   (a2) E = K V^T                      Eq.  (e)
 *   (a3) z(i) = E(i, cl(i)); c = V z    Eqs. (z), (c)
 *   (a4) D = -2E + C~; cl <- argmin_c D(i, c); V <- V(cl)   Eq. (d)
 * in a loop (Alg. 1). All arithmetic runs in the CUDA kernels of
 * libkkm.so (sm_100a); this header and the ctypes binding only marshal.
 * Beyond the paper's loop: K's symmetry is exploited (f1,
 * kkm_params.symmetric); the cluster sums can be updated by the moved points
 * only and the labels seeded by K-means++ (f3, kkm_params.incremental,
 * kkm_seed_kmeanspp); new points can be assigned to fitted clusters (f4,
 * kkm_predict).
 *
 * Conventions
 *   - Every function returns an int status (KKM_OK = 0); on failure
 *     kkm_last_error() returns a thread-local message. After KKM_ECUDA or
 *     KKM_ENCCL a handle is poisoned: destroy it (and abort the communicator).
 *   - Handles are not thread-safe; use one handle per (rank, stream).
 *   - "device" pointers are CUDA global memory of the current device;
 *     pointers documented "host or device" are classified with
 *     cudaPointerGetAttributes and copied with cudaMemcpyAsync on the handle's
 *     stream (pinned host memory is the fast path).
 *   - Matrices are row-major. n = number of points, d = features, k = clusters.
 *   - Multi-GPU: ranks own contiguous point blocks [kkm_shard_begin(r),
 *     kkm_shard_begin(r+1)), the paper's 1D column blocks of K (
 *     K is symmetric so row blocks of K are its column blocks). Collective
 *     functions must be called by every rank of the communicator.
 * Readings of the paper that the semantics depend on:
 *   A1 Gaussian kernel exp(-gamma ||x-y||^2); A3 distances add K(i,i);
 *   A4 fixed max_iter (+ optional stop when nothing changes); A5 round-robin
 *   init cl(j) = j mod k on the global index; A6 lowest cluster index wins
 *   ties; A7 empty clusters get +inf distance and stay empty; A8 objective
 *   J = tr K - sum_c |L_c| ||mu_c||^2; A14 iteration t uses the labels entering it.
 */
#ifndef KKM_H
#define KKM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define KKM_OK 0
#define KKM_EINVAL 1  /* bad argument (sizes, params, null pointer, rank range)  */
#define KKM_ELABEL 2  /* an init / set label is outside [0, k)                  */
#define KKM_ENOMEM 3  /* workspace too small, or MATERIALIZE does not fit         */
#define KKM_EUNSUP 4  /* valid but unsupported combination                       */
#define KKM_ECUDA 5   /* CUDA runtime/driver error (handle poisoned)             */
#define KKM_ENCCL 6   /* NCCL error (handle poisoned)                           */
#define KKM_ESTATE 7  /* call out of order (e.g. fit on a poisoned handle)       */

/* ---- kernel function kappa (A1) ------------------------------ */
#define KKM_KERNEL_LINEAR 0   /* kappa(x,y) = x.y    */
#define KKM_KERNEL_POLY 1     /* kappa(x,y) = (gamma x.y + coef0)^degree (Eq. k) */
#define KKM_KERNEL_GAUSSIAN 2 /* kappa(x,y) = exp(-gamma ||x - y||^2)  (A1)     */

/* ---- where K lives ------------------------------------------------------ */
#define KKM_PATH_AUTO 0        /* materialise if the K block fits 160 GB, else stream         */
#define KKM_PATH_MATERIALIZE 1 /* K rows of this rank stored fp32 in HBM once               */
#define KKM_PATH_STREAM 2      /* K tiles recomputed every iteration by the fused tensor-core
                                  kernel and reduced in TMEM/registers; K never stored.
                                  Needs FP16X3/BF16X3 (else KKM_EUNSUP). k > 16: one launch
                                  per group of 16 clusters (host reads k+1 ints per iter.) */

/* ---- symmetric storage of a materialised K (f1) ---------------------------- */
#define KKM_SYM_AUTO 0
#define KKM_SYM_OFF 1
#define KKM_SYM_ON 2
#define KKM_KSTORE_AUTO 0
#define KKM_KSTORE_FP32 1
#define KKM_KSTORE_FP16 2
#define KKM_KSTORE_FP16X2 3

/* ---- precision of the a1 contraction (reading A9) ----------------------- */
#define KKM_PREC_BF16X3 0    /* tcgen05 kind::f16: hi*hi + hi*lo + lo*hi, bf16 split of x;
                                 product error ~2^-17 |x||y|                               */
#define KKM_PREC_FP32_SIMT 1 /* fp32 CUDA-core FMA (correctness baseline)                 */
#define KKM_PREC_FP16X3 2    /* tcgen05 kind::f16, 3 MMAs on an fp16 split of 2^e_i x_i (per-row
                                power-of-two scale); product error ~2^-21 |x||y|; default */

/* ---- kkm_debug_read selectors --------------------------------------------*/
#define KKM_DBG_E 0      /* double [n_local x k]: E of the last iteration       */
#define KKM_DBG_CNORM 1  /* double [k]: c (centroid norms ||mu_c||^2), +inf empty */
#define KKM_DBG_SIZES 2  /* int32  [k]: |L_c| of the labels entering the last it. */
#define KKM_DBG_DIAG 3   /* double [n_local]: K(i,i)                              */
#define KKM_DBG_DFULL 4  /* double [n_local x k]: K_ii - 2E + c of the last iter.  */
#define KKM_DBG_LABELS_PREV 5 /* int32 [n]: labels entering the last iteration     */

/* ---- phase timers (kkm_phase_ms) ----------------------------------------- */
#define KKM_PH_INIT_PREP 0  /* X copy/gather, norms, bf16 split, diag           */
#define KKM_PH_INIT_GEMM 1  /* a1: K = kappa(X X^T) materialisation             */
#define KKM_PH_SPMM 2       /* a2 per fit (sum over iterations)                 */
#define KKM_PH_CNORM 3      /* a3 incl. its collective; where a3 and a4 run as ONE
                               launch (single-CTA small n; the grid-wide update of
                               the 16-bit band paths, k <= 64) it includes a4      */
#define KKM_PH_ASSIGN 4     /* a4 incl. the labels allgather (0 when fused into a3) */
#define KKM_PH_A2_KERNEL 5  /* the dominant a2 kernel alone (spmm_tc over the 16-bit bands /
                               spmm_sym / spmm_onehot / spmm_group / the streaming kernels),
                               summed over the loop's launches */
#define KKM_NPHASES 6

typedef struct kkm_params {
  int32_t kind;            /* KKM_KERNEL_*                                         */
  double gamma;            /* poly: > 0; Gaussian: >= 0; ignored for linear        */
  double coef0;            /* poly offset c of Eq. (k)                             */
  int32_t degree;          /* poly degree >= 1                                    */
  int32_t k;               /* clusters, 1 <= k <= min(n, 900) (KKM_EUNSUP above 900)  */
  int32_t max_iter;        /* iterations per kkm_fit call, >= 0 (100)      */
  int32_t stop_on_no_change; /* 1: stop early when no label changes (A4)          */
  int32_t path;            /* KKM_PATH_*                                           */
  int32_t precision;       /* KKM_PREC_*                                           */
  int32_t timing;          /* 1: record per-phase CUDA-event times (kkm_phase_ms) */
  int32_t grid_rows;       /* 1.5D process grid pr x (nranks/pr), column-major ranks
                              (P:604); 0 or 1 = the 1D algorithm (Alg. 1). Must divide
                              nranks. See kkm_init.                                   */
  int32_t symmetric;       /* f1, 1D runs: compute / store only the upper triangle of K (half
                              the K bytes and GEMM flops when materialised -- k <= 32 with
                              16-bit band storage, k <= 16 with fp32 bands -- and half the MMA
                              work when streaming, any k).
                              KKM_SYM_AUTO (0): streaming always; materialised when
                              n >= 8192 (below, the extra kernels cost more than the
                              halved K read saves). KKM_SYM_ON (2): whenever eligible.
                              KKM_SYM_OFF (1): never.                                 */
  int32_t incremental;     /* f3 (time to solution). 0: recompute S = K V^T every
                              iteration (Alg. 1; default). 1: after an iteration in
                              which m <= n/16 labels changed, update S of the own rows
                              by the moved points only -- the fused streaming kernel
                              over them, added with their new and subtracted with
                              their old label (~4 m n d flops instead of a full pass;
                              exact up to rounding, S kept in fp64); otherwise a full
                              pass. 1D and a tensor-core precision only (KKM_EUNSUP). */
  int32_t kstore;          /* f4, materialised K storage of the f1 bands.
                              KKM_KSTORE_FP32 (1): fp32 (the paper's precision), a2 by
                              the one-hot FFMA2 kernel (sym.cuh).
                              KKM_KSTORE_FP16X2 (3): two fp16 planes hi = RN(K 2^e),
                              lo = RN(K 2^e - hi), with 2^e the largest power of two such that
                              a bound on |K| times 2^e is <= 60000 (linear: max ||x||^2; poly:
                              (gamma max ||x||^2 + |coef0|)^degree; Gaussian: 1): 4 bytes per
                              value like fp32, relative error <= 2^-21 + 2^-24 (fp32-class), and a2 on
                              the tensor cores (spmm_tc.cuh) with S summed in int64 fixed point.
                              KKM_KSTORE_FP16 (2): the hi plane only -- half the bytes, each
                              value rounded to 2^-11 relative (DESIGN A27 bounds E / D / J).
                              KKM_KSTORE_AUTO (0, default): FP16X2 whenever the run stores the
                              f1 bands with a tensor-core precision (1D, k <= 32; see
                              `symmetric`), else FP32.
                              FP16 and FP16X2 need a tensor-core precision and a materialised
                              1D run with k <= 32 and symmetric != OFF (they imply the f1 bands
                              for any n); else KKM_EUNSUP.                                */
  int32_t reserved[2];     /* must be zero                                         */
} kkm_params;

typedef struct kkm_ctx *kkm_handle;

/* ---- planner introspection (kkm_plan_query) ------------------------------- */
#define KKM_LAYOUT_FULL 0         /* K rows of the A set x the B set, materialised (Alg. 1 / Alg. 2)  */
#define KKM_LAYOUT_STREAM 1       /* the same tile recomputed per iteration, K never stored             */
#define KKM_LAYOUT_SYM_BANDS 2    /* f1: upper-triangle bands of 1024 rows, fp32 (sym.cuh)             */
#define KKM_LAYOUT_SYM_BANDS16 3  /* f1: the bands as 16-bit planes in pieces of <= 1024 rows (spmm_tc) */
#define KKM_LAYOUT_SYM_STREAM 4   /* f1: upper-triangle tiles of the label-sorted K, recomputed (ssym) */
#define KKM_XCHG_NONE 0           /* one rank                                                           */
#define KKM_XCHG_PARTIALS 1       /* per iteration: allgather of (k+1) partials, labels, sizes (1D/1.5D) */
#define KKM_XCHG_S_ALLREDUCE 2    /* per iteration: one allreduce of S (n x k), a3/a4 replicated; opt-in
                                     KKM_LSA=1 (16-bit bands, k <= 64, <= 8 ranks on one NVLink
                                     domain): no allreduce -- the fused a3/a4 kernel reads every
                                     rank's S from NCCL symmetric windows and splits the rows over
                                     the ranks                                     */
#define KKM_XCHG_S_REDUCE_SCATTER 3 /* per iteration: reduce-scatter of S to the 1D blocks + partials   */
typedef struct kkm_plan_info {
  int32_t path;          /* effective KKM_PATH_MATERIALIZE or KKM_PATH_STREAM                    */
  int32_t layout;        /* KKM_LAYOUT_*                                                          */
  int32_t exchange;      /* KKM_XCHG_* (before the opt-in peer-memory variant, see kkm_init)      */
  int32_t grid_rows, grid_cols;
  int32_t reserved;
  int64_t row0, nloc;    /* the rank's own 1D block of points                                     */
  int64_t a0, nA, b0, nB;/* KKM_LAYOUT_FULL / STREAM: the K tile's rows (A set) and columns (B set) */
  int64_t npieces;       /* rectangles of K (or of the label-sorted K) this rank computes           */
  int64_t ws_bytes;      /* = kkm_workspace_size                                                  */
} kkm_plan_info;

/* Fills *p with defaults: polynomial kernel (gamma 1, coef0 1, degree 2, the paper's
 * benchmark kernel P:640), k = 2, max_iter = 100, AUTO, FP16X3. */
int kkm_default_params(kkm_params *p);

/* First row owned by `rank` of `nranks` for n points: min(n, rank * ceil(n / nranks)).
 * Every rank but the last owns exactly ceil(n / nranks) rows (the last may own fewer,
 * or none), so labels allgather in place without compaction. rank == nranks gives n.
 * Pure; no CUDA. Returns -1 on bad arguments. */
int64_t kkm_shard_begin(int64_t n, int32_t rank, int32_t nranks);

/* Bytes of device workspace kkm_init needs for this rank (pure; no CUDA).
 * Includes the materialised K block when the effective path is MATERIALIZE: the
 * rank's n_local x ceil32(n) fp32 rows, or with symmetric storage (KKM_SYM_AUTO, 1D,
 * k <= 32 for 16-bit bands) its share of the upper-triangle bands (1024 rows x ceil(n - 1024 I)
 * columns each, bands spread over the ranks by area): ~n^2/(2P) floats. */
int kkm_workspace_size(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks,
                       size_t *bytes);

/* Pure planner introspection (no CUDA): what rank `rank` of `nranks` computes and exchanges, so the
 * decomposition can be checked for any P on a host without GPUs (tests/test_plan_cover.py).
 *   info:   out (required).
 *   pieces: NULL, or host int64[cap][5]: the rank's rectangles (r0, nr, c0, nc, cdiag) of K in
 *           global indices -- of the label-sorted K for KKM_LAYOUT_SYM_STREAM. The rank adds the
 *           row part S(i, cl(j)) += K(i, j) for every (i, j) of the rectangle and, for columns
 *           j >= cdiag, also the column part S(j, cl(i)) += K(i, j) (symmetry); cdiag = n for
 *           layouts without column parts. At most cap rectangles are written; info->npieces is the
 *           total. Same errors as kkm_workspace_size. */
int kkm_plan_query(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks, kkm_plan_info *info,
                   int64_t *pieces, int64_t cap);

/* Creates a handle and runs the one-time part of the path.
 * Sharding (P = nranks, B = ceil(n / P), pr = grid_rows, pc = P / pr, rank = i + j * pr):
 *   - rank r owns the 1D block [r B, (r+1) B) of points (its labels, E rows, distances);
 *   - it computes E partials for the points of column block j = 1D blocks [j pr, (j+1) pr)
 *     against the points of row block i = 1D blocks [i pc, (i+1) pc) (K_ij of the 2D grid,
 *     P:440-487), then a ReduceScatter over the pr ranks of process column j leaves each rank
 *     the full E of its own 1D block (the paper's column-split Reduce-Scatter).
 *   pr = 1 is the 1D algorithm (column block = own block, row block = all points).
 *   X_local:  rows [kkm_shard_begin(rank), kkm_shard_begin(rank+1)) of X, fp32,
 *             row-major with leading dimension ldx >= d; host or device. It is
 *             read during the call only (copied into the workspace). With
 *             nranks > 1 the blocks are allgathered over `nccl_comm` (Alg. 1
 *             line 1).
 *   init_labels: NULL -> round-robin (A5); else n int32 in [0,k) (host or device,
 *             identical on every rank).
 *   workspace: device buffer of >= kkm_workspace_size bytes, 256-B aligned,
 *             owned by the caller, must outlive the handle.
 *   cuda_stream: cudaStream_t (NULL = legacy default stream).
 *   nccl_comm:   ncclComm_t of nranks ranks (NULL iff nranks == 1). Borrowed.
 * Computes norms, the 16-bit hi/lo split of X (fp16 with a per-row power-of-two scale for
 * FP16X3, the default; bf16 for BF16X3), diag K(i,i) and, when materialising, K[rows, :] with
 * the a1 GEMM + kappa epilogue. Collective. */
int kkm_init(kkm_handle *out, const kkm_params *p, const float *X_local, int64_t n, int64_t d,
             int64_t ldx, int32_t rank, int32_t nranks, const int32_t *init_labels,
             void *workspace, size_t ws_bytes, void *cuda_stream, void *nccl_comm);

/* Runs up to max_iter iterations from the current labels (repeated calls resume).
 *   iters_run:   host, out (may be NULL).
 *   J_trace:     host, length >= max_iter + 1, or NULL. J_trace[t] = J of the
 *                labels entering iteration t; J_trace[iters_run] = J of the final
 *                labels (A8). fp64.
 *   changed:     host, length >= max_iter, or NULL: #labels changed by iteration t.
 * Synchronises the stream once at the end (and once per iteration when
 * stop_on_no_change is set). Collective. */
int kkm_fit(kkm_handle h, int32_t *iters_run, double *J_trace, int64_t *changed);

/* Copies the current labels of all n points (identical on every rank) into
 * labels_out (host or device, n int32). Synchronises the stream. */
int kkm_assign(kkm_handle h, int32_t *labels_out);

/* J of the current labels (one E/c pass; fp64). Collective. */
int kkm_objective(kkm_handle h, double *J);

/* Replaces the current labels (n int32 in [0,k), host or device, identical on
 * every rank): used for teacher-forced parity and for resuming. KKM_ELABEL if any
 * label is outside [0, k); the handle then keeps its current labels. */
int kkm_set_labels(kkm_handle h, const int32_t *labels);

/* Out-of-sample assignment: assigns m new points y to the
 * clusters of the CURRENT labels with the same distance as an iteration,
 *   D(y, c) = kappa(y, y) - (2/|L_c|) sum_{j in L_c} kappa(y, x_j) + c(c)
 * (Eq. d of PAPER.md §2.2 P:160-168 with Eq. e for a row of K(Y, X); c = ||mu_c||^2,
 * Eq. c), lowest index on ties, empty clusters never chosen (A6, A7). K(Y, X) is
 * never stored: the fused streaming kernel runs with A = Y, B = X sorted by label.
 *   Y:          host or device, m x d fp32 row-major, row pitch ldy >= d floats.
 *   labels_out: host or device, m int32 (out).
 *   D_out:      host or device, m x k fp64 (out), or NULL. +inf for empty clusters.
 *   workspace:  device scratch of >= kkm_predict_workspace_size(h, m) bytes, 256-B
 *               aligned, owned by the caller; or NULL: the library then takes it from
 *               the stream-ordered allocator for this call (slower: the pages are
 *               mapped on every call; KKM_ENOMEM if that fails).
 * Local to the calling rank (every rank holds all of X and the labels). Needs
 * c of the current labels: valid after kkm_fit or kkm_objective; otherwise one
 * kkm_objective pass is run first when nranks == 1 and KKM_ESTATE is returned
 * when nranks > 1 (that pass is collective). KKM_EUNSUP for FP32_SIMT handles.
 * Synchronises the stream. */
int kkm_predict(kkm_handle h, const float *Y, int64_t m, int64_t ldy, int32_t *labels_out, double *D_out,
                void *workspace, size_t ws_bytes);

/* Bytes of device scratch kkm_predict needs for m points (about m*(4*ld + 4*dp + 8*k*splits)
 * + n*4*dp for materialising handles; ld = d rounded up to 4, dp = d rounded up to 64). */
int kkm_predict_workspace_size(kkm_handle h, int64_t m, size_t *bytes);

/* K-means++ seeding in feature space (the paper's P:567 leaves it as
 * future work): c_0 = floor(u[0] n); then c_t = the smallest index i whose running sum of
 * D = min_{s<t} ||phi(x) - phi(c_s)||^2 = K(x,x) - 2 K(x,c_s) + K(c_s,c_s) exceeds u[t] * sum D
 * (D^2 sampling; the previous center again if every D is 0). Distances are evaluated in fp64
 * from the fp32 points. The labels become the lowest-index nearest center of every point
 * (as kkm_set_labels: replaces the current labels).
 *   u:           host, k uniforms in [0, 1) -- the random draws are the caller's.
 *   centers_out: host or device, k int64 point indices (out), or NULL.
 * Every rank computes the same result locally (X is replicated); no communication.
 * Temporary device memory ~12 n bytes (stream-ordered). Synchronises the stream. */
int kkm_seed_kmeanspp(kkm_handle h, const double *u, int64_t *centers_out);

/* Copies an internal array of the last iteration (selectors KKM_DBG_*) to dst
 * (host or device). Synchronises. Test hook. */
int kkm_debug_read(kkm_handle h, int32_t what, void *dst);

/* Evaluates K[i0:i0+m, j0:j0+nc] (global indices, fp32) with the SAME a1
 * mainloop + kappa epilogue the handle uses, into dst (host or device, m x nc
 * row-major). Test hook for kernel-value parity. Independent of the stored K. */
int kkm_kernel_tile(kkm_handle h, int64_t i0, int64_t j0, int32_t m, int32_t nc, float *dst);

/* Reads back row i (global index) of the K this rank STORED when materialising, as the a2
 * kernels will read it: dst (host) receives n doubles, dst[j] = the stored K(i, j) (fp32 bands
 * or full rows as stored; 16-bit bands: (hi + lo) * 2^-e, or hi * 2^-e for FP16) for every
 * column j the rank stores for row i -- the f1 band piece holding row i stores j >= the band
 * start, full K rows the rank's B set -- and NaN for the others. KKM_ESTATE when the handle
 * streams (nothing stored) or the rank does not store row i. Synchronises. Test hook for the
 * kernel-value parity of the storage formats (DESIGN A27). */
int kkm_stored_k_row(kkm_handle h, int64_t i, double *dst);

/* Per-phase milliseconds (KKM_NPHASES floats, host) accumulated since init
 * when params.timing = 1; zeros otherwise. */
int kkm_phase_ms(kkm_handle h, float *ms);

/* Number of CUDA kernels this library launched on the handle's stream since
 * init (for bench.py's gpu_launches). */
int kkm_launch_count(kkm_handle h, int64_t *count);

/* Frees the handle (workspace and communicator stay the caller's). With the opt-in peer-memory
 * update (KKM_LSA=1, see KKM_XCHG_S_ALLREDUCE) it also deregisters the NCCL symmetric window,
 * which is collective: every rank destroys its handle, before kkm_comm_destroy. */
int kkm_destroy(kkm_handle h);

/* Thread-local message for the last non-zero status of this thread. */
const char *kkm_last_error(void);

/* NCCL bootstrap: rank 0 calls kkm_get_unique_id, broadcasts the 128 bytes
 * (e.g. with torch.distributed), every rank calls kkm_comm_init with the
 * current device set. kkm_comm_destroy finalises. */
int kkm_get_unique_id(char id[128]);
int kkm_comm_init(void **comm, int32_t nranks, int32_t rank, const char id[128]);
int kkm_comm_destroy(void *comm);

#ifdef __cplusplus
}
#endif
#endif /* KKM_H */
