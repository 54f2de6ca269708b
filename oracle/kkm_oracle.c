/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of exact Kernel
 * K-means as arXiv 2601.17136 formulates it (§2.2, lines 86-171).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library. It shares no code, header, table or
 * constant with the CUDA path (paper_2601_17136_b200/), and the CUDA path never
 * calls it.
 *
 * Every function cites the passage it follows ("P:n" = PAPER.md line n;
 * "A<n>" = a reading of the paper listed in DESIGN.md §3). Loops follow the
 * paper's definitions directly; the only parallelism is OpenMP over output
 * rows, with every row summed sequentially in ascending index order, so
 * results are bitwise independent of the thread count.
 *
 * Parity pins: tests/test_oracle.py (hand-derived iterations, SPEC hand values,
 * Lloyd equivalence for the linear kernel, explicit-feature-map equivalence for
 * the degree-2 polynomial kernel, closed forms for the Gaussian kernel,
 * brute force over all labelings, monotonicity, identities, invariances).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_LINEAR 0
#define ORC_POLY 1
#define ORC_GAUSSIAN 2

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ELABEL 2
#define ORC_ENOMEM 3

/* kappa(x, y), Eq. (k) P:99-103 for the polynomial kernel, B = K for the linear
 * kernel, and the Gaussian kernel exp(-gamma ||x - y||^2) by reading A1
 * (the paper never defines it; BASELINE.json north_star requires it). Computed
 * "by definition", not by matrix identities: the Gaussian uses the direct
 * difference form, the polynomial an integer power by repeated multiplication. */
double orc_kappa(const float *x, const float *y, int64_t d, int kind, double gamma,
                 double coef0, int degree) {
  if (kind == ORC_GAUSSIAN) {
    double s = 0.0;
    for (int64_t t = 0; t < d; ++t) {
      double diff = (double)x[t] - (double)y[t];
      s += diff * diff;
    }
    return exp(-gamma * s);
  }
  double b = 0.0; /* B(i,j) = P(i,:) . P(j,:), Eq. (b) */
  for (int64_t t = 0; t < d; ++t) b += (double)x[t] * (double)y[t];
  if (kind == ORC_LINEAR) return b;
  double base = gamma * b + coef0, r = 1.0;
  for (int e = 0; e < degree; ++e) r *= base;
  return r;
}

static int check_kernel(int kind, double gamma, int degree) {
  if (kind == ORC_POLY && degree < 1) return ORC_EINVAL;
  if (kind == ORC_GAUSSIAN && gamma < 0.0) return ORC_EINVAL;
  if (kind < 0 || kind > 2) return ORC_EINVAL;
  return ORC_OK;
}

/* Rows `rows[0..nrows)` of K = kappa(P P^T) (Eqs. b, k), out is
 * nrows x n row-major. X is n x d fp32 row-major with leading dimension ldx. */
int orc_kernel_rows(const float *X, int64_t n, int64_t d, int64_t ldx, const int64_t *rows,
                    int64_t nrows, int kind, double gamma, double coef0, int degree,
                    double *out) {
  if (n < 1 || d < 1 || ldx < d || nrows < 0) return ORC_EINVAL;
  if (check_kernel(kind, gamma, degree)) return ORC_EINVAL;
  for (int64_t r = 0; r < nrows; ++r)
    if (rows[r] < 0 || rows[r] >= n) return ORC_EINVAL;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nrows; ++r) {
    const float *xi = X + rows[r] * ldx;
    for (int64_t j = 0; j < n; ++j)
      out[r * n + j] = orc_kappa(xi, X + j * ldx, d, kind, gamma, coef0, degree);
  }
  return ORC_OK;
}

/* diag K(i,i) for rows[0..nrows): the ||phi(x_i)||^2 term the paper's D omits
 * (reading A3). */
int orc_kernel_diag(const float *X, int64_t n, int64_t d, int64_t ldx, const int64_t *rows,
                    int64_t nrows, int kind, double gamma, double coef0, int degree,
                    double *diag) {
  if (n < 1 || d < 1 || ldx < d || check_kernel(kind, gamma, degree)) return ORC_EINVAL;
  for (int64_t r = 0; r < nrows; ++r) {
    if (rows[r] < 0 || rows[r] >= n) return ORC_EINVAL;
    const float *xi = X + rows[r] * ldx;
    diag[r] = orc_kappa(xi, xi, d, kind, gamma, coef0, degree);
  }
  return ORC_OK;
}

/* Round-robin initialisation, P:566 ("assigning points to clusters in a
 * round-robin fashion"), reading A5: cl(j) = j mod k over the global index. */
int orc_round_robin(int64_t n, int32_t k, int32_t *labels) {
  if (n < 1 || k < 1) return ORC_EINVAL;
  for (int64_t j = 0; j < n; ++j) labels[j] = (int32_t)(j % k);
  return ORC_OK;
}

/* |L_c| = number of points with cl(j) = c (the denominators of Eq. v). */
int orc_sizes(const int32_t *labels, int64_t n, int32_t k, int64_t *sizes) {
  if (n < 0 || k < 1) return ORC_EINVAL;
  for (int32_t c = 0; c < k; ++c) sizes[c] = 0;
  for (int64_t j = 0; j < n; ++j) {
    if (labels[j] < 0 || labels[j] >= k) return ORC_ELABEL;
    sizes[labels[j]] += 1;
  }
  return ORC_OK;
}

/* V(c, j) = 1/|L_c| if point j is in cluster c, else 0: Eq. (v).
 * Dense k x n, for the brute-force tests and for orc_E_dense. */
int orc_build_V(const int32_t *labels, int64_t n, int32_t k, double *V) {
  int64_t *sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  if (!sizes) return ORC_ENOMEM;
  int rc = orc_sizes(labels, n, k, sizes);
  if (rc == ORC_OK) {
    for (int64_t t = 0; t < (int64_t)k * n; ++t) V[t] = 0.0;
    for (int64_t j = 0; j < n; ++j) V[(int64_t)labels[j] * n + j] = 1.0 / (double)sizes[labels[j]];
  }
  free(sizes);
  return rc;
}

/* E = K V^T, Eq. (e), for the given K rows (nrows x n):
 * E(i,c) = sum_j K(i,j) V(c,j) = (1/|L_c|) sum_{j: cl(j)=c} K(i,j), the sum taken in
 * ascending j. Columns of empty clusters (|L_c| = 0, Eq. v undefined, reading A7)
 * are set to 0 and never used. */
int orc_E_rows(const double *Krows, int64_t nrows, int64_t n, const int32_t *labels, int32_t k,
               double *E) {
  if (nrows < 0 || n < 1 || k < 1) return ORC_EINVAL;
  int64_t *sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  if (!sizes) return ORC_ENOMEM;
  int rc = orc_sizes(labels, n, k, sizes);
  if (rc != ORC_OK) {
    free(sizes);
    return rc;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nrows; ++i) {
    for (int32_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int64_t j = 0; j < n; ++j)
        if (labels[j] == c) s += Krows[i * n + j];
      E[i * k + c] = sizes[c] > 0 ? s / (double)sizes[c] : 0.0;
    }
  }
  free(sizes);
  return ORC_OK;
}

/* z(i) = E(i, cl(i)), Eq. (z); c = V z, Eq. (c) P:144-146:
 * cnorm(c) = sum_i V(c,i) z(i) = (1/|L_c|) sum_{i in L_c} z(i) = ||mu_c||^2.
 * E_all is n x k (all points). Empty clusters get +inf (reading A7). */
int orc_cnorm(const double *E_all, const int32_t *labels, int64_t n, int32_t k, double *cnorm) {
  if (n < 1 || k < 1) return ORC_EINVAL;
  int64_t *sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  double *z = (double *)malloc(sizeof(double) * (size_t)n);
  if (!sizes || !z) {
    free(sizes);
    free(z);
    return ORC_ENOMEM;
  }
  int rc = orc_sizes(labels, n, k, sizes);
  if (rc == ORC_OK) {
    for (int64_t i = 0; i < n; ++i) z[i] = E_all[i * k + labels[i]]; /* mask, Eq. (z) */
    for (int32_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int64_t i = 0; i < n; ++i)
        if (labels[i] == c) s += z[i] / (double)sizes[c]; /* V z, Eq. (c) */
      cnorm[c] = sizes[c] > 0 ? s : INFINITY;
    }
  }
  free(sizes);
  free(z);
  return rc;
}

/* Objective, reading A8: J(cl) = sum_i ||phi(x_i) - mu_cl(i)||^2
 *                          = tr K - sum_{c: |L_c| > 0} |L_c| cnorm(c). */
int orc_objective(const double *diag, const int32_t *labels, int64_t n, int32_t k,
                  const double *cnorm, double *J) {
  if (n < 1 || k < 1) return ORC_EINVAL;
  int64_t *sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  if (!sizes) return ORC_ENOMEM;
  int rc = orc_sizes(labels, n, k, sizes);
  if (rc == ORC_OK) {
    double tr = 0.0, s = 0.0;
    for (int64_t i = 0; i < n; ++i) tr += diag[i];
    for (int32_t c = 0; c < k; ++c)
      if (sizes[c] > 0) s += (double)sizes[c] * cnorm[c];
    *J = tr - s;
  }
  free(sizes);
  return rc;
}

/* J of a given labelling straight from the points, for sizes where K cannot be stored (the
 * BASELINE configs 2-3 at full size). Reading A8 with the centroid of Eq. (c) (P:144-158,
 * mu_c = (1/|L_c|) sum_{j in L_c} phi(x_j)):
 *   J = sum_i ||phi(x_i) - mu_cl(i)||^2 = tr K - sum_{c: |L_c| > 0} (1/|L_c|) sum_{i in L_c} sum_{j in L_c} K(i,j)
 * (expanding the square; the mean of Eq. z/c is this double sum over |L_c|^2). kappa is the
 * definition (orc_kappa) and is symmetric exactly (same operations in the same order for (i,j) and
 * (j,i)), so each cluster's double sum is taken as sum_i K(i,i) + 2 sum_{i<j} K(i,j):
 *   W(i) = sum_{j in L_cl(i), j > i} K(i,j)   (ascending j; parallel over i only),
 *   T_c  = sum_{i in L_c} K(i,i) + 2 sum_{i in L_c} W(i)   (ascending i).
 * Every sum runs in a fixed order: the result is independent of the thread count.
 * labels: n int32 in [0,k). Out: *J. Cost sum_c |L_c|^2 / 2 kernel evaluations. */
int orc_objective_X(const float *X, int64_t n, int64_t d, int64_t ldx, const int32_t *labels, int32_t k,
                    int kind, double gamma, double coef0, int degree, double *J) {
  if (n < 1 || d < 1 || ldx < d || k < 1 || check_kernel(kind, gamma, degree)) return ORC_EINVAL;
  int64_t *sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k + 1));
  int64_t *members = (int64_t *)malloc(sizeof(int64_t) * (size_t)n); /* points of each cluster, ascending */
  int64_t *rank = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);    /* position of i in its cluster */
  double *W = (double *)malloc(sizeof(double) * (size_t)n);
  double *Kii = (double *)malloc(sizeof(double) * (size_t)n);
  int rc = (!sizes || !start || !members || !rank || !W || !Kii) ? ORC_ENOMEM : ORC_OK;
  if (rc == ORC_OK) rc = orc_sizes(labels, n, k, sizes);
  if (rc == ORC_OK) {
    start[0] = 0;
    for (int32_t c = 0; c < k; ++c) start[c + 1] = start[c] + sizes[c];
    for (int32_t c = 0; c < k; ++c) sizes[c] = 0; /* reused as fill counters */
    for (int64_t i = 0; i < n; ++i) {
      const int32_t c = labels[i];
      rank[i] = sizes[c];
      members[start[c] + sizes[c]++] = i;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
      const int32_t c = labels[i];
      const float *xi = X + i * ldx;
      Kii[i] = orc_kappa(xi, xi, d, kind, gamma, coef0, degree);
      double w = 0.0;
      for (int64_t p = start[c] + rank[i] + 1; p < start[c + 1]; ++p)
        w += orc_kappa(xi, X + members[p] * ldx, d, kind, gamma, coef0, degree);
      W[i] = w;
    }
    double tr = 0.0, within = 0.0;
    for (int64_t i = 0; i < n; ++i) tr += Kii[i];
    for (int32_t c = 0; c < k; ++c) {
      const int64_t sz = start[c + 1] - start[c];
      if (sz == 0) continue; /* empty clusters are excluded (reading A7) */
      double diag_sum = 0.0, off = 0.0;
      for (int64_t p = start[c]; p < start[c + 1]; ++p) {
        diag_sum += Kii[members[p]];
        off += W[members[p]];
      }
      within += (diag_sum + 2.0 * off) / (double)sz;
    }
    *J = tr - within;
  }
  free(sizes);
  free(start);
  free(members);
  free(rank);
  free(W);
  free(Kii);
  return rc;
}

/* D = -2E + C~, Eq. (d) P:160-167 (C~'s rows all equal c, Eq. ct), plus the
 * omitted K(i,i) (reading A3) for Dfull; row-wise argmin with the lowest index
 * winning ties (reading A6), computed on the shifted D. Empty clusters
 * (cnorm = +inf) are never chosen (reading A7). Dfull may be NULL. */
int orc_assign(const double *E, const double *diag, const double *cnorm, int64_t nrows,
               int32_t k, double *Dfull, int32_t *new_labels) {
  if (nrows < 0 || k < 1) return ORC_EINVAL;
  for (int64_t i = 0; i < nrows; ++i) {
    int32_t best = 0;
    double best_d = INFINITY;
    for (int32_t c = 0; c < k; ++c) {
      double dsh = isinf(cnorm[c]) ? INFINITY : -2.0 * E[i * k + c] + cnorm[c];
      if (Dfull) Dfull[i * k + c] = diag[i] + dsh;
      if (dsh < best_d) {
        best_d = dsh;
        best = c;
      }
    }
    new_labels[i] = best;
  }
  return ORC_OK;
}

/* The clustering loop of Alg. 1 on one process with K materialised
 * (n x n fp64): per iteration t, with the labels cl_t entering it (reading A14):
 * sizes, E = K V^T (Eq. e), z and c (Eqs. z, c), J_t (A8), D (Eq. d), argmin, V update.
 * Runs max_iter iterations (reading A4), optionally stopping when no label changes.
 * Outputs: labels (in/out, length n), J_trace[0..iters] (J_trace[iters] = J of the
 * final labels), changed_trace[0..iters), *iters_run. label_trace (optional,
 * (max_iter+1) x n) records cl_0 .. cl_iters. */
int orc_fit(const double *K, const double *diag, int64_t n, int32_t k, int32_t max_iter,
            int32_t stop_on_no_change, int32_t *labels, double *J_trace,
            int64_t *changed_trace, int32_t *iters_run, int32_t *label_trace) {
  if (n < 1 || k < 1 || k > n || max_iter < 0) return ORC_EINVAL;
  for (int64_t j = 0; j < n; ++j)
    if (labels[j] < 0 || labels[j] >= k) return ORC_ELABEL;
  double *E = (double *)malloc(sizeof(double) * (size_t)(n * k));
  double *cnorm = (double *)malloc(sizeof(double) * (size_t)k);
  int32_t *nl = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!E || !cnorm || !nl) {
    free(E);
    free(cnorm);
    free(nl);
    return ORC_ENOMEM;
  }
  int rc = ORC_OK;
  int32_t t = 0;
  if (label_trace) memcpy(label_trace, labels, sizeof(int32_t) * (size_t)n);
  for (t = 0; t < max_iter; ++t) {
    if ((rc = orc_E_rows(K, n, n, labels, k, E))) break;
    if ((rc = orc_cnorm(E, labels, n, k, cnorm))) break;
    if ((rc = orc_objective(diag, labels, n, k, cnorm, &J_trace[t]))) break;
    if ((rc = orc_assign(E, diag, cnorm, n, k, NULL, nl))) break;
    int64_t changed = 0;
    for (int64_t j = 0; j < n; ++j) changed += (nl[j] != labels[j]);
    changed_trace[t] = changed;
    memcpy(labels, nl, sizeof(int32_t) * (size_t)n);
    if (label_trace) memcpy(label_trace + (int64_t)(t + 1) * n, labels, sizeof(int32_t) * (size_t)n);
    if (stop_on_no_change && changed == 0) {
      ++t;
      break;
    }
  }
  if (rc == ORC_OK) { /* J of the final labels: one more E / c pass */
    rc = orc_E_rows(K, n, n, labels, k, E);
    if (rc == ORC_OK) rc = orc_cnorm(E, labels, n, k, cnorm);
    if (rc == ORC_OK) rc = orc_objective(diag, labels, n, k, cnorm, &J_trace[t]);
    *iters_run = t;
  }
  free(E);
  free(cnorm);
  free(nl);
  return rc;
}

/* Out-of-sample assignment (reading A21 extended): for each new point y,
 * the feature-space distance to each centroid of the training labels cl,
 *   D(y, c) = kappa(y, y) - (2/|L_c|) sum_{j in L_c} kappa(y, x_j) + c(c),
 * the same Eq. (d) with E(y, c) = (1/|L_c|) sum_{j in L_c} kappa(y, x_j) (Eq. e for
 * a row of K(Y, X)) and c = ||mu_c||^2 of the training clustering (Eq. c). Lowest index wins
 * ties, empty clusters are never chosen (A6, A7). cnorm: the k centroid norms (e.g. from
 * orc_cnorm on the training E). Y is m x d fp32 row-major (ld d). Dfull may be NULL. */
int orc_predict(const float *X, int64_t n, const float *Y, int64_t m, int64_t d, const int32_t *labels,
                int32_t k, const double *cnorm, int kind, double gamma, double coef0, int degree,
                int32_t *out_labels, double *Dfull) {
  if (n < 1 || m < 0 || d < 1 || k < 1 || check_kernel(kind, gamma, degree)) return ORC_EINVAL;
  int64_t *sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  if (!sizes) return ORC_ENOMEM;
  int rc = orc_sizes(labels, n, k, sizes);
  if (rc != ORC_OK) {
    free(sizes);
    return rc;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    const float *y = Y + i * d;
    const double kyy = orc_kappa(y, y, d, kind, gamma, coef0, degree);
    int32_t best = 0;
    double best_d = INFINITY;
    for (int32_t c = 0; c < k; ++c) {
      double dsh = INFINITY;
      if (sizes[c] > 0) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j)
          if (labels[j] == c) s += orc_kappa(y, X + j * d, d, kind, gamma, coef0, degree);
        dsh = -2.0 * (s / (double)sizes[c]) + cnorm[c];
      }
      if (Dfull) Dfull[i * k + c] = kyy + dsh;
      if (dsh < best_d) {
        best_d = dsh;
        best = c;
      }
    }
    out_labels[i] = best;
  }
  free(sizes);
  return ORC_OK;
}

/* K-means++ seeding in feature space ("K-means++ ... future work";
 * Arthur & Vassilvitskii's D^2 sampling with ||phi(x) - phi(c)||^2 = K(x,x) - 2 K(x,c) + K(c,c)).
 * u[0..k-1]: uniforms in [0,1) supplied by the caller (the random draws are inputs).
 *   c_0 = floor(u[0] * n);
 *   for t = 1..k-1: D(x) = min_{s<t} dist(x, c_s); c_t = the smallest index i with
 *     sum_{j<=i} D(j) > u[t] * sum_j D(j)   (inverse CDF, sums in index order, fp64);
 *     if every D is 0 (fewer than t distinct points), c_t = c_{t-1}.
 *   labels(x) = the lowest s attaining min_s dist(x, c_s) (A6).
 * centers: k int64 out; labels: n int32 out. */
int orc_kmeanspp(const float *X, int64_t n, int64_t d, int32_t k, int kind, double gamma, double coef0, int degree,
                 const double *u, int64_t *centers, int32_t *labels) {
  if (n < 1 || d < 1 || k < 1 || k > n || check_kernel(kind, gamma, degree)) return ORC_EINVAL;
  double *D = (double *)malloc(sizeof(double) * (size_t)n);
  if (!D) return ORC_ENOMEM;
  int64_t c = (int64_t)(u[0] * (double)n);
  if (c >= n) c = n - 1;
  centers[0] = c;
  for (int32_t t = 0; t < k; ++t) {
    const float *xc = X + centers[t] * d;
    const double kcc = orc_kappa(xc, xc, d, kind, gamma, coef0, degree);
    for (int64_t i = 0; i < n; ++i) {
      const float *xi = X + i * d;
      const double dist = orc_kappa(xi, xi, d, kind, gamma, coef0, degree) -
                          2.0 * orc_kappa(xi, xc, d, kind, gamma, coef0, degree) + kcc;
      if (t == 0 || dist < D[i]) {
        D[i] = dist;
        labels[i] = t;
      }
    }
    if (t + 1 == k) break;
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += D[i] > 0.0 ? D[i] : 0.0;
    int64_t pick = centers[t];
    if (total > 0.0) {
      const double target = u[t + 1] * total;
      double run = 0.0;
      pick = -1;
      for (int64_t i = 0; i < n; ++i) {
        run += D[i] > 0.0 ? D[i] : 0.0;
        if (run > target) {
          pick = i;
          break;
        }
      }
      if (pick < 0) {  /* rounding at the top end: the last point with D > 0 */
        for (int64_t i = n - 1; i >= 0; --i)
          if (D[i] > 0.0) {
            pick = i;
            break;
          }
      }
    }
    centers[t + 1] = pick;
  }
  free(D);
  return ORC_OK;
}
