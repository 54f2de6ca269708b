"""CPU model of the fp16x3 tensor-core accumulation bias (DESIGN A9) and of the remedies, on the
HAR / MNIST recipes: every tcgen05 MMA (K = 16) is modelled as the exact sum of its 16 products
added to the fp32 accumulator and truncated toward zero (RZ), in the kernel's issue order per
k-step: corr += hi*lo, corr += lo*hi, main += hi*hi. Reports the mean signed / max relative error
of b = x.y and the J error (oracle fp64 J of the same labels from the modelled K) for
  S0  the current kernels (one main + one correction accumulator over all of d),
  S1  S0 + Gaussian r^2 from tensor-core self dot products (n_i = the kernel's own b_ii),
  S2c S0 with the main accumulator restarted every c K-blocks of 64 (drained with fp32 RN adds).
Not part of the product; a design study for the precision item.

  python tools/bias_model.py --config har200k --n 1500
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def rz32(x):
    f = x.astype(np.float32)
    f64 = f.astype(np.float64)
    over = np.abs(f64) > np.abs(x)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f


def split_fp16(X):
    """prep_rows_kernel split 2: per-row power-of-two s with max|x s| in [2^13, 2^14)."""
    amax = np.abs(X).max(axis=1)
    e = np.frexp(amax)[1]
    s = np.ldexp(1.0, 14 - e).astype(np.float32)
    xs = X.astype(np.float32) * s[:, None]
    hi = xs.astype(np.float16)
    lo = (xs - hi.astype(np.float32)).astype(np.float16)
    return hi.astype(np.float64), lo.astype(np.float64), (1.0 / s).astype(np.float32)


def tc_dot(hi, lo, chain_kb=0, merged=False):
    """Modelled main and correction accumulators of hi/lo x hi/lo^T (n x n). merged: the hi*lo and
    lo*hi MMAs go into the main accumulator too (one accumulator per chain)."""
    n, d = hi.shape
    dp = -(-d // 64) * 64
    H = np.zeros((n, dp))
    L = np.zeros((n, dp))
    H[:, :d] = hi
    L[:, :d] = lo
    main = np.zeros((n, n), dtype=np.float32)
    corr = np.zeros((n, n), dtype=np.float32)
    drained = np.zeros((n, n), dtype=np.float32)
    for ks in range(dp // 16):
        sl = slice(16 * ks, 16 * ks + 16)
        if merged:
            main = rz32(main.astype(np.float64) + H[:, sl] @ L[:, sl].T)
            main = rz32(main.astype(np.float64) + L[:, sl] @ H[:, sl].T)
        else:
            corr = rz32(corr.astype(np.float64) + H[:, sl] @ L[:, sl].T)
            corr = rz32(corr.astype(np.float64) + L[:, sl] @ H[:, sl].T)
        main = rz32(main.astype(np.float64) + H[:, sl] @ H[:, sl].T)
        if chain_kb and (ks + 1) % (4 * chain_kb) == 0:  # drain: fp32 RN add, restart the chain
            drained = (drained + main).astype(np.float32)
            main[:] = 0
    return (drained + main).astype(np.float32), corr


def kmat(b, rs, X, kind, gamma, coef0, degree, self_norms=False):
    bb = (b.astype(np.float64)) * rs[:, None] * rs[None, :]
    if kind == oracle.GAUSSIAN:
        if self_norms:
            nrm = np.diag(bb).copy()
        else:
            nrm = np.sum(X.astype(np.float64) ** 2, axis=1).astype(np.float32).astype(np.float64)
        r2 = np.maximum(nrm[:, None] + nrm[None, :] - 2 * bb, 0)
        np.fill_diagonal(r2, 0)
        return np.exp(-gamma * r2)
    if kind == oracle.POLY:
        return (gamma * bb + coef0) ** degree
    return bb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="har200k")
    ap.add_argument("--n", type=int, default=1500)
    ap.add_argument("--d", type=int, default=0, help="blobs with this d instead of the recipe")
    ap.add_argument("--poly", action="store_true", help="with --d: poly(1/d, 1, 2) instead of Gaussian")
    a = ap.parse_args()
    if a.d:
        X = synth.blobs(a.n, a.d, 4, seed=3080, sep=4.0)
        cfg = (dict(kind=oracle.POLY, gamma=1.0 / a.d, coef0=1.0, degree=2, k=4) if a.poly else
               dict(kind=oracle.GAUSSIAN, gamma=0.5 / a.d, coef0=0.0, degree=1, k=4))
    else:
        X, cfg = synth.make_config(a.config, n=a.n)
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    k = cfg["k"]
    if cfg["kind"] == oracle.GAUSSIAN:  # kkm_init centers X on its column means for the Gaussian kernel
        X = (X.astype(np.float64) - X.astype(np.float64).mean(axis=0)).astype(np.float32)
    Kx = oracle.kernel_matrix(X, *args)
    diag = np.diag(Kx).copy()
    bx = X.astype(np.float64) @ X.astype(np.float64).T
    ref = oracle.fit_K(Kx, diag, k, 15)  # converged-ish labels from the exact K
    lab = ref["labels"]
    Jx = oracle.objective(diag, lab, k, oracle.cnorm(oracle.E_rows(Kx, lab, k), lab, k))
    hi, lo, rs = split_fp16(X)
    print(f"{a.config if not a.d else f'blobs d={a.d}'} n={a.n} d={X.shape[1]} J={Jx:.6e} J/trK={Jx / diag.sum():.3f}")
    for name, chain, selfn, merged in [("S0 current", 0, False, False), ("S1 self-norms", 0, True, False),
                                       ("S2 chain 4", 4, False, False), ("S2 chain 2", 2, False, False),
                                       ("S3 merged ch2", 2, False, True), ("S3 merged ch1", 1, False, True),
                                       ("S1+S3 merged ch2", 2, True, True), ("S1+S3 merged ch3", 3, True, True)]:
        if selfn and cfg["kind"] != oracle.GAUSSIAN:
            continue
        m, c = tc_dot(hi, lo, chain, merged)
        b = (m + c).astype(np.float32)
        bb = b.astype(np.float64) * rs[:, None] * rs[None, :]
        scale = np.sqrt(np.outer(np.diag(bx), np.diag(bx)))
        rel = (bb - bx) / np.maximum(scale, 1e-30)
        K = kmat(b, rs, X, *args, self_norms=selfn)
        Km = K.copy()
        J = oracle.objective(np.diag(Km).copy(), lab, k, oracle.cnorm(oracle.E_rows(Km, lab, k), lab, k))
        print(f"  {name:16s} b: mean signed {rel.mean():+.2e} max|.| {np.abs(rel).max():.2e}   "
              f"K max|dK| {np.abs(K - Kx).max():.2e}   J rel {(J - Jx) / Jx:+.2e}")


if __name__ == "__main__":
    main()
