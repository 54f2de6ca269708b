"""ORACLE -- TEST INFRASTRUCTURE ONLY (see kkm_oracle.c header).

numpy/ctypes wrapper around the plain fp64 C oracle of exact Kernel K-means
(§2.2). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product path
(paper_2601_17136_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kkm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

LINEAR, POLY, GAUSSIAN = 0, 1, 2
_ERR = {1: "EINVAL", 2: "ELABEL", 3: "ENOMEM"}


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, OpenMP; no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", _LIB, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        sig = {
            "orc_kernel_rows": [P, i64, i64, i64, P, i64, ctypes.c_int, f64, f64, ctypes.c_int, P],
            "orc_kernel_diag": [P, i64, i64, i64, P, i64, ctypes.c_int, f64, f64, ctypes.c_int, P],
            "orc_round_robin": [i64, i32, P],
            "orc_sizes": [P, i64, i32, P],
            "orc_build_V": [P, i64, i32, P],
            "orc_E_rows": [P, i64, i64, P, i32, P],
            "orc_cnorm": [P, P, i64, i32, P],
            "orc_objective": [P, P, i64, i32, P, P],
            "orc_objective_X": [P, i64, i64, i64, P, i32, ctypes.c_int, f64, f64, ctypes.c_int, P],
            "orc_assign": [P, P, P, i64, i32, P, P],
            "orc_fit": [P, P, i64, i32, i32, i32, P, P, P, P, P],
            "orc_predict": [P, i64, P, i64, i64, P, i32, P, ctypes.c_int, f64, f64, ctypes.c_int, P, P],
            "orc_kmeanspp": [P, i64, i64, i32, ctypes.c_int, f64, f64, ctypes.c_int, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _lib.orc_kappa.argtypes = [P, P, i64, ctypes.c_int, f64, f64, ctypes.c_int]
        _lib.orc_kappa.restype = f64
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what}: {_ERR.get(rc, rc)}")


def _X(X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim != 2:
        raise ValueError("X must be 2-D")
    return X


def kappa(x, y, kind, gamma=1.0, coef0=0.0, degree=1) -> float:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    return lib().orc_kappa(_p(x), _p(y), x.size, kind, gamma, coef0, degree)


def kernel_rows(X, rows, kind, gamma=1.0, coef0=0.0, degree=1) -> np.ndarray:
    """K[rows, :] = kappa(X[rows], X) in fp64 (Eqs. b, k)."""
    X = _X(X)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((rows.size, X.shape[0]), dtype=np.float64)
    _check(lib().orc_kernel_rows(_p(X), X.shape[0], X.shape[1], X.shape[1], _p(rows), rows.size,
                                 kind, gamma, coef0, degree, _p(out)), "kernel_rows")
    return out


def kernel_matrix(X, kind, gamma=1.0, coef0=0.0, degree=1) -> np.ndarray:
    return kernel_rows(X, np.arange(_X(X).shape[0]), kind, gamma, coef0, degree)


def kernel_diag(X, kind, gamma=1.0, coef0=0.0, degree=1, rows=None) -> np.ndarray:
    X = _X(X)
    rows = np.arange(X.shape[0]) if rows is None else rows
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(rows.size, dtype=np.float64)
    _check(lib().orc_kernel_diag(_p(X), X.shape[0], X.shape[1], X.shape[1], _p(rows), rows.size,
                                 kind, gamma, coef0, degree, _p(out)), "kernel_diag")
    return out


def round_robin(n, k) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    _check(lib().orc_round_robin(n, k, _p(out)), "round_robin")
    return out


def sizes(labels, k) -> np.ndarray:
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    out = np.empty(k, dtype=np.int64)
    _check(lib().orc_sizes(_p(labels), labels.size, k, _p(out)), "sizes")
    return out


def build_V(labels, k) -> np.ndarray:
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    V = np.empty((k, labels.size), dtype=np.float64)
    _check(lib().orc_build_V(_p(labels), labels.size, k, _p(V)), "build_V")
    return V


def E_rows(Krows, labels, k) -> np.ndarray:
    """E = K V^T for the given K rows (Eq. e)."""
    Krows = np.ascontiguousarray(np.atleast_2d(Krows), dtype=np.float64)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    E = np.empty((Krows.shape[0], k), dtype=np.float64)
    _check(lib().orc_E_rows(_p(Krows), Krows.shape[0], Krows.shape[1], _p(labels), k, _p(E)),
           "E_rows")
    return E


def cnorm(E_all, labels, k) -> np.ndarray:
    E_all = np.ascontiguousarray(E_all, dtype=np.float64)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    out = np.empty(k, dtype=np.float64)
    _check(lib().orc_cnorm(_p(E_all), _p(labels), labels.size, k, _p(out)), "cnorm")
    return out


def objective(diag, labels, k, cn) -> float:
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    cn = np.ascontiguousarray(cn, dtype=np.float64)
    J = np.zeros(1, dtype=np.float64)
    _check(lib().orc_objective(_p(diag), _p(labels), labels.size, k, _p(cn), _p(J)), "objective")
    return float(J[0])


def objective_X(X, labels, k, kind, gamma=1.0, coef0=0.0, degree=1) -> float:
    """J of the labelling straight from the points (reading A8: tr K minus the within-cluster
    double sums over |L_c|), without storing K: for the full-size configs."""
    X = _X(X)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    J = np.zeros(1, dtype=np.float64)
    _check(lib().orc_objective_X(_p(X), X.shape[0], X.shape[1], X.shape[1], _p(labels), k, kind,
                                 gamma, coef0, degree, _p(J)), "objective_X")
    return float(J[0])


def assign(E, diag, cn):
    """Eq. (d) + argmin: returns (new_labels, Dfull)."""
    E = np.ascontiguousarray(E, dtype=np.float64)
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    cn = np.ascontiguousarray(cn, dtype=np.float64)
    n, k = E.shape
    D = np.empty((n, k), dtype=np.float64)
    nl = np.empty(n, dtype=np.int32)
    _check(lib().orc_assign(_p(E), _p(diag), _p(cn), n, k, _p(D), _p(nl)), "assign")
    return nl, D


def iteration(K, diag, labels, k):
    """One clustering iteration (Alg. 1 body) on a materialised K.
    Returns dict(E, cnorm, J, Dfull, new_labels, sizes)."""
    E = E_rows(K, labels, k)
    cn = cnorm(E, labels, k)
    J = objective(diag, labels, k, cn)
    nl, D = assign(E, diag, cn)
    return dict(E=E, cnorm=cn, J=J, Dfull=D, new_labels=nl, sizes=sizes(labels, k))


def fit_K(K, diag, k, max_iter, init_labels=None, stop_on_no_change=False, keep_trace=False):
    """The clustering loop on a materialised fp64 K. Returns dict(labels, J_trace,
    changed, iters, label_trace)."""
    K = np.ascontiguousarray(K, dtype=np.float64)
    n = K.shape[0]
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    labels = round_robin(n, k) if init_labels is None else np.array(init_labels, dtype=np.int32)
    J = np.zeros(max_iter + 1, dtype=np.float64)
    ch = np.zeros(max(max_iter, 1), dtype=np.int64)
    it = np.zeros(1, dtype=np.int32)
    tr = np.zeros((max_iter + 1, n), dtype=np.int32) if keep_trace else None
    _check(lib().orc_fit(_p(K), _p(diag), n, k, max_iter, int(stop_on_no_change), _p(labels),
                         _p(J), _p(ch), _p(it), _p(tr) if keep_trace else None), "fit")
    iters = int(it[0])
    return dict(labels=labels, J_trace=J[:iters + 1], changed=ch[:iters], iters=iters,
                label_trace=None if tr is None else tr[:iters + 1])


def fit(X, k, kind, gamma=1.0, coef0=0.0, degree=1, max_iter=30, init_labels=None,
        stop_on_no_change=False, keep_trace=False):
    """Exact Kernel K-means on X with K materialised in fp64 (small n only)."""
    K = kernel_matrix(X, kind, gamma, coef0, degree)
    diag = kernel_diag(X, kind, gamma, coef0, degree)
    out = fit_K(K, diag, k, max_iter, init_labels, stop_on_no_change, keep_trace)
    out["K"], out["diag"] = K, diag
    return out


def predict(X, labels, k, cn, Y, kind, gamma=1.0, coef0=0.0, degree=1):
    """Out-of-sample assignment of Y to the clusters of (X, labels) with centroid norms cn.
    Returns (labels_Y, Dfull_Y)."""
    X = _X(X)
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    cn = np.ascontiguousarray(cn, dtype=np.float64)
    m = Y.shape[0]
    out = np.empty(m, dtype=np.int32)
    D = np.empty((m, k), dtype=np.float64)
    _check(lib().orc_predict(_p(X), X.shape[0], _p(Y), m, X.shape[1], _p(labels), k, _p(cn), kind,
                             gamma, coef0, degree, _p(out), _p(D)), "predict")
    return out, D


def kmeanspp(X, k, u, kind, gamma=1.0, coef0=0.0, degree=1):
    """K-means++ seeding in feature space with the caller's uniforms u[0..k-1].
    Returns (centers int64[k], labels int32[n])."""
    X = _X(X)
    u = np.ascontiguousarray(u, dtype=np.float64)
    centers = np.empty(k, dtype=np.int64)
    labels = np.empty(X.shape[0], dtype=np.int32)
    _check(lib().orc_kmeanspp(_p(X), X.shape[0], X.shape[1], k, kind, gamma, coef0, degree, _p(u),
                              _p(centers), _p(labels)), "kmeanspp")
    return centers, labels
