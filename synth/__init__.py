"""Seeded synthetic inputs for the Kernel K-means hot path (test/bench infrastructure).

This module is the ONE thing the oracle side (``oracle/``) and the CUDA side
(``paper_2601_17136_b200``) share: it produces point matrices X (n x d, float32,
row-major) and kernel parameters. It holds none of the method's arithmetic
(no kernel function, no cluster sums, no distances) -- only random numbers.

Every generator is counter-based: row i is a pure function of (seed, i), so
any row range can be generated independently and bit-identically (shards on
different ranks, sampled rows for row-sampled parity). Points are "shuffled"
by seed because the round-robin init cl_j = j mod k (reading
A5 in DESIGN.md) depends on the data order.

Recipes follow SURVEY.md §8(d) "Synthetic inputs"; DESIGN.md restates them.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "counter_uniform", "counter_normal", "rings", "blobs", "mnist_like",
    "har_like", "median_gamma", "CONFIGS", "make_config",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & _M64
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
    return z ^ (z >> np.uint64(31))


def _keys(seed: int, stream: int, rows: np.ndarray) -> np.ndarray:
    base = _splitmix64(np.array([(seed & 0xFFFFFFFF) << 20 | (stream & 0xFFFFF)], dtype=np.uint64))
    return _splitmix64(base ^ (rows.astype(np.uint64) * np.uint64(0xD1B54A32D192ED03) & _M64))


def counter_bits(seed: int, stream: int, rows: np.ndarray, ncols: int) -> np.ndarray:
    """uint64 bits[len(rows), ncols]; entry (r, c) depends only on (seed, stream, rows[r], c)."""
    rows = np.asarray(rows, dtype=np.int64)
    with np.errstate(over="ignore"):
        key = _keys(seed, stream, rows)[:, None]
        cols = (np.arange(ncols, dtype=np.uint64) * np.uint64(0x8CB92BA72F3D8DD7)) & _M64
        return _splitmix64(key ^ cols[None, :])


def counter_uniform(seed: int, stream: int, rows: np.ndarray, ncols: int) -> np.ndarray:
    """float64 in [0, 1) with 53 random bits."""
    b = counter_bits(seed, stream, rows, ncols)
    return (b >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def counter_normal(seed: int, stream: int, rows: np.ndarray, ncols: int) -> np.ndarray:
    """Standard normals by Box-Muller from two counter streams (host libm only)."""
    u1 = counter_uniform(seed, 2 * stream + 1, rows, ncols)
    u2 = counter_uniform(seed, 2 * stream + 2, rows, ncols)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def _rows(n: int, row_begin: int, row_end: int | None, rows=None) -> np.ndarray:
    if rows is not None:
        rows = np.asarray(rows, dtype=np.int64)
        if rows.size and (rows.min() < 0 or rows.max() >= n):
            raise ValueError("row index out of range")
        return rows
    row_end = n if row_end is None else row_end
    if not (0 <= row_begin <= row_end <= n):
        raise ValueError(f"bad row range [{row_begin},{row_end}) for n={n}")
    return np.arange(row_begin, row_end, dtype=np.int64)


# ---------------------------------------------------------------- config 1
def rings(n: int = 1000, seed: int = 1, radii=(1.0, 3.0), noise: float = 0.1,
          row_begin: int = 0, row_end: int | None = None, return_truth: bool = False, rows=None):
    """Two concentric rings in 2-D: radius r in {1, 3}, angle U[0, 2pi),
    radial noise N(0, noise^2). Ring membership is a keyed hash of the row index, so the
    data order is shuffled relative to the round-robin init."""
    rows = _rows(n, row_begin, row_end, rows)
    ring = (counter_bits(seed, 0, rows, 1)[:, 0] & np.uint64(1)).astype(np.int64)
    ang = 2.0 * np.pi * counter_uniform(seed, 1, rows, 1)[:, 0]
    rad = np.asarray(radii, dtype=np.float64)[ring] + noise * counter_normal(seed, 2, rows, 1)[:, 0]
    X = np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1).astype(np.float32)
    return (X, ring.astype(np.int32)) if return_truth else X


# ---------------------------------------------------------------- blobs (tests)
def blobs(n: int, d: int, k: int, seed: int = 7, sep: float = 10.0, std: float = 1.0,
          row_begin: int = 0, row_end: int | None = None, return_truth: bool = False, rows=None):
    """k isotropic Gaussian blobs; centres N(0, sep^2 I). Margin-separated for small k."""
    centers = sep * counter_normal(seed, 10, np.arange(k), d)
    rows = _rows(n, row_begin, row_end, rows)
    lab = (counter_bits(seed, 11, rows, 1)[:, 0] % np.uint64(k)).astype(np.int64)
    X = (centers[lab] + std * counter_normal(seed, 12, rows, d)).astype(np.float32)
    return (X, lab.astype(np.int32)) if return_truth else X


# ---------------------------------------------------------------- config 2/4/5
_MNIST_SIDE = 28


def _gauss_blur(img: np.ndarray, sigma: float) -> np.ndarray:
    r = int(np.ceil(3 * sigma))
    t = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-0.5 * (t / sigma) ** 2)
    g /= g.sum()
    out = np.apply_along_axis(lambda v: np.convolve(v, g, mode="same"), 0, img)
    return np.apply_along_axis(lambda v: np.convolve(v, g, mode="same"), 1, out)


def mnist_prototypes(seed: int, nclass: int = 10) -> np.ndarray:
    """nclass prototypes of 28x28: 3-6 Gaussian-blurred random strokes each, max 1."""
    S = _MNIST_SIDE
    protos = np.zeros((nclass, S, S))
    for c in range(nclass):
        u = counter_uniform(seed, 100 + c, np.arange(1), 64)[0]
        nstroke = 3 + int(u[0] * 4)
        img = np.zeros((S, S))
        for s in range(nstroke):
            y0, x0, y1, x1 = 6 + 16 * u[1 + 4 * s: 5 + 4 * s]
            for t in np.linspace(0.0, 1.0, 48):
                y, x = y0 + t * (y1 - y0), x0 + t * (x1 - x0)
                iy, ix = int(round(y)), int(round(x))
                img[max(iy - 1, 0):iy + 1, max(ix - 1, 0):ix + 1] = 1.0
        img = _gauss_blur(img, 0.8)
        protos[c] = img / img.max()
    return protos


def _parallel_chunks(nrows: int, chunk: int, fn):
    """Runs fn(c0, c1) over [0, nrows) in chunks on host threads (numpy releases the GIL);
    every row is a pure function of (seed, index), so the result does not depend on the split."""
    starts = list(range(0, nrows, chunk))
    workers = max(1, min(len(starts), len(os.sched_getaffinity(0))))
    if workers == 1:
        for c0 in starts:
            fn(c0, min(nrows, c0 + chunk))
        return
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(lambda c0: fn(c0, min(nrows, c0 + chunk)), starts))


def mnist_like(n: int = 60000, seed: int = 2, row_begin: int = 0, row_end: int | None = None,
               return_truth: bool = False, chunk: int = 8192, rows=None):
    """MNIST-shaped rows (d = 784) per SURVEY §8(d) cfg2: class = keyed hash mod 10,
    prototype shifted by +-2 px, contrast U[0.7, 1], N(0, 0.1^2) noise only on the
    prototype's support (> 0.05), clipped to [0, 1], quantised to multiples of 1/255."""
    S = _MNIST_SIDE
    protos = mnist_prototypes(seed)
    rows_all = _rows(n, row_begin, row_end, rows)
    X = np.empty((rows_all.size, S * S), dtype=np.float32)
    truth = np.empty(rows_all.size, dtype=np.int32)

    def work(c0, c1):
        rows = rows_all[c0:c1]
        bits = counter_bits(seed, 200, rows, 3)
        cls = (bits[:, 0] % np.uint64(10)).astype(np.int64)
        dy = (bits[:, 1] % np.uint64(5)).astype(np.int64) - 2
        dx = (bits[:, 2] % np.uint64(5)).astype(np.int64) - 2
        contrast = 0.7 + 0.3 * counter_uniform(seed, 201, rows, 1)
        img = np.empty((rows.size, S, S))
        for sy in range(-2, 3):
            for sx in range(-2, 3):
                m = (dy == sy) & (dx == sx)
                if m.any():
                    img[m] = np.roll(protos[cls[m]], shift=(sy, sx), axis=(1, 2))
        img = img.reshape(rows.size, S * S) * contrast
        support = img > 0.05
        img = img + support * (0.1 * counter_normal(seed, 202, rows, S * S))
        img = np.clip(img, 0.0, 1.0)
        X[c0:c1] = (np.rint(img * 255.0) / 255.0).astype(np.float32)
        truth[c0:c1] = cls

    _parallel_chunks(rows_all.size, chunk, work)
    return (X, truth) if return_truth else X


# ---------------------------------------------------------------- config 3
def har_like(n: int = 200000, seed: int = 3, d: int = 561, latent: int = 20, nclass: int = 6,
             row_begin: int = 0, row_end: int | None = None, return_truth: bool = False,
             chunk: int = 8192, rows=None):
    """HAR-shaped rows per SURVEY §8(d) cfg3: mu_c ~ N(0, 9 I_20), A in R^{d x 20} with
    N(0, 1/20) entries, x = tanh(0.5 A (mu_c + eps) + 0.05 xi); x in (-1, 1)."""
    mu = 3.0 * counter_normal(seed, 300, np.arange(nclass), latent)
    A = counter_normal(seed, 301, np.arange(d), latent) / np.sqrt(latent)
    rows_all = _rows(n, row_begin, row_end, rows)
    X = np.empty((rows_all.size, d), dtype=np.float32)
    truth = np.empty(rows_all.size, dtype=np.int32)

    def work(c0, c1):
        rows = rows_all[c0:c1]
        cls = (counter_bits(seed, 302, rows, 1)[:, 0] % np.uint64(nclass)).astype(np.int64)
        z = mu[cls] + counter_normal(seed, 303, rows, latent)
        X[c0:c1] = np.tanh(0.5 * z @ A.T + 0.05 * counter_normal(seed, 304, rows, d))
        truth[c0:c1] = cls

    _parallel_chunks(rows_all.size, chunk, work)
    return (X, truth) if return_truth else X


def median_gamma(gen, n: int, seed: int, pairs: int = 4096) -> float:
    """Gaussian gamma by the median heuristic (reading A15): 1 / median ||x_i - x_j||^2
    over `pairs` keyed random pairs, fp64. `gen(rows)` yields the given rows."""
    b = counter_bits(seed, 900, np.arange(pairs), 2)
    ii = (b[:, 0] % np.uint64(n)).astype(np.int64)
    jj = (b[:, 1] % np.uint64(n)).astype(np.int64)
    jj = np.where(jj == ii, (jj + 1) % n, jj)
    xi = gen(ii).astype(np.float64)
    xj = gen(jj).astype(np.float64)
    r2 = np.sum((xi - xj) ** 2, axis=1)
    return float(1.0 / np.median(r2))


# ---------------------------------------------------------------- BASELINE.json configs
KIND_LINEAR, KIND_POLY, KIND_GAUSSIAN = 0, 1, 2

CONFIGS = {
    # name: (n, d, k, kind, seed, iterations)  -- BASELINE.json "configs", SURVEY §8(d)
    "rings": dict(n=1000, d=2, k=2, kind=KIND_GAUSSIAN, seed=1, iters=30, gamma=1.0),
    "mnist60k": dict(n=60000, d=784, k=10, kind=KIND_POLY, seed=2, iters=100,
                     gamma=1.0, coef0=1.0, degree=2),
    "har200k": dict(n=200000, d=561, k=6, kind=KIND_GAUSSIAN, seed=3, iters=100),
    "mnist1m": dict(n=1000000, d=784, k=10, kind=KIND_GAUSSIAN, seed=4, iters=30),
    "mnist8m": dict(n=8100000, d=784, k=10, kind=KIND_POLY, seed=5, iters=3,
                    gamma=1.0, coef0=1.0, degree=2),
}


def row_generator(name: str, n: int | None = None):
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    seed = cfg["seed"]
    fn = {"rings": rings, "har200k": har_like}.get(name, mnist_like if name.startswith("mnist") else None)
    if fn is None:
        raise KeyError(name)
    return lambda rows: fn(n, seed, rows=rows)


def make_config(name: str, n: int | None = None, row_begin: int = 0, row_end: int | None = None):
    """Returns (X rows [row_begin,row_end) float32, params dict) for a BASELINE.json config.
    `n` overrides the point count (the generator recipe and kernel params stay the same)."""
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    gen = row_generator(name, cfg["n"])
    X = gen(np.arange(row_begin, cfg["n"] if row_end is None else row_end))
    if cfg["kind"] == KIND_GAUSSIAN and "gamma" not in cfg:
        cfg["gamma"] = median_gamma(gen, cfg["n"], cfg["seed"])
    cfg.setdefault("coef0", 0.0)
    cfg.setdefault("degree", 1)
    return X, cfg
