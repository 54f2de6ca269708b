"""Oracle parity at the BASELINE.json configs' full sizes (SURVEY §8(c) "GPU-vs-oracle comparison
protocol", row-sampled for configs 3-5): the labels are injected (teacher forcing), ONE GPU
iteration runs in the launch configuration the path uses at that size, and for sampled rows i the
oracle computes the exact fp64 K row (n kernel evaluations, Eqs. b, k P:92-104) and from it E_i.
(Eq. e); D_i. = K_ii - 2 E_i. + c (Eq. d) with c from its definition
c_c = mean over L_c of E_ic (Eq. c) evaluated on the GPU's own E; the new labels by the
lowest-index argmin (A6). Sizes are exact. J of converged labels is recomputed from the points by
the oracle (oracle.objective_X, reading A8) at configs 1-3.

Injected labels: the generator's class of each point with 10 % of the points moved to a seeded
random cluster (a realistic segment structure for the label-sorted streaming kernels), or
round-robin (A5). Nothing here comes from the CUDA path except the values under test."""
import numpy as np
import pytest

import oracle
import synth
from parity import TAU, check_labels, j_tol, row_scale

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_17136_b200 as kkm  # noqa: E402


def noisy_truth(truth, k, frac=0.1, seed=0):
    rng = np.random.default_rng(seed)
    lab = np.asarray(truth, dtype=np.int64) % k
    move = rng.random(lab.size) < frac
    lab[move] = rng.integers(0, k, int(move.sum()))
    return lab.astype(np.int32)


def sample_rows(n, m=160, seed=1):
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(n, m, replace=False).tolist())
    rows |= {0, 1, n // 2, n - 2, n - 1}
    return np.array(sorted(rows), dtype=np.int64)


def sampled_iteration(h, X, lab, k, args, rows):
    """Injects `lab`, runs one iteration, checks the sampled rows against the oracle."""
    n = X.shape[0]
    h.set_labels(lab)
    it, J, ch = h.fit()
    assert it == 1
    E = h.debug_read(kkm.DBG_E)
    D = h.debug_read(kkm.DBG_DFULL)
    cn = h.debug_read(kkm.DBG_CNORM)
    sizes = h.debug_read(kkm.DBG_SIZES)
    new = h.assign().cpu().numpy()
    assert np.array_equal(h.debug_read(kkm.DBG_LABELS_PREV), lab)
    assert np.array_equal(sizes, np.bincount(lab, minlength=k))  # exact
    # c from its definition on the GPU's own E (Eq. c): c_c = (1/|L_c|) sum_{i in L_c} E_ic
    cn_def = np.array([E[lab == c, c].mean() if (lab == c).any() else np.inf for c in range(k)])
    fin = np.isfinite(cn_def)
    assert np.array_equal(np.isfinite(cn), fin)
    assert np.allclose(cn[fin], cn_def[fin], rtol=1e-12, atol=0)
    Kr = oracle.kernel_rows(X, rows, *args)
    diag = oracle.kernel_diag(X, *args, rows=rows)
    Er = oracle.E_rows(Kr, lab, k)
    scale = row_scale(Er, diag, cn_def)
    errE = np.abs(E[rows] - Er) / scale[:, None]
    assert (errE <= TAU).all(), f"E: worst {errE.max():.3e} of scale (tau {TAU})"
    nl, Dr = oracle.assign(Er, diag, cn_def)
    with np.errstate(invalid="ignore"):
        errD = np.where(np.isfinite(Dr), np.abs(D[rows] - Dr), 0.0) / scale[:, None]
    assert np.array_equal(np.isfinite(D[rows]), np.isfinite(Dr))
    assert (errD <= TAU).all(), f"Dfull: worst {errD.max():.3e}"
    check_labels(new[rows], nl, Dr, scale)
    # J = tr K - sum_c |L_c| c_c (A8) with the oracle's diagonal and the GPU's c
    diag_all = oracle.kernel_diag(X, *args)
    J_def = diag_all.sum() - (sizes[fin] * cn[fin]).sum()
    assert abs(J[0] - J_def) <= 1e-9 * abs(J_def)
    assert ch[0] == int((new != lab).sum())
    return float(errE.max()), float(errD.max())


def _handle(X, k, args, **kw):
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    return kkm.KernelKMeans(Xd, X.shape[0], k, *args, max_iter=1, **kw)


def test_config4_recipe_streaming_symmetric_sampled():
    """BASELINE configs[3] recipe (n = 1,000,000, d = 784, k = 10, Gaussian, median gamma): K
    (4 TB) cannot be stored, so AUTO streams it with the upper-triangle kernel (ssym_kernel:
    3907 row tiles in 32 x 32 supertiles, units of 16 column tiles taken dynamically, int64
    fixed-point S at n max K_ii 2^s < 2^61). Two injected labelings."""
    name = "mnist1m"
    n = synth.CONFIGS[name]["n"]
    X, truth = synth.mnist_like(n, synth.CONFIGS[name]["seed"], return_truth=True)
    gen = synth.row_generator(name)
    gamma = synth.median_gamma(gen, n, synth.CONFIGS[name]["seed"])
    args = (oracle.GAUSSIAN, gamma, 0.0, 1)
    k = 10
    h = _handle(X, k, args)
    rows = sample_rows(n, 128)
    sampled_iteration(h, X, noisy_truth(truth, k), k, args, rows)
    sampled_iteration(h, X, oracle.round_robin(n, k), k, args, rows)
    h.destroy()


def test_config5_recipe_streaming_symmetric_sampled():
    """BASELINE configs[4] recipe (MNIST8m-shaped: n = 8,100,000, d = 784, k = 10, poly(1,1,2)) on
    ONE GPU: the streaming f1 kernel over 31641 row tiles (~5e8 pair tiles, ~100 s), the int64
    fixed-point S at n = 8.1M. One injected labeling, 64 sampled rows (8.1M exact kernel
    evaluations each)."""
    name = "mnist8m"
    n = synth.CONFIGS[name]["n"]
    X, truth = synth.mnist_like(n, synth.CONFIGS[name]["seed"], return_truth=True)
    cfg = synth.CONFIGS[name]
    args = (cfg["kind"], cfg.get("gamma") or 1.0, cfg.get("coef0", 1.0), cfg.get("degree", 2))
    k = cfg["k"]
    h = _handle(X, k, args)
    rows = sample_rows(n, 64, seed=8)
    sampled_iteration(h, X, noisy_truth(truth, k, seed=8), k, args, rows)
    h.destroy()


@pytest.mark.parametrize("k", [10, 21])
def test_streaming_full_kernel_300k_sampled(k):
    """The full (non-symmetric) streaming kernel at n = 300,000 (MNIST recipe, poly(1,1,2)):
    1172 column tiles split over the work units (tc3_stream_kernel, int64 fixed-point S, any k in
    one launch: k = 21 has 20 segment boundaries inside the units)."""
    n = 300000
    X, truth = synth.mnist_like(n, 4, return_truth=True)
    args = (oracle.POLY, 1.0, 1.0, 2)
    h = _handle(X, k, args, path=kkm.PATH_STREAM, symmetric=kkm.SYM_OFF)
    rows = sample_rows(n, 96, seed=k)
    sampled_iteration(h, X, noisy_truth(truth, k, seed=k), k, args, rows)
    h.destroy()


def test_config3_materialised_full_size_sampled():
    """BASELINE configs[2] at full size (HAR-shaped n = 200,000, d = 561, k = 6, Gaussian): AUTO
    materialises the f1 upper-triangle bands as hi + lo fp16 planes (80 GB) and runs a2 on the
    tensor cores (spmm_tc_kernel); two injected labelings."""
    X, cfg = synth.make_config("har200k")
    truth = synth.har_like(cfg["n"], cfg["seed"], return_truth=True)[1]
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    k = cfg["k"]
    h = _handle(X, k, args)
    rows = sample_rows(cfg["n"], 128, seed=3)
    sampled_iteration(h, X, noisy_truth(truth, k, seed=3), k, args, rows)
    sampled_iteration(h, X, oracle.round_robin(cfg["n"], k), k, args, rows)
    h.destroy()


@pytest.mark.parametrize("name,iters", [("rings", 30), ("mnist60k", 100), ("har200k", 30)])
def test_full_size_objective_at_convergence(name, iters):
    """north_star "final objective within 1e-5 relative": the bench launch configuration runs to
    the configs' iteration counts from round robin; the oracle recomputes J of the GPU's final
    labels from the points (objective_X: tr K minus the within-cluster double sums, reading A8)."""
    X, cfg = synth.make_config(name)
    n, k = X.shape[0], cfg["k"]
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    Xd = torch.from_numpy(X).cuda()
    h = kkm.KernelKMeans(Xd, n, k, *args, max_iter=iters)
    h.fit()
    lab = h.assign().cpu().numpy()
    J = h.objective()
    h.destroy()
    Jref = oracle.objective_X(X, lab, k, *args)
    diag = oracle.kernel_diag(X, *args)
    print(f"\n{name}: J {J:.12e} oracle {Jref:.12e} rel {(J - Jref) / abs(Jref):+.3e}")
    assert abs(J - Jref) <= j_tol(Jref, diag), (J, Jref, abs(J - Jref) / abs(Jref))
