"""Pins for the fp64 CPU oracle (oracle/), checked against things other than itself:
hand-derived worked iterations, SPEC hand values, textbook Lloyd K-means (linear kernel),
Lloyd on the explicit degree-2 feature map, library routines (numpy matmul, scipy cdist),
closed forms, brute force over all labelings, invariants and invariances.
See DESIGN.md §4 for which pin covers which oracle function."""
import itertools
import json
import os

import numpy as np
import pytest
from scipy.spatial.distance import cdist

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- P1: SPEC hand values
def test_spec_hand_values():
    g = _gold("spec_hand_values.json")
    assert oracle.kappa(g["gemm_nt"]["A"], g["gemm_nt"]["B"], oracle.LINEAR) == g["gemm_nt"]["out"]
    # B = x.y = 2 with x = y = [1, 1]; B = 0 with orthogonal vectors
    assert oracle.kappa([1, 1], [1, 1], oracle.POLY, 1.0, 1.0, 2) == g["poly_of_2"]["out"]
    assert oracle.kappa([1, 0], [0, 5], oracle.POLY, 1.0, 1.0, 2) == g["poly_of_0"]["out"]
    V = oracle.build_V(g["assignment_values"]["cl"], 2)
    assert np.allclose(V.sum(axis=0), g["assignment_values"]["values"])
    assert (np.count_nonzero(V, axis=0) == 1).all()
    V = oracle.build_V(g["assignment_singletons"]["cl"], 3)
    assert np.allclose(V.sum(axis=0), 1.0)
    # S:81 gives E^T = V K; Eq. (e) is E = K V^T, so E(K^T) == (V K)^T
    s = g["spmm_transposed"]
    K = np.array(s["K"], dtype=np.float64)
    assert np.allclose(oracle.E_rows(K.T, s["cl"], 1).T, s["Et"])
    assert np.allclose(oracle.E_rows(K, s["cl"], 1), [[1.5], [3.5]])  # catches a transposed operand
    # mask + spmv (Eqs. z, c): singleton clusters give cnorm = z
    m = g["mask"]
    E = np.array(m["Et"], dtype=np.float64).T
    assert np.allclose(oracle.cnorm(E, m["cl"], 2), m["z"])
    sp = g["spmv"]
    assert np.allclose(oracle.cnorm(np.array(sp["z"], dtype=np.float64)[:, None], sp["cl"], 1),
                       sp["c"])
    ds = g["distance"]
    _, D = oracle.assign(np.array(ds["Et"], dtype=np.float64).T, [0.0], ds["c"])
    assert np.allclose(D, ds["D"])
    am = g["argmin"]
    Dt = np.array(am["Dt"], dtype=np.float64)
    nl, _ = oracle.assign(-Dt.T / 2.0, np.zeros(2), np.zeros(2))
    assert nl.tolist() == am["cl"]
    for rr in g["round_robin"]:
        assert oracle.round_robin(rr["n"], rr["k"]).tolist() == rr["cl"]


# ---------------------------------------------------------------- P2/P3: hand iterations
@pytest.mark.parametrize("name", ["hand_linear_x0134.json", "hand_poly_x0134.json"])
def test_hand_iteration(name):
    g = _gold(name)
    X = np.array(g["X"], dtype=np.float32)
    args = (g["kind"], g["gamma"], g["coef0"], g["degree"])
    K = oracle.kernel_matrix(X, *args)
    if "K" in g:
        assert np.array_equal(K, np.array(g["K"], dtype=np.float64))
    diag = oracle.kernel_diag(X, *args)
    it = oracle.iteration(K, diag, g["labels0"], g["k"])
    assert np.allclose(it["E"], g["E0"], rtol=0, atol=1e-12)
    assert np.allclose(it["cnorm"], g["cnorm0"], rtol=0, atol=1e-12)
    assert abs(it["J"] - g["J0"]) < 1e-12
    assert np.allclose(it["Dfull"], g["Dfull0"], rtol=0, atol=1e-12)
    assert it["new_labels"].tolist() == g["labels1"]
    fit = oracle.fit_K(K, diag, g["k"], 5, init_labels=g["labels0"], keep_trace=True)
    assert fit["label_trace"][1].tolist() == g["labels1"]
    assert fit["label_trace"][2].tolist() == g["labels2"]
    assert abs(fit["J_trace"][0] - g["J0"]) < 1e-12 and abs(fit["J_trace"][1] - g["J1"]) < 1e-12
    it1 = oracle.iteration(K, diag, g["labels1"], g["k"])
    assert np.allclose(it1["cnorm"], g["cnorm1"], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- kernel values vs libraries
def test_kernel_values_vs_library():
    rng = np.random.default_rng(0)
    X = rng.normal(size=(40, 7)).astype(np.float32)
    X64 = X.astype(np.float64)
    B = X64 @ X64.T
    assert np.allclose(oracle.kernel_matrix(X, oracle.LINEAR), B, rtol=1e-13, atol=1e-12)
    assert np.allclose(oracle.kernel_matrix(X, oracle.POLY, 0.3, 1.5, 3), (0.3 * B + 1.5) ** 3,
                       rtol=1e-12)
    G = np.exp(-0.7 * cdist(X64, X64, "sqeuclidean"))
    assert np.allclose(oracle.kernel_matrix(X, oracle.GAUSSIAN, 0.7), G, rtol=1e-12, atol=1e-15)
    assert np.allclose(oracle.kernel_diag(X, oracle.GAUSSIAN, 0.7), 1.0)
    # two points at distance r^2 = 1 with gamma = ln 2 -> 0.5
    assert abs(oracle.kappa([0, 0], [1, 0], oracle.GAUSSIAN, np.log(2.0)) - 0.5) < 1e-15
    rows = np.array([3, 17, 39])
    assert np.array_equal(oracle.kernel_rows(X, rows, oracle.POLY, 1, 1, 2),
                          oracle.kernel_matrix(X, oracle.POLY, 1, 1, 2)[rows])


# ---------------------------------------------------------------- P4: linear == Lloyd
def lloyd(F, k, labels, iters):
    """Textbook Lloyd's K-means on explicit features F (n x m), fp64: centroid = mean,
    distance = ||f - mu||^2, lowest index on ties, empty cluster never chosen."""
    labels = np.array(labels)
    trace, J = [labels.copy()], []
    for _ in range(iters):
        mu = np.stack([F[labels == c].mean(axis=0) if (labels == c).any()
                       else np.full(F.shape[1], np.nan) for c in range(k)])
        dist = np.stack([((F - mu[c]) ** 2).sum(axis=1) if (labels == c).any()
                         else np.full(F.shape[0], np.inf) for c in range(k)], axis=1)
        J.append(float(sum(((F[labels == c] - mu[c]) ** 2).sum() for c in range(k)
                           if (labels == c).any())))
        labels = np.argmin(dist, axis=1)
        trace.append(labels.copy())
    return trace, J


def _margin_ok(F, k, labels):
    """True if every point's nearest / second-nearest centroid gap is comfortably large,
    so summation-order rounding cannot flip an assignment."""
    mu = [F[labels == c].mean(axis=0) for c in range(k) if (labels == c).any()]
    dist = np.stack([((F - m) ** 2).sum(axis=1) for m in mu], axis=1)
    s = np.sort(dist, axis=1)
    return s.shape[1] < 2 or (s[:, 1] - s[:, 0]).min() > 1e-9 * max(1.0, s.max())


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_linear_equals_lloyd(seed):
    X = synth.blobs(90, 3, 4, seed=seed, sep=3.0)
    X64 = X.astype(np.float64)
    init = oracle.round_robin(90, 4)
    fit = oracle.fit(X, 4, oracle.LINEAR, max_iter=12, init_labels=init, keep_trace=True)
    trace, J = lloyd(X64, 4, init, 12)
    for t in range(12):
        assert _margin_ok(X64, 4, trace[t])
        assert np.array_equal(fit["label_trace"][t + 1], trace[t + 1]), t
        assert abs(fit["J_trace"][t] - J[t]) <= 1e-9 * max(1.0, J[t])  # J == SSE (P4)


# ---------------------------------------------------------------- P5: poly2 == Lloyd on phi
def feature_map_poly2(X, gamma, coef0):
    """phi(x) = [gamma vec(x x^T), sqrt(2 gamma c0) x, c0]: phi(x).phi(y) = (gamma x.y + c0)^2."""
    X = X.astype(np.float64)
    outer = gamma * np.einsum("ni,nj->nij", X, X).reshape(X.shape[0], -1)
    return np.hstack([outer, np.sqrt(2 * gamma * coef0) * X, np.full((X.shape[0], 1), coef0)])


@pytest.mark.parametrize("seed", [4, 5])
def test_poly2_equals_lloyd_on_feature_map(seed):
    X = synth.rings(120, seed=seed)
    F = feature_map_poly2(X, 0.8, 1.3)
    assert np.allclose(F @ F.T, (0.8 * X.astype(np.float64) @ X.astype(np.float64).T + 1.3) ** 2)
    init = oracle.round_robin(120, 3)
    fit = oracle.fit(X, 3, oracle.POLY, 0.8, 1.3, 2, max_iter=10, init_labels=init, keep_trace=True)
    trace, J = lloyd(F, 3, init, 10)
    for t in range(10):
        assert _margin_ok(F, 3, trace[t])
        assert np.array_equal(fit["label_trace"][t + 1], trace[t + 1]), t
        assert abs(fit["J_trace"][t] - J[t]) <= 1e-9 * max(1.0, J[t])


# ---------------------------------------------------------------- Gaussian closed forms
def test_gaussian_cnorm_closed_form():
    """cnorm_c = ||mu_c||^2 = (1/|L_c|^2) sum_{j,l in L_c} K(j,l): the double-sum closed form
    (a different route than mask + SpMV, Eqs. z, c)."""
    X = synth.rings(60, seed=3)
    K = np.exp(-0.9 * cdist(X.astype(np.float64), X.astype(np.float64), "sqeuclidean"))
    labels = (np.arange(60) * 7) % 4
    E = oracle.E_rows(K, labels, 4)
    cn = oracle.cnorm(E, labels, 4)
    for c in range(4):
        m = labels == c
        assert abs(cn[c] - K[np.ix_(m, m)].sum() / m.sum() ** 2) < 1e-13
    # D_full(i,c) = ||phi(x_i) - mu_c||^2 = K_ii - 2/|L| sum_j K_ij + cnorm_c
    nl, D = oracle.assign(E, np.ones(60), cn)
    for c in range(4):
        m = labels == c
        ref = 1.0 - 2.0 * K[:, m].sum(axis=1) / m.sum() + K[np.ix_(m, m)].sum() / m.sum() ** 2
        assert np.allclose(D[:, c], ref, rtol=0, atol=1e-12)


def test_gaussian_gamma_zero():
    """gamma = 0 -> K == 1 -> every D equal -> all points to cluster 0 (A6), J = 0 after."""
    X = synth.rings(50, seed=2)
    fit = oracle.fit(X, 3, oracle.GAUSSIAN, 0.0, max_iter=4, keep_trace=True)
    assert (fit["label_trace"][1] == 0).all()
    assert np.allclose(fit["J_trace"][1:], 0.0, atol=1e-12)
    assert (fit["label_trace"][-1] == 0).all()  # empty clusters stay empty (A7)


# ---------------------------------------------------------------- P7 / P8
def test_k_equals_one():
    X = synth.blobs(40, 5, 3, seed=9)
    fit = oracle.fit(X, 1, oracle.POLY, 1.0, 1.0, 2, max_iter=3)
    K = fit["K"]
    Jc = np.trace(K) - K.sum() / 40.0
    assert (fit["labels"] == 0).all()
    assert np.allclose(fit["J_trace"], Jc, rtol=1e-12)


def test_k_equals_n_singletons():
    X = synth.blobs(12, 3, 3, seed=11)
    fit = oracle.fit(X, 12, oracle.GAUSSIAN, 0.5, max_iter=3)
    assert fit["labels"].tolist() == list(range(12))
    assert np.allclose(fit["J_trace"], 0.0, atol=1e-12)
    assert (fit["changed"] == 0).all()


# ---------------------------------------------------------------- P9: monotonicity
@pytest.mark.parametrize("kind,args", [(oracle.LINEAR, ()), (oracle.POLY, (1.0, 1.0, 2)),
                                        (oracle.GAUSSIAN, (0.5,))])
def test_monotone(kind, args):
    for seed in range(8):
        X = synth.blobs(64, 4, 5, seed=100 + seed, sep=2.0)
        fit = oracle.fit(X, 5, kind, *args, max_iter=15)
        J = fit["J_trace"]
        assert (np.diff(J) <= 1e-12 * np.abs(J[:-1]) + 1e-12).all(), J


# ---------------------------------------------------------------- P10: identities
def test_identities():
    X = synth.mnist_like(200, seed=2)
    K = oracle.kernel_matrix(X, oracle.POLY, 1.0, 1.0, 2)
    labels = oracle.round_robin(200, 7)
    E = oracle.E_rows(K, labels, 7)
    sz = oracle.sizes(labels, 7)
    assert np.allclose((E * sz[None, :]).sum(axis=1), K.sum(axis=1), rtol=1e-12)
    cn = oracle.cnorm(E, labels, 7)
    z = E[np.arange(200), labels]
    assert abs(z.sum() - (sz * cn).sum()) <= 1e-12 * abs(z.sum())
    assert (cn >= 0).all()
    _, D = oracle.assign(E, np.diag(K), cn)
    assert (D >= -1e-9 * np.abs(D).max()).all()


# ---------------------------------------------------------------- P11: invariances
def test_invariances():
    X = synth.rings(80, seed=6)
    a = oracle.fit(X, 3, oracle.GAUSSIAN, 0.8, max_iter=8, keep_trace=True)
    b = oracle.fit(X + np.float32(5.0), 3, oracle.GAUSSIAN, 0.8, max_iter=8, keep_trace=True)
    assert np.array_equal(a["label_trace"], b["label_trace"])
    c = oracle.fit(X * np.float32(2.0), 3, oracle.GAUSSIAN, 0.2, max_iter=8, keep_trace=True)
    assert np.array_equal(a["label_trace"], c["label_trace"])
    lin = oracle.fit(X, 3, oracle.LINEAR, max_iter=8, keep_trace=True)
    lin2 = oracle.fit(X - np.float32(1.5), 3, oracle.LINEAR, max_iter=8, keep_trace=True)
    assert np.array_equal(lin["label_trace"], lin2["label_trace"])
    perm = np.random.default_rng(1).permutation(80)
    init = oracle.round_robin(80, 3)
    p = oracle.fit(X[perm], 3, oracle.GAUSSIAN, 0.8, max_iter=8, init_labels=init[perm])
    assert np.array_equal(p["labels"], a["labels"][perm])


# ---------------------------------------------------------------- P12: brute force
@pytest.mark.parametrize("kind,args", [(oracle.LINEAR, ()), (oracle.POLY, (1.0, 1.0, 2))])
def test_bruteforce_all_labelings(kind, args):
    X = synth.blobs(9, 2, 2, seed=21, sep=1.5)
    K = oracle.kernel_matrix(X, kind, *args)
    diag = np.diag(K).copy()
    F = X.astype(np.float64) if kind == oracle.LINEAR else feature_map_poly2(X, 1.0, 1.0)
    for bits in itertools.product([0, 1], repeat=9):
        lab = np.array(bits, dtype=np.int32)
        E = oracle.E_rows(K, lab, 2)
        J = oracle.objective(diag, lab, 2, oracle.cnorm(E, lab, 2))
        Jb = sum(((F[lab == c] - F[lab == c].mean(axis=0)) ** 2).sum() for c in (0, 1)
                 if (lab == c).any())
        assert abs(J - Jb) <= 1e-9 * max(1.0, Jb)
    fit = oracle.fit(X, 2, kind, *args, max_iter=50, stop_on_no_change=True)
    assert fit["changed"][-1] == 0
    E = oracle.E_rows(K, fit["labels"], 2)
    _, D = oracle.assign(E, diag, oracle.cnorm(E, fit["labels"], 2))
    own = D[np.arange(9), fit["labels"]]
    assert (own <= D.min(axis=1) + 1e-12 * np.abs(D).max()).all()


# ---------------------------------------------------------------- empty clusters / errors
def test_empty_cluster_never_chosen():
    X = synth.blobs(30, 2, 3, seed=5)
    init = np.zeros(30, dtype=np.int32)
    init[::2] = 1  # cluster 2 empty
    fit = oracle.fit(X, 3, oracle.LINEAR, max_iter=5, init_labels=init, keep_trace=True)
    assert not (fit["label_trace"] == 2).any()
    E = oracle.E_rows(fit["K"], init, 3)
    assert np.isinf(oracle.cnorm(E, init, 3)[2])


def test_errors():
    with pytest.raises(ValueError, match="ELABEL"):
        oracle.sizes([0, 3], 2)
    X = synth.blobs(5, 2, 2)
    with pytest.raises(ValueError, match="EINVAL"):
        oracle.fit(X, 6, oracle.LINEAR, max_iter=1)
    with pytest.raises(ValueError, match="EINVAL"):
        oracle.kernel_rows(X, [0], oracle.POLY, 1.0, 1.0, 0)


def test_thread_count_independence(monkeypatch):
    """OpenMP over rows with sequential per-row sums: bitwise identical for any thread count."""
    import subprocess
    import sys
    code = ("import numpy as np, oracle, synth; X = synth.mnist_like(300, 2);"
            "f = oracle.fit(X, 5, oracle.POLY, 1.0, 1.0, 2, max_iter=3);"
            "print(repr(f['J_trace'].tolist()), f['labels'].sum())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {subprocess.check_output([sys.executable, "-c", code], cwd=root,
                                    env=dict(os.environ, OMP_NUM_THREADS=str(t))).strip()
            for t in (1, 3)}
    assert len(outs) == 1


# ---------------------------------------------------------------- f4: out-of-sample assignment
def test_predict_on_training_points_equals_assign():
    """Predicting the training points reproduces the iteration's distances (Eq. d) exactly."""
    X = synth.blobs(80, 4, 3, seed=31, sep=3.0)
    K = oracle.kernel_matrix(X, oracle.POLY, 0.5, 1.0, 2)
    diag = np.diag(K).copy()
    lab = oracle.round_robin(80, 3)
    it = oracle.iteration(K, diag, lab, 3)
    nl, D = oracle.predict(X, lab, 3, it["cnorm"], X, oracle.POLY, 0.5, 1.0, 2)
    assert np.array_equal(nl, it["new_labels"])
    assert np.allclose(D, it["Dfull"], rtol=1e-12, atol=1e-9)


def test_predict_linear_is_nearest_centroid():
    """Linear kernel: D(y, c) = ||y - mu_c||^2 with explicit centroids (textbook)."""
    X = synth.blobs(120, 5, 4, seed=32, sep=4.0)
    Y = synth.blobs(50, 5, 4, seed=33, sep=4.0)
    lab = (np.arange(120) * 7) % 4
    K = oracle.kernel_matrix(X, oracle.LINEAR)
    cn = oracle.cnorm(oracle.E_rows(K, lab, 4), lab, 4)
    nl, D = oracle.predict(X, lab, 4, cn, Y, oracle.LINEAR)
    mu = np.stack([X[lab == c].astype(np.float64).mean(axis=0) for c in range(4)])
    ref = ((Y.astype(np.float64)[:, None, :] - mu[None]) ** 2).sum(axis=2)
    assert np.allclose(D, ref, rtol=1e-10, atol=1e-9)
    assert np.array_equal(nl, ref.argmin(axis=1))


def test_predict_empty_cluster_and_gaussian():
    X = synth.rings(60, seed=8)
    lab = np.zeros(60, dtype=np.int32)
    lab[30:] = 2  # cluster 1 empty
    K = oracle.kernel_matrix(X, oracle.GAUSSIAN, 0.7)
    cn = oracle.cnorm(oracle.E_rows(K, lab, 3), lab, 3)
    Y = synth.rings(20, seed=9)
    nl, D = oracle.predict(X, lab, 3, cn, Y, oracle.GAUSSIAN, 0.7)
    assert not (nl == 1).any() and np.isinf(D[:, 1]).all()
    # Gaussian: D(y, c) = 1 - 2 mean_j K(y, x_j) + (1/|L|^2) sum K  (closed form via scipy cdist)
    from scipy.spatial.distance import cdist
    Ky = np.exp(-0.7 * cdist(Y.astype(np.float64), X.astype(np.float64), "sqeuclidean"))
    for c in (0, 2):
        m = lab == c
        ref = 1.0 - 2.0 * Ky[:, m].mean(axis=1) + K[np.ix_(m, m)].sum() / m.sum() ** 2
        assert np.allclose(D[:, c], ref, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- f3: K-means++ seeding
def _kpp_numpy(F, k, u):
    """Textbook k-means++ (Arthur & Vassilvitskii) on explicit features F with the given
    uniforms: inverse CDF by numpy cumsum + searchsorted."""
    n = F.shape[0]
    cen = [min(int(u[0] * n), n - 1)]
    D = ((F - F[cen[0]]) ** 2).sum(axis=1)
    for t in range(1, k):
        Dp = np.maximum(D, 0.0)
        cdf = np.cumsum(Dp)
        cen.append(int(np.searchsorted(cdf, u[t] * cdf[-1], side="right")) if cdf[-1] > 0 else cen[-1])
        D = np.minimum(D, ((F - F[cen[-1]]) ** 2).sum(axis=1))
    dist = np.stack([((F - F[c]) ** 2).sum(axis=1) for c in cen], axis=1)
    return np.array(cen), dist.argmin(axis=1)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_kmeanspp_linear_is_textbook(seed):
    X = synth.blobs(300, 4, 6, seed=70 + seed, sep=3.0)
    u = np.random.default_rng(seed).random(6)
    c, lab = oracle.kmeanspp(X, 6, u, oracle.LINEAR)
    c_ref, lab_ref = _kpp_numpy(X.astype(np.float64), 6, u)
    assert np.array_equal(c, c_ref)
    assert np.array_equal(lab, lab_ref)


def test_kmeanspp_poly2_feature_map_and_special_cases():
    X = synth.rings(200, seed=11)
    u = np.random.default_rng(5).random(4)
    c, lab = oracle.kmeanspp(X, 4, u, oracle.POLY, 0.8, 1.3, 2)
    c_ref, lab_ref = _kpp_numpy(feature_map_poly2(X, 0.8, 1.3), 4, u)
    assert np.array_equal(c, c_ref) and np.array_equal(lab, lab_ref)
    # k = 1: the first draw picks the center, every point in cluster 0
    c1, l1 = oracle.kmeanspp(X, 1, [0.5], oracle.GAUSSIAN, 0.7)
    assert c1.tolist() == [100] and (l1 == 0).all()
    # each center is its own nearest center (distance 0) and centers are distinct while D > 0
    assert len(set(c.tolist())) == 4 and all(lab[ci] == t for t, ci in enumerate(c))
    # duplicate points: D = 0 points are never drawn; with all points equal, centers repeat
    Xd = np.repeat(X[:3], 5, axis=0)
    cd, ld = oracle.kmeanspp(Xd, 5, np.random.default_rng(1).random(5), oracle.GAUSSIAN, 0.7)
    assert len(set(map(tuple, Xd[cd[:3]]))) == 3
    assert (cd[3:] == cd[2]).all()


# ---------------------------------------------------------------- P13 quality (not parity)
def test_quality_rings_and_blobs_recovered():
    """blobs recovered, rings ARI -- with K-means++ seeding (the
    round-robin start of A5 lands in another local optimum of J on the rings, ARI ~0.27)."""
    from sklearn.metrics import adjusted_rand_score
    X, truth = synth.rings(1000, seed=1, return_truth=True)
    _, lab0 = oracle.kmeanspp(X, 2, np.random.default_rng(0).random(2), oracle.GAUSSIAN, 1.0)
    fit = oracle.fit(X, 2, oracle.GAUSSIAN, 1.0, max_iter=30, init_labels=lab0)
    assert adjusted_rand_score(truth, fit["labels"]) == 1.0
    Xb, tb = synth.blobs(600, 8, 5, seed=2, sep=10.0, return_truth=True)
    _, lb = oracle.kmeanspp(Xb, 5, np.random.default_rng(1).random(5), oracle.LINEAR)
    fb = oracle.fit(Xb, 5, oracle.LINEAR, max_iter=30, init_labels=lb)
    assert adjusted_rand_score(tb, fb["labels"]) == 1.0


# ---------------------------------------------------------------- objective_X (J from the points)
@pytest.mark.parametrize("kind,args", [(oracle.LINEAR, ()), (oracle.POLY, (1.0, 1.0, 2)),
                                       (oracle.POLY, (0.7, 0.4, 3))])
def test_objective_X_bruteforce_feature_space(kind, args):
    """A8 by brute force: J(cl) = sum_i ||phi(x_i) - mu_cl(i)||^2 with explicit features (linear:
    x itself; poly deg 2: the explicit map), for all 2^9 labelings of 9 points; poly deg 3 against
    the K V^T path (orc_objective) instead (no explicit map here)."""
    X = synth.blobs(9, 2, 2, seed=23, sep=1.5)
    K = oracle.kernel_matrix(X, kind, *args)
    diag = np.diag(K).copy()
    F = None
    if kind == oracle.LINEAR:
        F = X.astype(np.float64)
    elif args[2] == 2:
        F = feature_map_poly2(X, args[0], args[1])
    for bits in itertools.product([0, 1], repeat=9):
        lab = np.array(bits, dtype=np.int32)
        J = oracle.objective_X(X, lab, 2, kind, *args)
        if F is not None:
            Jb = sum(((F[lab == c] - F[lab == c].mean(axis=0)) ** 2).sum() for c in (0, 1) if (lab == c).any())
        else:
            Jb = oracle.objective(diag, lab, 2, oracle.cnorm(oracle.E_rows(K, lab, 2), lab, 2))
        assert abs(J - Jb) <= 1e-10 * max(1.0, abs(Jb)), (bits, J, Jb)


@pytest.mark.parametrize("name,n,k", [("mnist60k", 500, 10), ("har200k", 400, 6), ("rings", 300, 2)])
def test_objective_X_equals_iteration_J(name, n, k):
    """The same J as the iteration's E / c path (Eqs. e, z, c + A8) on the configs' recipes, for
    round-robin, random and empty-cluster labelings; Gaussian gamma = 0 gives J = 0 (K = 1)."""
    X, cfg = synth.make_config(name, n=n)
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    K = oracle.kernel_matrix(X, *args)
    diag = np.diag(K).copy()
    rng = np.random.default_rng(5)
    labs = [oracle.round_robin(n, k), rng.integers(0, k, n).astype(np.int32)]
    e = rng.integers(0, k, n).astype(np.int32)
    e[e == 1] = 0  # cluster 1 empty
    labs.append(e)
    for lab in labs:
        Jd = oracle.objective(diag, lab, k, oracle.cnorm(oracle.E_rows(K, lab, k), lab, k))
        J = oracle.objective_X(X, lab, k, *args)
        assert abs(J - Jd) <= 1e-11 * float(np.abs(diag).sum()), (J, Jd)
    if cfg["kind"] == oracle.GAUSSIAN:
        assert oracle.objective_X(X, labs[1], k, oracle.GAUSSIAN, 0.0) == 0.0


def test_objective_X_thread_independence(monkeypatch):
    X = synth.blobs(700, 5, 4, seed=9)
    lab = np.random.default_rng(1).integers(0, 4, 700).astype(np.int32)
    a = oracle.objective_X(X, lab, 4, oracle.GAUSSIAN, 0.1)
    import subprocess
    import sys
    code = ("import numpy as np, oracle, synth; X = synth.blobs(700, 5, 4, seed=9); "
            "lab = np.random.default_rng(1).integers(0, 4, 700).astype(np.int32); "
            "print(repr(oracle.objective_X(X, lab, 4, oracle.GAUSSIAN, 0.1)))")
    env = dict(os.environ, OMP_NUM_THREADS="1",
               PYTHONPATH=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = subprocess.check_output([sys.executable, "-c", code], env=env, text=True).strip()
    assert float(out) == a
