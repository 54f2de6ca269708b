"""GPU parity of kkm_predict (out-of-sample assignment) against
oracle.predict (pinned in tests/test_oracle.py) on seeded held-out rows of the paper's
workload recipes, under the tolerance rules of tests/parity.py."""
import numpy as np
import pytest

import oracle
import synth
from parity import TAU, check_labels

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_17136_b200 as kkm  # noqa: E402

MODES = [(kkm.PREC_FP16X3, kkm.PATH_MATERIALIZE), (kkm.PREC_FP16X3, kkm.PATH_STREAM)]
MODE_IDS = ["fp16x3", "fp16x3-stream"]


def _fit(X, k, kind, gamma, coef0, degree, iters, mode, init=None):
    prec, path = mode
    h = kkm.KernelKMeans(torch.from_numpy(X).cuda(), X.shape[0], k, kind, gamma, coef0, degree,
                         max_iter=iters, precision=prec, path=path, init_labels=init)
    if iters:
        h.fit()
    return h


def _check_predict(h, Xtr, Y, k, kind, gamma, coef0, degree):
    lab = h.assign().cpu().numpy()
    K = oracle.kernel_matrix(Xtr, kind, gamma, coef0, degree)
    cn = oracle.cnorm(oracle.E_rows(K, lab, k), lab, k)
    nl, D = oracle.predict(Xtr, lab, k, cn, Y, kind, gamma, coef0, degree)
    lg, Dg = h.predict(Y, return_distances=True)
    kyy = oracle.kernel_diag(Y, kind, gamma, coef0, degree)
    fin = np.isfinite(cn)
    assert np.array_equal(np.isfinite(Dg), np.isfinite(D))
    E = np.where(np.isfinite(D), (kyy[:, None] + np.where(fin, cn, 0)[None] - np.where(np.isfinite(D), D, 0)) / 2, 0)
    scale = np.abs(kyy) + 2 * np.abs(E).max(axis=1) + abs(cn[fin].max())
    with np.errstate(invalid="ignore"):
        err = np.where(np.isfinite(D), np.abs(Dg - D), 0)
    assert (err <= TAU * scale[:, None]).all(), (err / scale[:, None]).max()
    check_labels(lg, nl, np.where(np.isfinite(D), D, np.inf), scale)
    # device input / device output, and library-allocated scratch, give the same answer
    lg2 = h.predict(torch.from_numpy(Y).cuda()).cpu().numpy()
    assert np.array_equal(lg2, lg)
    lg3, Dg3 = h.predict(Y, return_distances=True, use_workspace=False)
    assert np.array_equal(lg3, lg) and np.array_equal(Dg3, Dg)
    return lg, nl


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
def test_predict_mnist_poly(mode):
    """configs[1] recipe: train on 3000 rows, assign 1000 held-out rows (ragged vs 256-row tiles)."""
    Xa, cfg = synth.make_config("mnist60k", n=4000)
    Xtr, Y = Xa[:3000], Xa[3000:]
    h = _fit(Xtr, 10, cfg["kind"], 1.0, 1.0, 2, 3, mode)
    _check_predict(h, Xtr, Y, 10, cfg["kind"], 1.0, 1.0, 2)
    h.destroy()


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
def test_predict_har_gaussian(mode):
    """configs[2] recipe (d = 561, Gaussian with the median gamma)."""
    Xa, cfg = synth.make_config("har200k", n=3200)
    Xtr, Y = Xa[:2500], Xa[2500:]
    h = _fit(Xtr, 6, cfg["kind"], cfg["gamma"], 0.0, 1, 3, mode)
    _check_predict(h, Xtr, Y, 6, cfg["kind"], cfg["gamma"], 0.0, 1)
    h.destroy()


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
@pytest.mark.parametrize("k", [21, 70])
def test_predict_many_clusters(mode, k):
    """k > 16: the streaming kernel runs once per group of 16 clusters."""
    Xa = synth.blobs(1700, 8, k, seed=40 + k, sep=3.0)
    Xtr, Y = Xa[:1400], Xa[1400:]
    h = _fit(Xtr, k, oracle.POLY, 0.2, 1.0, 2, 2, mode)
    _check_predict(h, Xtr, Y, k, oracle.POLY, 0.2, 1.0, 2)
    h.destroy()


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
def test_predict_empty_cluster_and_no_fit(mode):
    """Labels set directly (no kkm_fit: predict runs the objective pass itself); an empty
    cluster gets D = +inf and is never chosen."""
    Xa = synth.blobs(500, 4, 3, seed=9)
    Xtr, Y = Xa[:400], Xa[400:]
    init = np.zeros(400, dtype=np.int32)
    init[::3] = 2
    h = _fit(Xtr, 3, oracle.LINEAR, 1.0, 0.0, 1, 0, mode, init=init)
    lg, _ = _check_predict(h, Xtr, Y, 3, oracle.LINEAR, 1.0, 0.0, 1)
    assert not (lg == 1).any()
    h.set_labels(init)  # invalidates c; recomputed on the next predict
    _check_predict(h, Xtr, Y, 3, oracle.LINEAR, 1.0, 0.0, 1)
    h.destroy()


def test_predict_training_points_and_errors():
    """Predicting the training points reproduces the next iteration's assignment (Eq. d)."""
    X, cfg = synth.make_config("rings")
    h = _fit(X, 2, cfg["kind"], cfg["gamma"], 0.0, 1, 5, MODES[0])
    lab = h.assign().cpu().numpy()
    K = oracle.kernel_matrix(X, cfg["kind"], cfg["gamma"])
    it = oracle.iteration(K, np.diag(K).copy(), lab, 2)
    lg = h.predict(X)
    scale = 1.0 + 2 * np.abs(it["E"]).max(axis=1) + it["cnorm"].max()
    check_labels(lg, it["new_labels"], it["Dfull"], scale)
    assert h.predict(np.zeros((0, 2), dtype=np.float32)).shape == (0,)
    with pytest.raises(ValueError):
        h.predict(np.zeros((4, 3), dtype=np.float32))
    h.destroy()
    hs = _fit(X, 2, cfg["kind"], cfg["gamma"], 0.0, 1, 1, (kkm.PREC_FP32_SIMT, kkm.PATH_MATERIALIZE))
    with pytest.raises(kkm.KKMError, match="EUNSUP"):
        hs.predict(X[:5])
    hs.destroy()
