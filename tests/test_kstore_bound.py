"""CPU check of the error bounds DESIGN.md A27 derives for 16-bit K storage (used as the GPU
tolerances in tests/test_gpu_kstore.py): K stored as RN_fp16(K 2^e) (FP16) or as hi + lo with
lo = RN_fp16(K 2^e - hi) (FP16X2), 2^e the largest power of two with bound(|K|) 2^e <= 60000.
numpy's float16 rounds to nearest even like the GPU's cvt.rn.f16.f32, so the emulation below
stores exactly what the epilogue stores (from the fp64 K of the oracle instead of the fp32 one).
The quantities are computed by the oracle (oracle.E_rows / cnorm / objective / assign) from the
emulated K and compared with the same quantities from the exact K."""
import numpy as np
import pytest

import oracle
import synth

U = 2.0 ** -11


def scale_exp(kmax):
    return int(np.floor(np.log2(60000.0 / (kmax * 1.0001))))


def stored(K, kmax, planes):
    e = scale_exp(kmax)
    Ks = (K * 2.0 ** e).astype(np.float32)
    hi = Ks.astype(np.float16).astype(np.float64)
    if planes == 1:
        return hi * 2.0 ** -e
    lo = (Ks - hi.astype(np.float32)).astype(np.float16).astype(np.float64)  # residual exact in fp32
    return (hi + lo) * 2.0 ** -e


@pytest.mark.parametrize("name,n,kind", [("mnist60k", 600, oracle.POLY), ("har200k", 500, oracle.GAUSSIAN),
                                         ("rings", 400, oracle.GAUSSIAN)])
def test_a27_bounds(name, n, kind):
    X, cfg = synth.make_config(name, n=n)
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    K = oracle.kernel_matrix(X, *args)
    diag = oracle.kernel_diag(X, *args)
    norms = (X.astype(np.float64) ** 2).sum(axis=1)
    kmax = {oracle.LINEAR: norms.max(), oracle.POLY: (cfg["gamma"] * norms.max() + abs(cfg["coef0"])) ** cfg["degree"],
            oracle.GAUSSIAN: 1.0}[kind]
    assert np.abs(K).max() <= kmax * (1 + 1e-12)  # the storage bound covers |K| (|K_ij| <= max K_ii)
    k = cfg["k"]
    labels = np.random.default_rng(0).integers(0, k, n).astype(np.int32)
    E = oracle.E_rows(K, labels, k)
    cn = oracle.cnorm(E, labels, k)
    J = oracle.objective(diag, labels, k, cn)
    _, D = oracle.assign(E, diag, cn)
    scale = np.abs(diag) + 2 * np.abs(E).max(axis=1) + cn[np.isfinite(cn)].max()
    for planes, rel in ((1, U), (2, 2.0 ** -21)):
        Kq = stored(K, kmax, planes)
        # per value: the 16-bit rounding (relative), the fp32 K it is made from (2^-24, relative)
        # and the fp16 subnormal floor 2^-25 of the scaled value (absolute, x 2^-e unscaled)
        floor = 2.0 ** -25 * 2.0 ** -scale_exp(kmax)
        assert (np.abs(Kq - K) <= (rel + 2.0 ** -24) * np.abs(K) + floor).all()
        Eq = oracle.E_rows(Kq, labels, k)
        cq = oracle.cnorm(Eq, labels, k)
        Jq = oracle.objective(diag, labels, k, cq)  # tr K from the exact diagonal, as on the GPU
        _, Dq = oracle.assign(Eq, diag, cq)
        assert (np.abs(Eq - E) <= rel * scale[:, None]).all()
        assert (np.abs(cq - cn) <= rel * scale.max()).all()
        assert (np.abs(Dq - D) <= 3 * rel * scale[:, None]).all()
        jb = sum(np.abs(K[np.ix_(labels == c, labels == c)]).sum() / max((labels == c).sum(), 1) for c in range(k))
        assert abs(Jq - J) <= rel * jb + 1e-12 * abs(J)
        if planes == 2:  # hi + lo is fp32-class: within the standard 1e-4 / 1e-5 rules with room
            assert (np.abs(Dq - D) <= 1e-6 * scale[:, None]).all()
            assert abs(Jq - J) <= 1e-7 * abs(J) + 1e-9 * np.abs(diag).sum()
