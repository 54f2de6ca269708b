"""Parity rules between the CUDA path and the fp64 oracle.

tau = 1e-4 (BASELINE.json north_star: "Kernel values and distances must agree within 1e-4
relative in the stated GPU precision"), with "relative" made well defined near zero:
  K:      |dK_ij| <= tau * max(|K_ij|, sqrt(K_ii K_jj))
  E, D:   |dD_ic| <= tau * scale_i,  scale_i = K_ii + 2 max_c |E_ic| + max_{c non-empty} c_c
  c:      |dc_c|  <= tau * max_i scale_i
  labels: identical, except where the GPU's pick is within 2 tau scale_i of the oracle's
          minimum (a near tie: "identical except for points whose best/second-best gap is
          below that tolerance")
  sizes:  bit-exact when the labels are identical
  J:      |dJ| <= max(1e-5 |J|, 1e-7 tr K)   ("final objective within 1e-5 relative"; the
          floor is the fp32 storage error of K (the paper's precision), ~2^-24 per
          entry: J = sum_i (K_ii - z_i) carries ~6e-8 tr K of rounding, so relative error is
          meaningless as J -> 0, e.g. k = n singletons where J = 0 exactly)
"""
import numpy as np

TAU = 1e-4
TAU_J = 1e-5


def j_tol(J, diag):
    return max(TAU_J * abs(J), 1e-7 * float(np.sum(np.abs(diag))))


def check_kernel_values(Kg, Kr, diag_rows, diag_cols, tau=TAU):
    Kg = np.asarray(Kg, dtype=np.float64)
    bound = tau * np.maximum(np.abs(Kr), np.sqrt(np.outer(diag_rows, diag_cols)))
    err = np.abs(Kg - Kr)
    bad = err > bound
    assert not bad.any(), (f"{bad.sum()} K entries out of tolerance; worst rel "
                           f"{(err / np.maximum(bound / tau, 1e-300)).max():.3e}")
    return float((err / np.maximum(bound / tau, 1e-300)).max())


def row_scale(E_ref, diag, cnorm_ref):
    fin = np.isfinite(cnorm_ref)
    cmax = cnorm_ref[fin].max() if fin.any() else 0.0
    return np.abs(diag) + 2.0 * np.abs(E_ref).max(axis=1) + abs(cmax)


def check_labels(lab_g, lab_r, Dfull_ref, scale, tau=TAU):
    lab_g = np.asarray(lab_g)
    lab_r = np.asarray(lab_r)
    diff = np.nonzero(lab_g != lab_r)[0]
    if diff.size:
        rows = np.arange(Dfull_ref.shape[0])
        dmin = Dfull_ref[rows, lab_r]
        dpick = Dfull_ref[rows, lab_g]
        near = dpick <= dmin + 2 * tau * scale
        bad = diff[~near[diff]]
        assert bad.size == 0, f"{bad.size} label mismatches that are not near-ties (rows {bad[:10]})"
    return int(diff.size)


def check_iteration(gpu, ref, diag, tau=TAU, rows=None):
    """gpu/ref dicts with E, cnorm, Dfull, new_labels (and optionally sizes, J).
    rows: global indices of the sampled rows E/Dfull refer to (None = all)."""
    scale = row_scale(ref["E"], diag, ref["cnorm"])
    for key in ("E", "Dfull"):
        with np.errstate(invalid="ignore"):  # inf - inf on empty clusters (checked below)
            err = np.abs(np.asarray(gpu[key]) - ref[key])
        fin = np.isfinite(ref[key])
        assert np.array_equal(np.isfinite(gpu[key]), fin), key
        bound = tau * scale[:, None]
        bad = (err > bound) & fin
        assert not bad.any(), f"{key}: {bad.sum()} entries out of tolerance, worst {np.nanmax(err / bound):.3e}"
    fin = np.isfinite(ref["cnorm"])
    assert np.array_equal(np.isfinite(gpu["cnorm"]), fin)
    cerr = np.abs(gpu["cnorm"][fin] - ref["cnorm"][fin])
    assert (cerr <= tau * scale.max()).all(), cerr.max()
    nmis = check_labels(gpu["new_labels"], ref["new_labels"], ref["Dfull"], scale, tau)
    if "sizes" in gpu and "sizes" in ref:
        assert np.array_equal(np.asarray(gpu["sizes"]), np.asarray(ref["sizes"]))
    if "J" in gpu and "J" in ref and rows is None:
        assert abs(gpu["J"] - ref["J"]) <= j_tol(ref["J"], diag), (gpu["J"], ref["J"])
    return nmis
