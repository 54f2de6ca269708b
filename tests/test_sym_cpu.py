"""f1 (symmetric K storage, csrc/sym.cuh) schedule on CPU: bands of TB rows storing only the
columns j >= band start, spread over P ranks largest-first to the least-loaded rank; each rank's
S = row part (its bands, by column labels) + column part (its bands' off-diagonal tiles, by the
rows' labels, landing on the rows of later bands). Summed over ranks (the ReduceScatter) this
must equal S = K V^T-style sums from the full K (oracle), for ragged bands and any P. The
band sizes are scaled down (TB = 8) so the cases stay tiny."""
import numpy as np
import pytest

import oracle
import synth


def lpt_owner(n, TB, P):
    T = -(-n // TB)
    load = [0.0] * P
    owner = []
    for I in range(T):
        rows = min(TB, n - I * TB)
        ldb = -(-(n - I * TB) // 32) * 32
        r = min(range(P), key=lambda q: (load[q], q))
        load[r] += rows * ldb
        owner.append(r)
    return owner


def rank_S(K, lab, k, TB, owner, rank):
    n = K.shape[0]
    S = np.zeros((n, k))
    for I, r in enumerate(owner):
        if r != rank:
            continue
        i0, i1 = I * TB, min(n, (I + 1) * TB)
        band = K[i0:i1, i0:]                     # the stored band (upper triangle + diagonal tile)
        for c in range(k):                       # row part: by the labels of the columns
            S[i0:i1, c] += band[:, lab[i0:] == c].sum(axis=1)
        off = band[:, i1 - i0:]                  # column part: off-diagonal tiles only
        for c in range(k):                       # by the labels of the band's rows
            S[i1:, c] += off[lab[i0:i1] == c].sum(axis=0)
    return S


@pytest.mark.parametrize("n,TB,P", [(37, 8, 1), (37, 8, 2), (64, 8, 3), (41, 8, 4), (5, 8, 2), (96, 32, 3)])
def test_symmetric_decomposition(n, TB, P):
    X = synth.blobs(n, 3, 4, seed=n)
    K = oracle.kernel_matrix(X, oracle.POLY, 0.5, 1.0, 2)
    lab = (np.arange(n) * 7 + 3) % 4
    owner = lpt_owner(n, TB, P)
    S = sum(rank_S(K, lab, 4, TB, owner, r) for r in range(P))
    sizes = np.bincount(lab, minlength=4)
    E_ref = oracle.E_rows(K, lab, 4)
    assert np.allclose(S / np.maximum(sizes, 1), E_ref, rtol=1e-12, atol=1e-9)


def test_lpt_balances_area():
    owner = lpt_owner(60000, 1024, 4)
    area = np.zeros(4)
    for I, r in enumerate(owner):
        area[r] += min(1024, 60000 - I * 1024) * (60000 - I * 1024)
    assert area.max() < 1.1 * area.min()
