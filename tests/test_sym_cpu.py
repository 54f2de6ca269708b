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


def stream_units(n, tile, block, P):
    """tc2_stream_sym units as make_plan builds them: (row tile, globally aligned column block
    of <= `block` tiles, from the row tile's own tile on), spread largest first to the
    least-loaded rank (stable order), each rank's list in row-major order."""
    T = -(-n // tile)
    allu = [(tm, max(tm, b * block), min(T, (b + 1) * block) - max(tm, b * block))
            for tm in range(T) for b in range(tm // block, -(-T // block))]
    order = sorted(range(len(allu)), key=lambda i: -allu[i][2])  # stable
    load, owner = [0] * P, [0] * len(allu)
    for i in order:
        r = min(range(P), key=lambda q: (load[q], q))
        load[r] += allu[i][2]
        owner[i] = r
    return [[u for i, u in enumerate(allu) if owner[i] == r] for r in range(P)]


@pytest.mark.parametrize("n,tile,block,P", [(37, 8, 2, 1), (37, 8, 2, 3), (64, 8, 3, 2), (50, 4, 64, 4)])
def test_symmetric_streaming_decomposition(n, tile, block, P):
    """Upper-triangle tiles of the label-sorted K: row sums by the column segments on every
    tile, column sums by the row segments off the diagonal tiles, summed in int64 fixed point
    over the ranks == S from the full K (exactly the same integers for any P)."""
    X = synth.blobs(n, 3, 4, seed=n + P)
    lab = (np.arange(n) * 5 + 1) % 4
    perm = np.argsort(lab, kind="stable")  # the label-sorted order
    Ks = oracle.kernel_matrix(X, oracle.POLY, 0.5, 1.0, 2)[np.ix_(perm, perm)]
    ls = lab[perm]
    scale = 2.0 ** 30

    def fx(v):
        return np.rint(v * scale).astype(np.int64)

    Sfix = np.zeros((n, 4), dtype=np.int64)
    for units in stream_units(n, tile, block, P):
        for tm, tn0, ntn in units:
            r0, r1 = tm * tile, min(n, (tm + 1) * tile)
            for tn in range(tn0, tn0 + ntn):
                c0, c1 = tn * tile, min(n, (tn + 1) * tile)
                blk = Ks[r0:r1, c0:c1]
                for c in range(4):  # row part, by the column labels
                    Sfix[r0:r1, c] += fx(blk[:, ls[c0:c1] == c].sum(axis=1))
                if tn != tm:  # column part off the diagonal tile, by the row labels
                    for c in range(4):
                        Sfix[c0:c1, c] += fx(blk[ls[r0:r1] == c].sum(axis=0))
    S = Sfix / scale
    S_ref = np.stack([Ks[:, ls == c].sum(axis=1) for c in range(4)], axis=1)
    assert np.allclose(S, S_ref, rtol=1e-7, atol=1e-6)
    # every upper-triangle tile exactly once
    T = -(-n // tile)
    seen = sorted((tm, tn) for units in stream_units(n, tile, block, P) for tm, tn0, nt in units
                  for tn in range(tn0, tn0 + nt))
    assert seen == [(a, b) for a in range(T) for b in range(a, T)]
