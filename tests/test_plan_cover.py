"""Virtual ranks on the CPU: the C++ planner (kkm_plan_query, the same make_plan that kkm_init
runs; no CUDA) is asked what every rank of P = 1..8 (1D, and the 1.5D grids 2x2, 2x4, 4x2)
computes, and the union of the ranks' rectangles is checked against the method:
  coverage -- the row parts and (by symmetry) the column parts of all ranks touch every
              entry (i, j) of K exactly once (of the label-sorted K for the streaming f1 layout);
  S / a3 / a4 -- the ranks' contributions, evaluated with the oracle's fp64 K and summed as the
              exchange step sums them (S allreduce / reduce-scatter), give E = K V^T (Eq. e) and
              then the oracle's c, J, Dfull and labels (Eqs. c, d; A6-A8).
The per-rank arithmetic is the oracle's; what is under test is the library's own decomposition
(bands, 512-row pieces, upper-triangle units, grids) for rank counts no GPU box here offers."""
import numpy as np
import pytest

import oracle
import synth

kkm = pytest.importorskip("paper_2601_17136_b200")

CASES = [  # (name, path, symmetric, kstore, grid_rows, expected layout)
    ("full-K", kkm.PATH_MATERIALIZE, kkm.SYM_OFF, kkm.KSTORE_FP32, 1, kkm.LAYOUT_FULL),
    ("stream", kkm.PATH_STREAM, kkm.SYM_OFF, kkm.KSTORE_AUTO, 1, kkm.LAYOUT_STREAM),
    ("sym-bands-fp32", kkm.PATH_MATERIALIZE, kkm.SYM_ON, kkm.KSTORE_FP32, 1, kkm.LAYOUT_SYM_BANDS),
    ("sym-bands-16", kkm.PATH_MATERIALIZE, kkm.SYM_ON, kkm.KSTORE_FP16X2, 1, kkm.LAYOUT_SYM_BANDS16),
    ("sym-stream", kkm.PATH_STREAM, kkm.SYM_AUTO, kkm.KSTORE_AUTO, 1, kkm.LAYOUT_SYM_STREAM),
]
GRIDS = [(4, 2), (8, 2), (8, 4), (2, 2)]  # (P, grid_rows): 1.5D, full K rows and streaming


def params(k, path, sym, kstore, grid_rows):
    p = kkm.default_params()
    p.k, p.kind, p.path, p.precision = k, kkm.KERNEL_GAUSSIAN, path, kkm.PREC_FP16X3
    p.symmetric, p.kstore, p.grid_rows = sym, kstore, grid_rows
    return p


def all_pieces(p, n, d, P):
    infos, pieces = [], []
    for r in range(P):
        info, pc = kkm.plan_query(p, n, d, rank=r, nranks=P)
        infos.append(info)
        pieces.append(pc)
    return infos, pieces


def coverage(pieces_by_rank, n):
    C = np.zeros((n, n), dtype=np.int16)
    for pcs in pieces_by_rank:
        for r0, nr, c0, nc, cd in pcs:
            C[r0:r0 + nr, c0:c0 + nc] += 1              # row part
            if cd < c0 + nc:                            # column part of the columns >= cdiag
                a = max(cd, c0)
                C[a:c0 + nc, r0:r0 + nr] += 1
    return C


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_plan_covers_K_exactly_once(case, P):
    name, path, sym, kstore, gr, layout = case
    n, d, k = 9001, 64, 10
    infos, pcs = all_pieces(params(k, path, sym, kstore, gr), n, d, P)
    assert all(i.layout == layout for i in infos), [i.layout for i in infos]
    C = coverage(pcs, n)
    assert C.min() == 1 and C.max() == 1, (C.min(), C.max())
    # the 1D blocks partition the points (kkm_shard_begin)
    assert [i.row0 for i in infos] == [kkm.shard_begin(n, r, P) for r in range(P)]
    assert sum(i.nloc for i in infos) == n
    if P > 1:
        xchg = {kkm.LAYOUT_FULL: kkm.XCHG_PARTIALS, kkm.LAYOUT_STREAM: kkm.XCHG_PARTIALS}.get(
            layout, kkm.XCHG_S_ALLREDUCE)
        assert all(i.exchange == xchg for i in infos)


@pytest.mark.parametrize("P,gr", GRIDS)
@pytest.mark.parametrize("path", [kkm.PATH_MATERIALIZE, kkm.PATH_STREAM], ids=["mat", "stream"])
def test_grid_15d_covers_K_exactly_once(P, gr, path):
    """Alg. 2: rank (i, j) = i + j pr computes the K tile [column block j] x [row block i]."""
    n, d, k = 7001, 64, 10
    infos, pcs = all_pieces(params(k, path, kkm.SYM_AUTO, kkm.KSTORE_AUTO, gr), n, d, P)
    assert all(i.grid_rows == gr and i.grid_cols == P // gr for i in infos)
    assert all(i.layout in (kkm.LAYOUT_FULL, kkm.LAYOUT_STREAM) for i in infos)
    C = coverage(pcs, n)
    assert C.min() == 1 and C.max() == 1


def simulate_S(pcs_by_rank, K, labels, k):
    """sum over ranks of each rank's row + column parts (the exchange step's sum)."""
    n = K.shape[0]
    S = np.zeros((n, k))
    V = np.zeros((n, k))
    V[np.arange(n), labels] = 1.0
    for pcs in pcs_by_rank:
        Sr = np.zeros((n, k))
        for r0, nr, c0, nc, cd in pcs:
            Sr[r0:r0 + nr] += K[r0:r0 + nr, c0:c0 + nc] @ V[c0:c0 + nc]
            if cd < c0 + nc:
                a = max(cd, c0)
                Sr[a:c0 + nc] += K[r0:r0 + nr, a:c0 + nc].T @ V[r0:r0 + nr]
        S += Sr
    return S


@pytest.mark.parametrize("P", [2, 8])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_virtual_ranks_iteration_equals_oracle(case, P):
    """One iteration assembled from the P ranks' contributions equals the 1-rank oracle iteration
    (E, c, J, Dfull, labels); the streaming f1 layout works on the label-sorted K (stable sort)."""
    name, path, sym, kstore, gr, layout = case
    X, cfg = synth.make_config("har200k", n=3001)
    k = 6
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    K = oracle.kernel_matrix(X, *args)
    diag = np.diag(K).copy()
    labels = oracle.round_robin(3001, k)
    labels[::7] = 2
    ref = oracle.iteration(K, diag, labels, k)
    _, pcs = all_pieces(params(k, path, sym, kstore, gr), 3001, X.shape[1], P)
    if layout == kkm.LAYOUT_SYM_STREAM:
        perm = np.argsort(labels, kind="stable")          # sorted position -> point (sort.cuh)
        Ss = simulate_S(pcs, K[np.ix_(perm, perm)], labels[perm], k)
        S = np.empty_like(Ss)
        S[perm] = Ss
    else:
        S = simulate_S(pcs, K, labels, k)
    sizes = np.bincount(labels, minlength=k)
    E = S / sizes
    assert np.allclose(E, ref["E"], rtol=1e-12, atol=1e-12)
    cn = oracle.cnorm(E, labels, k)
    J = oracle.objective(diag, labels, k, cn)
    new, D = oracle.assign(E, diag, cn)
    assert np.allclose(cn, ref["cnorm"], rtol=1e-12)
    assert abs(J - ref["J"]) <= 1e-12 * abs(ref["J"])
    assert np.array_equal(new, ref["new_labels"])
    assert np.allclose(D, ref["Dfull"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sym_stream_ranks_balanced_at_config4_size(P):
    """Streaming f1 at the config-4 size (n = 1M): each rank's contiguous run of the unit order
    holds 1/P of the upper-triangle tiles to within one unit (16 tiles), and the runs together
    are the whole triangle."""
    n = 1_000_000
    T = -(-n // 256)
    tiles = []
    for r in range(P):
        info, pc = kkm.plan_query(params(10, kkm.PATH_STREAM, kkm.SYM_AUTO, kkm.KSTORE_AUTO, 1), n, 784, rank=r,
                                  nranks=P)
        assert info.layout == kkm.LAYOUT_SYM_STREAM
        tiles.append(int(np.sum(-(-pc[:, 3] // 256))))   # column tiles of each unit
    assert sum(tiles) == T * (T + 1) // 2
    assert max(tiles) - min(tiles) <= 2 * 16, tiles
