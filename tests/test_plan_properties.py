"""Property test of the C++ planner (kkm_workspace_size: pure host code, no CUDA) over random
parameters: every combination either plans (positive, 256-byte-granular size; ranks of one job
plan consistently) or fails with a documented status -- never a crash or a silent mismatch."""
import pytest

hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

import paper_2601_17136_b200 as kkm  # noqa: E402

ERRS = ("EINVAL", "EUNSUP")


@settings(max_examples=300, deadline=None)
@given(n=st.integers(1, 300000), d=st.integers(1, 1200), k=st.integers(1, 80), nranks=st.sampled_from([1, 2, 3, 4, 8]),
       grid_rows=st.sampled_from([0, 1, 2, 4]), path=st.sampled_from([0, 1, 2]), prec=st.sampled_from([0, 1, 2]),
       sym=st.sampled_from([0, 1, 2]), inc=st.sampled_from([0, 1]), kind=st.sampled_from([0, 1, 2]),
       kstore=st.sampled_from([0, 1, 2, 3]))
def test_workspace_plan(n, d, k, nranks, grid_rows, path, prec, sym, inc, kind, kstore):
    p = kkm.default_params()
    p.k, p.kind, p.path, p.precision, p.symmetric, p.incremental = k, kind, path, prec, sym, inc
    p.kstore = kstore
    p.grid_rows = grid_rows
    sizes, errs = [], []
    for r in range(nranks):
        try:
            sizes.append(kkm.workspace_size(p, n, d, rank=r, nranks=nranks))
        except kkm.KKMError as e:
            errs.append(str(e))
    if errs:  # the plan is rank-independent: every rank fails, with a documented status
        assert len(errs) == nranks and all(any(c in m for c in ERRS) for m in errs), errs
        if k > n:
            assert all("EINVAL" in m for m in errs)
        return
    assert all(s > 0 and s % 256 == 0 for s in sizes)
    # documented rejections did not happen: k <= n, grid_rows divides nranks, incremental is 1D
    assert k <= n and (grid_rows <= 1 or nranks % grid_rows == 0)
    if inc:
        assert grid_rows <= 1 and prec != kkm.PREC_FP32_SIMT
    if path == kkm.PATH_STREAM:
        assert prec != kkm.PREC_FP32_SIMT
    if kstore in (kkm.KSTORE_FP16, kkm.KSTORE_FP16X2):  # 16-bit bands: materialised 1D f1 only
        assert prec != kkm.PREC_FP32_SIMT and k <= 32 and grid_rows <= 1 and sym != kkm.SYM_OFF  # NL = 16 or 32
        assert path != kkm.PATH_STREAM
        # the bands (about n^2 / 2 values over the ranks) at 2 or 4 bytes per value
        tot = sum(sizes)
        per = 2 if kstore == kkm.KSTORE_FP16 else 4
        assert tot >= 0.45 * per * n * n * 0.999 - 1e6
