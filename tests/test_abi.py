"""CPU-only checks of the C-ABI boundary: libkkm.so loads, exports every function
include/kkm.h declares, and the pure (no-CUDA) entry points validate arguments."""
import ctypes
import os
import re

import pytest

import paper_2601_17136_b200 as kkm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "kkm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kkm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 17, names
    L = ctypes.CDLL(kkm.lib_path())
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_library_is_sm100a_and_in_tree():
    path = kkm.lib_path()
    assert os.path.dirname(path) == os.path.join(ROOT, "paper_2601_17136_b200")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_default_params_and_shards():
    p = kkm.default_params()
    assert (p.kind, p.gamma, p.coef0, p.degree, p.max_iter) == (kkm.KERNEL_POLY, 1.0, 1.0, 2, 100)
    for n, P in [(10, 3), (60000, 8), (5, 4), (1, 1)]:
        b = [kkm.shard_begin(n, r, P) for r in range(P + 1)]
        assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
        B = -(-n // P)
        assert all(y - x == B for x, y in zip(b, b[1:]) if y < n)
    assert kkm.shard_begin(5, -1, 2) == -1


def test_workspace_size_and_errors():
    p = kkm.default_params()
    p.k = 10
    nb = kkm.workspace_size(p, 60000, 784)
    ldk = 60000
    assert nb >= 60000 * ldk * 4 / 2  # K materialised (upper-triangle bands by default, f1)
    nb2 = kkm.workspace_size(p, 60000, 784, rank=1, nranks=4)
    assert nb2 < nb / 3
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(p, 5, 784)  # k > n
    q = kkm.default_params()
    q.k, q.kind, q.gamma = 3, kkm.KERNEL_GAUSSIAN, -1.0
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(q, 100, 4)
    q = kkm.default_params()
    q.k, q.degree = 3, 0
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(q, 100, 4)
    q = kkm.default_params()
    q.k, q.path, q.precision = 3, kkm.PATH_STREAM, kkm.PREC_FP32_SIMT
    with pytest.raises(kkm.KKMError, match="EUNSUP"):
        kkm.workspace_size(q, 100, 4)  # streaming needs a tensor-core precision
    q = kkm.default_params()
    q.k, q.path = 70, kkm.PATH_STREAM  # k > 16 streams in groups of 16 clusters
    assert kkm.workspace_size(q, 100, 4) > 0
    q = kkm.default_params()
    q.k = 10
    nb_stream = kkm.workspace_size(q, 1_000_000, 784)  # 4 TB of K: AUTO streams
    assert nb_stream < 20e9
    q.path = kkm.PATH_STREAM
    assert kkm.workspace_size(q, 1_000_000, 784) == nb_stream
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(p, 60000, 784, rank=4, nranks=4)
    q = kkm.default_params()
    q.k, q.grid_rows = 3, 3
    with pytest.raises(kkm.KKMError, match="EUNSUP"):
        kkm.workspace_size(q, 100, 4, rank=0, nranks=4)  # 3 does not divide 4
    q.grid_rows = 2  # 2 x 2 grid: K tile = column block (2 of 4 blocks) x row block (2 of 4)
    nb_15 = kkm.workspace_size(q, 60000, 784, rank=1, nranks=4)
    q.grid_rows = 1
    q.symmetric = kkm.SYM_OFF
    nb_1d = kkm.workspace_size(q, 60000, 784, rank=1, nranks=4)
    assert abs(nb_15 - nb_1d) < 0.05 * nb_1d  # same K-tile size, n^2 / P
    # f1: the symmetric bands hold ~n^2/2 floats (+ 1/R of them as column partials with fp32
    # storage), spread over the ranks by area
    q.symmetric = kkm.SYM_AUTO
    q.kstore = kkm.KSTORE_FP32
    kfull = 60000 * 60000 * 4
    nb_sym1 = kkm.workspace_size(q, 60000, 784)
    q.symmetric = kkm.SYM_OFF
    nb_full1 = kkm.workspace_size(q, 60000, 784)
    assert nb_full1 - kfull < 0.05 * kfull  # + X, its split copies and the small arrays
    assert 0.5 * kfull < nb_sym1 < 0.62 * kfull
    q.symmetric = kkm.SYM_AUTO
    shares = [kkm.workspace_size(q, 60000, 784, rank=r, nranks=4) for r in range(4)]
    assert max(shares) < 1.1 * min(shares) and sum(shares) < 0.7 * kfull
    q.symmetric = 3
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(q, 100, 4)
    q = kkm.default_params()
    q.reserved[1] = 1
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(q, 100, 4)
    # f4 fp16 K storage: half the band bytes, no fp32 column partials; only where it applies
    q = kkm.default_params()
    q.k = 10
    q.kstore = kkm.KSTORE_FP16
    nb_h = kkm.workspace_size(q, 60000, 784)
    assert 0.45 * nb_sym1 < nb_h < 0.5 * nb_sym1
    q.kstore = kkm.KSTORE_FP16X2  # hi + lo planes: the fp32 band bytes, still no fp32 column partials
    nb_h2 = kkm.workspace_size(q, 60000, 784)
    assert 0.85 * nb_sym1 < nb_h2 < 0.95 * nb_sym1
    q.kstore = kkm.KSTORE_AUTO  # = FP16X2 where the bands are stored with a tensor-core precision
    assert kkm.workspace_size(q, 60000, 784) == nb_h2
    q.precision = kkm.PREC_FP32_SIMT  # ... else fp32
    assert kkm.workspace_size(q, 60000, 784) > nb_h2
    q.precision = kkm.PREC_FP16X3
    q.kstore = 4
    with pytest.raises(kkm.KKMError, match="EINVAL"):
        kkm.workspace_size(q, 100, 4)
    for field, value in (("precision", kkm.PREC_FP32_SIMT), ("symmetric", kkm.SYM_OFF),
                         ("path", kkm.PATH_STREAM), ("grid_rows", 2)):
        q = kkm.default_params()
        q.kstore = kkm.KSTORE_FP16
        setattr(q, field, value)
        with pytest.raises(kkm.KKMError, match="EUNSUP"):
            kkm.workspace_size(q, 60000, 784, rank=0, nranks=2 if field == "grid_rows" else 1)
    q = kkm.default_params()
    q.kstore, q.k = kkm.KSTORE_FP16, 32  # 16-bit bands: 16- or 32-label one-hots (spmm_tc_kernel<NL>)
    assert kkm.workspace_size(q, 60000, 784) > 0
    q.k = 33
    with pytest.raises(kkm.KKMError, match="EUNSUP"):
        kkm.workspace_size(q, 60000, 784)
