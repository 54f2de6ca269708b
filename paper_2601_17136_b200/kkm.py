"""ctypes binding of include/kkm.h (argument marshalling only; every step of the
path runs in libkkm.so). Fails loudly if the CUDA library is missing -- there is
no CPU fallback."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KKM_LIBKKM: an alternative build of the same library (`make exp`, A/B experiments only)
_LIB_PATH = os.environ.get("KKM_LIBKKM") or os.path.join(_HERE, "libkkm.so")

OK, EINVAL, ELABEL, ENOMEM, EUNSUP, ECUDA, ENCCL, ESTATE = range(8)
_NAMES = {1: "KKM_EINVAL", 2: "KKM_ELABEL", 3: "KKM_ENOMEM", 4: "KKM_EUNSUP", 5: "KKM_ECUDA",
          6: "KKM_ENCCL", 7: "KKM_ESTATE"}
KERNEL_LINEAR, KERNEL_POLY, KERNEL_GAUSSIAN = 0, 1, 2
PATH_AUTO, PATH_MATERIALIZE, PATH_STREAM = 0, 1, 2
PREC_BF16X3, PREC_FP32_SIMT, PREC_FP16X3 = 0, 1, 2
SYM_AUTO, SYM_OFF, SYM_ON = 0, 1, 2
KSTORE_AUTO, KSTORE_FP32, KSTORE_FP16, KSTORE_FP16X2 = 0, 1, 2, 3
DBG_E, DBG_CNORM, DBG_SIZES, DBG_DIAG, DBG_DFULL, DBG_LABELS_PREV = range(6)
PHASES = ("init_prep", "init_gemm", "spmm", "cnorm", "assign", "a2_kernel")


class KKMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


LAYOUT_FULL, LAYOUT_STREAM, LAYOUT_SYM_BANDS, LAYOUT_SYM_BANDS16, LAYOUT_SYM_STREAM = range(5)
XCHG_NONE, XCHG_PARTIALS, XCHG_S_ALLREDUCE, XCHG_S_REDUCE_SCATTER = range(4)


class KKMPlanInfo(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("layout", ctypes.c_int32), ("exchange", ctypes.c_int32),
                ("grid_rows", ctypes.c_int32), ("grid_cols", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("row0", ctypes.c_int64), ("nloc", ctypes.c_int64), ("a0", ctypes.c_int64), ("nA", ctypes.c_int64),
                ("b0", ctypes.c_int64), ("nB", ctypes.c_int64), ("npieces", ctypes.c_int64),
                ("ws_bytes", ctypes.c_int64)]


class KKMParams(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gamma", ctypes.c_double), ("coef0", ctypes.c_double),
                ("degree", ctypes.c_int32), ("k", ctypes.c_int32), ("max_iter", ctypes.c_int32),
                ("stop_on_no_change", ctypes.c_int32), ("path", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("timing", ctypes.c_int32),
                ("grid_rows", ctypes.c_int32), ("symmetric", ctypes.c_int32),
                ("incremental", ctypes.c_int32), ("kstore", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 2)]


_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Loads libkkm.so (after torch, so both share torch's libnccl.so.2)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: build it with `make` (or "
                              "__graft_entry__.build()); there is no CPU fallback")
        import torch  # noqa: F401  (loads the CUDA runtime + NCCL first)
        L = ctypes.CDLL(_LIB_PATH)
        P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        sig = {
            "kkm_default_params": [P],
            "kkm_workspace_size": [P, i64, i64, i32, i32, P],
            "kkm_plan_query": [P, i64, i64, i32, i32, P, P, i64],
            "kkm_init": [P, P, P, i64, i64, i64, i32, i32, P, P, ctypes.c_size_t, P, P],
            "kkm_fit": [P, P, P, P],
            "kkm_assign": [P, P],
            "kkm_objective": [P, P],
            "kkm_set_labels": [P, P],
            "kkm_predict": [P, P, i64, i64, P, P, P, ctypes.c_size_t],
            "kkm_predict_workspace_size": [P, i64, P],
            "kkm_seed_kmeanspp": [P, P, P],
            "kkm_debug_read": [P, i32, P],
            "kkm_kernel_tile": [P, i64, i64, i32, i32, P],
            "kkm_stored_k_row": [P, i64, P],
            "kkm_phase_ms": [P, P],
            "kkm_launch_count": [P, P],
            "kkm_destroy": [P],
            "kkm_get_unique_id": [P],
            "kkm_comm_init": [P, i32, i32, P],
            "kkm_comm_destroy": [P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.kkm_shard_begin.argtypes = [i64, i32, i32]
        L.kkm_shard_begin.restype = i64
        L.kkm_last_error.argtypes = []
        L.kkm_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise KKMError(rc, lib().kkm_last_error().decode(errors="replace"))


def default_params() -> KKMParams:
    p = KKMParams()
    _check(lib().kkm_default_params(ctypes.byref(p)))
    return p


def shard_begin(n: int, rank: int, nranks: int) -> int:
    return int(lib().kkm_shard_begin(n, rank, nranks))


def workspace_size(p: KKMParams, n: int, d: int, rank: int = 0, nranks: int = 1) -> int:
    b = ctypes.c_size_t(0)
    _check(lib().kkm_workspace_size(ctypes.byref(p), n, d, rank, nranks, ctypes.byref(b)))
    return int(b.value)


def plan_query(p: KKMParams, n: int, d: int, rank: int = 0, nranks: int = 1):
    """(info, pieces int64[npieces, 5]) of the C++ planner for one rank (pure host code, no CUDA)."""
    info = KKMPlanInfo()
    _check(lib().kkm_plan_query(ctypes.byref(p), n, d, rank, nranks, ctypes.byref(info), None, 0))
    pieces = np.zeros((max(int(info.npieces), 1), 5), dtype=np.int64)
    _check(lib().kkm_plan_query(ctypes.byref(p), n, d, rank, nranks, ctypes.byref(info),
                                pieces.ctypes.data_as(ctypes.c_void_p), int(info.npieces)))
    return info, pieces[:int(info.npieces)]


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().kkm_get_unique_id(buf))
    return buf.raw


def comm_init(nranks: int, rank: int, uid: bytes) -> int:
    c = ctypes.c_void_p()
    _check(lib().kkm_comm_init(ctypes.byref(c), nranks, rank, ctypes.create_string_buffer(uid, 128)))
    return c.value


def comm_destroy(comm) -> None:
    if comm:
        _check(lib().kkm_comm_destroy(ctypes.c_void_p(comm)))


def _ptr(a):
    """Data pointer of a torch tensor or numpy array (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(a.data_ptr())


class KernelKMeans:
    """One rank's handle. X_local: rows [shard_begin(rank), shard_begin(rank+1)) of X as a
    float32 torch tensor (CUDA or pinned/pageable CPU) or numpy array; copied during init."""

    def __init__(self, X_local, n: int, k: int, kind: int = KERNEL_POLY, gamma: float = 1.0,
                 coef0: float = 1.0, degree: int = 2, max_iter: int = 100,
                 stop_on_no_change: bool = False, path: int = PATH_AUTO,
                 precision: int = PREC_FP16X3, timing: bool = False, init_labels=None,
                 rank: int = 0, nranks: int = 1, comm=None, stream=None, device=None,
                 workspace=None, grid_rows: int = 1, symmetric: int = SYM_AUTO, incremental: bool = False,
                 kstore: int = KSTORE_AUTO):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.n, self.k, self.rank, self.nranks = int(n), int(k), int(rank), int(nranks)
        self.d = int(X_local.shape[1])
        ldx = int(X_local.stride(0)) if hasattr(X_local, "stride") and callable(X_local.stride) \
            else int(X_local.strides[0] // 4)
        p = default_params()
        p.kind, p.gamma, p.coef0, p.degree = kind, gamma, coef0, degree
        p.k, p.max_iter, p.stop_on_no_change = k, max_iter, int(stop_on_no_change)
        p.path, p.precision, p.timing = path, precision, int(timing)
        p.grid_rows = grid_rows
        p.symmetric = symmetric
        p.incremental = int(incremental)
        p.kstore = kstore
        self.params = p
        self.max_iter = max_iter
        nb = workspace_size(p, self.n, self.d, rank, nranks)
        if workspace is None:
            workspace = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.device)
        self.workspace = workspace
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        self.n_local = shard_begin(self.n, rank + 1, nranks) - shard_begin(self.n, rank, nranks)
        if isinstance(init_labels, np.ndarray):
            init_labels = np.ascontiguousarray(init_labels, dtype=np.int32)
        h = ctypes.c_void_p()
        _check(lib().kkm_init(ctypes.byref(h), ctypes.byref(p), _ptr(X_local), self.n, self.d, ldx,
                              rank, nranks, _ptr(init_labels), _ptr(self.workspace),
                              self.workspace.numel(), ctypes.c_void_p(self.stream.cuda_stream),
                              ctypes.c_void_p(comm) if comm else None))
        self.h = h

    # ---- C-ABI mirrors
    def fit(self):
        it = ctypes.c_int32(0)
        J = np.zeros(self.max_iter + 1, dtype=np.float64)
        ch = np.zeros(max(self.max_iter, 1), dtype=np.int64)
        _check(lib().kkm_fit(self.h, ctypes.byref(it), _ptr(J), _ptr(ch)))
        t = it.value
        return t, J[:t + 1], ch[:t]

    def assign(self, out=None):
        if out is None:
            out = self.torch.empty(self.n, dtype=self.torch.int32, device=self.device)
        _check(lib().kkm_assign(self.h, _ptr(out)))
        return out

    def objective(self) -> float:
        J = ctypes.c_double(0.0)
        _check(lib().kkm_objective(self.h, ctypes.byref(J)))
        return J.value

    def set_labels(self, labels):
        if isinstance(labels, np.ndarray):
            labels = np.ascontiguousarray(labels, dtype=np.int32)
        _check(lib().kkm_set_labels(self.h, _ptr(labels)))

    def seed_kmeanspp(self, seed: int = 0, u=None) -> np.ndarray:
        """K-means++ seeding in feature space (kkm_seed_kmeanspp); replaces the current labels.
        u: the k uniforms in [0, 1) (default: numpy's generator seeded with `seed`). Returns the
        k center indices."""
        u = np.random.default_rng(seed).random(self.k) if u is None else u
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.shape != (self.k,):
            raise ValueError(f"u must hold k = {self.k} uniforms")
        centers = np.empty(self.k, dtype=np.int64)
        _check(lib().kkm_seed_kmeanspp(self.h, _ptr(u), _ptr(centers)))
        return centers

    def predict(self, Y, return_distances: bool = False, use_workspace: bool = True):
        """Out-of-sample assignment of the rows of Y (host numpy or device tensor, m x d fp32)
        to the clusters of the current labels (kkm_predict). Returns int32 labels (numpy for
        numpy input, else a tensor on the handle's device), plus the m x k fp64 distances.
        The scratch is a cached device buffer (use_workspace=False: the library allocates
        stream-ordered scratch per call instead)."""
        on_host = isinstance(Y, np.ndarray)
        if on_host:
            Y = np.ascontiguousarray(Y, dtype=np.float32)
            m, ldy = Y.shape[0], (Y.shape[1] if Y.ndim == 2 else 0)
        else:
            if Y.dtype != self.torch.float32 or Y.stride(-1) != 1:
                raise ValueError("Y must be fp32 with unit column stride")
            m, ldy = Y.shape[0], Y.stride(0)
        if Y.ndim != 2 or Y.shape[1] != self.d:
            raise ValueError(f"Y must be m x {self.d}")
        if on_host:
            lab = np.empty(m, dtype=np.int32)
            D = np.empty((m, self.k), dtype=np.float64) if return_distances else None
        else:
            lab = self.torch.empty(m, dtype=self.torch.int32, device=self.device)
            D = (self.torch.empty((m, self.k), dtype=self.torch.float64, device=self.device)
                 if return_distances else None)
        ws, nws = None, 0
        if use_workspace:
            nb = ctypes.c_size_t(0)
            _check(lib().kkm_predict_workspace_size(self.h, m, ctypes.byref(nb)))
            ws = getattr(self, "_predict_ws", None)
            if ws is None or ws.numel() < nb.value:  # kept across calls
                self._predict_ws = None
                ws = self._predict_ws = self.torch.empty(max(nb.value, 256), dtype=self.torch.uint8,
                                                         device=self.device)
            nws = ws.numel()
        _check(lib().kkm_predict(self.h, _ptr(Y), m, ldy, _ptr(lab), _ptr(D), _ptr(ws), nws))
        return (lab, D) if return_distances else lab

    def debug_read(self, what: int) -> np.ndarray:
        shapes = {DBG_E: ((self.n_local, self.k), np.float64), DBG_CNORM: ((self.k,), np.float64),
                  DBG_SIZES: ((self.k,), np.int32), DBG_DIAG: ((self.n_local,), np.float64),
                  DBG_DFULL: ((self.n_local, self.k), np.float64),
                  DBG_LABELS_PREV: ((self.n,), np.int32)}
        shape, dt = shapes[what]
        out = np.zeros(shape, dtype=dt)
        _check(lib().kkm_debug_read(self.h, what, _ptr(out)))
        return out

    def kernel_tile(self, i0: int, j0: int, m: int, nc: int) -> np.ndarray:
        out = np.zeros((m, nc), dtype=np.float32)
        _check(lib().kkm_kernel_tile(self.h, i0, j0, m, nc, _ptr(out)))
        return out

    def stored_k_row(self, i: int) -> np.ndarray:
        """Row i of the K this rank stored (kkm_stored_k_row): n doubles, NaN where not stored."""
        out = np.empty(self.n, dtype=np.float64)
        _check(lib().kkm_stored_k_row(self.h, int(i), _ptr(out)))
        return out

    def phase_ms(self) -> dict:
        ms = (ctypes.c_float * len(PHASES))()
        _check(lib().kkm_phase_ms(self.h, ms))
        return dict(zip(PHASES, list(ms)))

    def launch_count(self) -> int:
        c = ctypes.c_int64(0)
        _check(lib().kkm_launch_count(self.h, ctypes.byref(c)))
        return c.value

    def destroy(self):
        """Destroys the handle and drops the binding's device buffers (the workspace it
        allocated, the predict scratch), so their memory returns to torch's allocator."""
        if getattr(self, "h", None):
            _check(lib().kkm_destroy(self.h))
            self.h = None
        self.workspace = None
        self._predict_ws = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
