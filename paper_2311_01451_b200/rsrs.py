"""Thin ctypes binding of librsrs.so (include/rsrs.h) -- argument marshalling only.

Every step of the factorization, solve and apply runs in the library's own
sm_100a kernels.  PyTorch supplies device memory and streams (tensors are
passed by data_ptr()).  There is no CPU fallback: if librsrs.so is missing the
import fails loudly, and without a GPU every compute call raises RSRSError
(RSRS_ERR_CUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librsrs.so")
SAMPLER_PATH = os.path.join(_HERE, "libsampler.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make -C paper_2311_01451_b200/csrc` "
                      "(or __graft_entry__.build()); there is no fallback implementation")
_lib = ctypes.CDLL(LIB_PATH)

RSRS_OK, RSRS_ERR_INVALID, RSRS_ERR_SAMPLES, RSRS_ERR_SINGULAR = 0, 1, 2, 3
RSRS_ERR_CUDA, RSRS_ERR_NCCL, RSRS_ERR_NOMEM, RSRS_ERR_STATE = 4, 5, 6, 7
RSRS_F64, RSRS_C128 = 0, 1
STATUS_NAMES = {0: "OK", 1: "INVALID", 2: "SAMPLES", 3: "SINGULAR", 4: "CUDA", 5: "NCCL", 6: "NOMEM", 7: "STATE"}

# Every symbol include/rsrs.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "rsrs_build_tree", "rsrs_tree_info", "rsrs_tree_perm", "rsrs_tree_level_size", "rsrs_tree_level",
    "rsrs_plan_samples", "rsrs_tree_destroy", "rsrs_factor", "rsrs_solve", "rsrs_apply",
    "rsrs_factor_stats", "rsrs_factor_ranks", "rsrs_factor_top", "rsrs_factor_destroy", "rsrs_factor_profile",
    "rsrs_last_error", "rsrs_version", "rsrs_memory_info", "rsrs_release_memory",
    "rsrs_tree_partition", "rsrs_dist_owner", "rsrs_dist_halo_plan", "rsrs_dist_move_plan",
    "rsrs_comm_unique_id", "rsrs_comm_init", "rsrs_comm_destroy", "rsrs_comm_selftest",
    "rsrs_factor_emulated", "rsrs_solve_emulated", "rsrs_apply_emulated", "rsrs_factor_coupling",
    "rsrs_factor_atol",
]


class RSRSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"RSRS_ERR_{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Opts(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("level_growth", ctypes.c_double), ("id_scale", ctypes.c_double),
                ("oversample", ctypes.c_int), ("top_level", ctypes.c_int), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int), ("nccl_comm", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("profile", ctypes.c_int), ("gather_level", ctypes.c_int), ("symmetric", ctypes.c_int),
                ("direct_gram", ctypes.c_int), ("push_updates", ctypes.c_int),
                ("estimate_coupling", ctypes.c_int), ("noise_factor", ctypes.c_double),
                ("triangular", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("p", ctypes.c_int64), ("L", ctypes.c_int), ("top_level", ctypes.c_int),
                ("nlevels_compressed", ctypes.c_int), ("nsteps", ctypes.c_int64), ("top_size", ctypes.c_int64),
                ("max_rank", ctypes.c_int64), ("memory_scalars", ctypes.c_int64), ("factor_ms", ctypes.c_double),
                ("flops_model", ctypes.c_double), ("bytes_model", ctypes.c_double), ("launches", ctypes.c_int64),
                ("solve_launches", ctypes.c_int64), ("flops_survey", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_vp, _i64, _i32, _d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
_lib.rsrs_last_error.restype = ctypes.c_char_p
_lib.rsrs_version.restype = ctypes.c_char_p
_lib.rsrs_build_tree.argtypes = [_vp, _i64, _i32, _i32, _vp, _d, _i32, ctypes.POINTER(_vp)]
_lib.rsrs_tree_info.argtypes = [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i64)]
_lib.rsrs_tree_perm.argtypes = [_vp, _vp]
_lib.rsrs_tree_level_size.argtypes = [_vp, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
_lib.rsrs_tree_level.argtypes = [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.rsrs_plan_samples.argtypes = [_vp, _i32, _i32, ctypes.POINTER(_i64)]
_lib.rsrs_tree_destroy.argtypes = [_vp]
_lib.rsrs_tree_destroy.restype = None
_lib.rsrs_factor.argtypes = [_vp, _i32, _i64, _vp, _vp, _vp, _vp, _i64, ctypes.POINTER(Opts), ctypes.POINTER(_vp)]
_lib.rsrs_solve.argtypes = [_vp, _vp, _i64, _i64, _vp]
_lib.rsrs_apply.argtypes = [_vp, _vp, _i64, _i64, _vp]
_lib.rsrs_factor_stats.argtypes = [_vp, ctypes.POINTER(Stats)]
_lib.rsrs_factor_ranks.argtypes = [_vp, _i32, _vp, _i64]
_lib.rsrs_factor_top.argtypes = [_vp, _vp, _i64, ctypes.POINTER(_i64)]
_lib.rsrs_factor_coupling.argtypes = [_vp, _i32, _vp, _i64]
_lib.rsrs_factor_coupling.restype = ctypes.c_int
_lib.rsrs_factor_atol.argtypes = [_vp, _i32, ctypes.POINTER(_d)]
_lib.rsrs_factor_atol.restype = ctypes.c_int
_lib.rsrs_factor_profile.argtypes = [_vp, _i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(_d),
                                     ctypes.POINTER(_d), ctypes.POINTER(_d), ctypes.POINTER(_i64)]
_lib.rsrs_factor_profile.restype = ctypes.c_int
NUM_KERNEL_CLASSES = 12
_lib.rsrs_tree_partition.argtypes = [_vp, _i32, _i32, _i32, _vp, ctypes.POINTER(_i32)]
_lib.rsrs_dist_owner.argtypes = [_vp, _i32, _i32, _i32, _i32, _vp]
_lib.rsrs_dist_halo_plan.argtypes = [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _vp, _i64,
                                     ctypes.POINTER(_i64)]
_lib.rsrs_dist_move_plan.argtypes = [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i64, ctypes.POINTER(_i64)]
_lib.rsrs_comm_unique_id.argtypes = [_vp]
_lib.rsrs_comm_init.argtypes = [_i32, _i32, _vp, ctypes.POINTER(_vp)]
_lib.rsrs_comm_destroy.argtypes = [_vp]
_lib.rsrs_comm_destroy.restype = None
_lib.rsrs_comm_selftest.argtypes = [_vp, _i32, _i32]
_lib.rsrs_comm_selftest.restype = ctypes.c_int
_lib.rsrs_factor_emulated.argtypes = [_vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _i64, ctypes.POINTER(Opts), _vp]
_lib.rsrs_solve_emulated.argtypes = [_vp, _i32, _vp, _i64, _i64]
_lib.rsrs_apply_emulated.argtypes = [_vp, _i32, _vp, _i64, _i64]
for _n in ("rsrs_tree_partition", "rsrs_dist_owner", "rsrs_dist_halo_plan", "rsrs_dist_move_plan",
           "rsrs_comm_unique_id", "rsrs_comm_init", "rsrs_factor_emulated", "rsrs_solve_emulated",
           "rsrs_apply_emulated"):
    getattr(_lib, _n).restype = ctypes.c_int
_lib.rsrs_factor_destroy.argtypes = [_vp]
_lib.rsrs_factor_destroy.restype = None
for _n in ("rsrs_build_tree", "rsrs_tree_info", "rsrs_tree_perm", "rsrs_tree_level_size", "rsrs_tree_level",
           "rsrs_plan_samples", "rsrs_factor", "rsrs_solve", "rsrs_apply", "rsrs_factor_stats",
           "rsrs_factor_ranks", "rsrs_factor_top"):
    getattr(_lib, _n).restype = ctypes.c_int


def _check(st: int):
    if st != RSRS_OK:
        raise RSRSError(st, _lib.rsrs_last_error().decode())


def version() -> str:
    return _lib.rsrs_version().decode()


_lib.rsrs_memory_info.argtypes = [ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
_lib.rsrs_memory_info.restype = ctypes.c_int
_lib.rsrs_release_memory.argtypes = []
_lib.rsrs_release_memory.restype = None


def memory_info() -> dict:
    """Bytes of device memory the library's arena holds (reserved) and uses."""
    r, u = _i64(), _i64()
    _check(_lib.rsrs_memory_info(ctypes.byref(r), ctypes.byref(u)))
    return {"reserved": r.value, "in_use": u.value}


def release_memory() -> None:
    """Return the arena's idle chunks to the driver (synchronises the device)."""
    _lib.rsrs_release_memory()


def _ptr(t) -> int:
    """Device pointer of a CUDA tensor (or host pointer of a numpy array)."""
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _check_tensor(name, t, rows, min_cols=None, dtype=None, allow_1d=False, aligned_rows=True):
    """Argument validation the C ABI cannot do (it only sees a pointer and a leading dimension):
    a CUDA tensor of the factor's dtype with `rows` rows, unit column stride, a 16-byte aligned base
    and (sample arrays: aligned_rows) 16-byte aligned rows (the kernels stage rows with 16-byte
    cp.async); right-hand sides only need the aligned base."""
    import torch
    if not isinstance(t, torch.Tensor) or not (t.is_cuda or t.is_pinned()):
        raise ValueError(f"{name} must be a CUDA tensor or a pinned host tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if t.dtype not in (torch.float64, torch.complex128):
        raise ValueError(f"{name}: unsupported dtype {t.dtype} (float64 or complex128)")
    if t.dim() == 1 and allow_1d:
        if t.stride(0) != 1:
            raise ValueError(f"{name}: a 1-D right-hand side must be contiguous")
    elif t.dim() != 2:
        raise ValueError(f"{name} must be 2-D (rows x columns)" + (" or 1-D" if allow_1d else ""))
    elif t.stride(1) != 1:
        raise ValueError(f"{name}: column stride must be 1 (row-major rows)")
    if t.shape[0] != rows:
        raise ValueError(f"{name} has {t.shape[0]} rows, expected {rows}")
    if min_cols is not None and (t.dim() != 2 or t.shape[1] < min_cols):
        raise ValueError(f"{name} needs at least {min_cols} columns")
    if t.data_ptr() % 16:
        raise ValueError(f"{name}: data pointer not 16-byte aligned")
    if aligned_rows and t.dim() == 2 and (t.stride(0) * t.element_size()) % 16:
        raise ValueError(f"{name}: row stride not a multiple of 16 bytes")


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


class Tree:
    """Handle of rsrs_build_tree (host integer work)."""

    def __init__(self, points: np.ndarray, leaf_max: int, root_lo=None, root_side: float = 0.0, nranks: int = 1):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        N, d = pts.shape
        lo = None if root_lo is None else np.ascontiguousarray(root_lo, dtype=np.float64)
        h = _vp()
        _check(_lib.rsrs_build_tree(pts.ctypes.data, N, d, int(leaf_max),
                                    None if lo is None else lo.ctypes.data, float(root_side), int(nranks),
                                    ctypes.byref(h)))
        self._h = h
        L, dd, NN = _i32(), _i32(), _i64()
        _check(_lib.rsrs_tree_info(h, ctypes.byref(L), ctypes.byref(dd), ctypes.byref(NN)))
        self.L, self.d, self.N = L.value, dd.value, NN.value

    @property
    def handle(self):
        return self._h

    def perm(self) -> np.ndarray:
        out = np.empty(self.N, dtype=np.int64)
        _check(_lib.rsrs_tree_perm(self._h, out.ctypes.data))
        return out

    def level(self, lev: int) -> dict:
        nb, nn = _i64(), _i64()
        _check(_lib.rsrs_tree_level_size(self._h, lev, ctypes.byref(nb), ctypes.byref(nn)))
        n = nb.value
        keys = np.empty(n, np.uint64)
        start = np.empty(n + 1, np.int64)
        parent = np.empty(n, np.int32)
        colour = np.empty(n, np.int32)
        off = np.empty(n + 1, np.int32)
        nbr = np.empty(max(nn.value, 1), np.int32)
        _check(_lib.rsrs_tree_level(self._h, lev, keys.ctypes.data, start.ctypes.data, parent.ctypes.data,
                                    colour.ctypes.data, off.ctypes.data, nbr.ctypes.data))
        return {"keys": keys, "start": start, "parent": parent, "colour": colour,
                "neighbours": [nbr[off[i]:off[i + 1]] for i in range(n)]}

    def partition(self, nranks: int, gather_level: int = -1, top_level: int = 2):
        """(first[nranks+1] tree positions of the ranks' leaf ranges, gather level used)."""
        first = np.empty(nranks + 1, np.int64)
        g = _i32()
        _check(_lib.rsrs_tree_partition(self._h, nranks, gather_level, top_level, first.ctypes.data, ctypes.byref(g)))
        return first, g.value

    def owner(self, level: int, nranks: int, gather_level: int = -1, top_level: int = 2) -> np.ndarray:
        nb, nn = _i64(), _i64()
        _check(_lib.rsrs_tree_level_size(self._h, level, ctypes.byref(nb), ctypes.byref(nn)))
        out = np.empty(max(nb.value, 1), np.int32)
        _check(_lib.rsrs_dist_owner(self._h, nranks, gather_level, top_level, level, out.ctypes.data))
        return out[:nb.value]

    def _plan(self, fn, args):
        n = _i64()
        _check(fn(*args, None, 0, ctypes.byref(n)))
        out = np.zeros((max(n.value, 1), 4), np.int32)
        _check(fn(*args, out.ctypes.data, out.shape[0], ctypes.byref(n)))
        return out[:n.value]

    def halo_plan(self, nranks, level, colour, nb, cnt, rank, gather_level=-1, top_level=2) -> np.ndarray:
        """Records {kind (0 send, 1 recv), peer, box, rows} of the (level, colour) halo exchange."""
        nb = np.ascontiguousarray(nb, np.int32)
        cnt = np.ascontiguousarray(cnt, np.int32)
        return self._plan(_lib.rsrs_dist_halo_plan, (self._h, nranks, gather_level, top_level, level, colour,
                                                     nb.ctypes.data, cnt.ctypes.data, rank))

    def move_plan(self, nranks, level, k, rank, gather_level=-1, top_level=2) -> np.ndarray:
        """Records {kind, peer, box, rows} of the skeleton-row moves level -> level-1."""
        k = np.ascontiguousarray(k, np.int32)
        return self._plan(_lib.rsrs_dist_move_plan, (self._h, nranks, gather_level, top_level, level,
                                                     k.ctypes.data, rank))

    def plan_samples(self, kmax_guess: int = 20, oversample: int = 10) -> int:
        p = _i64()
        _check(_lib.rsrs_plan_samples(self._h, kmax_guess, oversample, ctypes.byref(p)))
        return p.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.rsrs_tree_destroy(h)
            self._h = None


class Factorization:
    """Handle of rsrs_factor."""

    def __init__(self, handle, tree: Tree, dtype=None):
        self._h = handle
        self.tree_L = tree.L
        self.N = tree.N
        self.dtype = dtype

    def stats(self) -> dict:
        st = Stats()
        _check(_lib.rsrs_factor_stats(self._h, ctypes.byref(st)))
        return st.as_dict()

    def profile(self) -> list:
        """Per kernel class: name, device ms (opts.profile), algorithmic flops / bytes, launches."""
        out = []
        for c in range(NUM_KERNEL_CLASSES):
            nm, ms, fl, by, nl = ctypes.c_char_p(), _d(), _d(), _d(), _i64()
            _check(_lib.rsrs_factor_profile(self._h, c, ctypes.byref(nm), ctypes.byref(ms), ctypes.byref(fl),
                                            ctypes.byref(by), ctypes.byref(nl)))
            out.append({"name": nm.value.decode(), "ms": ms.value, "flops": fl.value, "bytes": by.value,
                        "launches": nl.value})
        return out

    def ranks(self, level: int, nboxes: int) -> np.ndarray:
        out = np.empty(max(nboxes, 1), np.int32)
        _check(_lib.rsrs_factor_ranks(self._h, level, out.ctypes.data, out.shape[0]))
        return out[:nboxes]

    def coupling(self, level: int, nboxes: int) -> np.ndarray:
        """(nboxes, 2) estimates of |A~(r_b, f)|_F, |A~(f, r_b)|_F (opts.estimate_coupling); -1: none."""
        out = np.empty(2 * max(nboxes, 1), np.float64)
        _check(_lib.rsrs_factor_coupling(self._h, level, out.ctypes.data, out.shape[0]))
        return out[:2 * nboxes].reshape(nboxes, 2)

    def atol(self, level: int) -> float:
        """ID tolerance the factorization used on `level` (0 if not compressed)."""
        v = _d()
        _check(_lib.rsrs_factor_atol(self._h, level, ctypes.byref(v)))
        return v.value

    def top(self) -> np.ndarray:
        n = _i64()
        _check(_lib.rsrs_factor_top(self._h, None, 0, ctypes.byref(n)))
        out = np.empty(max(n.value, 1), np.int64)
        _check(_lib.rsrs_factor_top(self._h, out.ctypes.data, out.shape[0], ctypes.byref(n)))
        return out[:n.value]

    def solve(self, B, stream=None):
        """B <- K^-1 B in place; B: CUDA tensor of the factor's dtype, (N,) or (N, nrhs) row-major,
        original order."""
        _check_tensor("B", B, self.N, dtype=self.dtype, allow_1d=True, aligned_rows=False)
        nrhs = 1 if B.dim() == 1 else B.shape[1]
        ldb = 1 if B.dim() == 1 else B.stride(0)
        _check(_lib.rsrs_solve(self._h, _ptr(B), ldb, nrhs, _stream_ptr(stream)))
        return B

    def apply(self, X, stream=None):
        """X <- K X in place (same layout as solve)."""
        _check_tensor("X", X, self.N, dtype=self.dtype, allow_1d=True, aligned_rows=False)
        nrhs = 1 if X.dim() == 1 else X.shape[1]
        ldx = 1 if X.dim() == 1 else X.stride(0)
        _check(_lib.rsrs_apply(self._h, _ptr(X), ldx, nrhs, _stream_ptr(stream)))
        return X

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.rsrs_factor_destroy(h)
            self._h = None


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return RSRS_F64
    if t.dtype == torch.complex128:
        return RSRS_C128
    raise ValueError(f"unsupported dtype {t.dtype} (float64 or complex128)")


def factor(tree: Tree, Y, Z, Omega, Psi, p: int, eps: float = 1e-6, level_growth: float = 1.0,
           id_scale: float = 1.0, oversample: int = 10, top_level: int = 2, stream=None,
           dtype: int | None = None, profile: bool = False, comm=None, rank: int = 0, nranks: int = 1,
           gather_level: int = -1, symmetric: bool = False, direct_gram: bool = False,
           push_updates: bool = False, estimate_coupling: bool = False,
           noise_factor: float = 0.0, triangular: bool = False) -> Factorization:
    """rsrs_factor on CUDA tensors (N x ld, tree order); Y, Z, Omega, Psi are OVERWRITTEN.
    Pinned host tensors are also accepted (end-to-end use): the library copies them into its own
    device store, overlapping the Y / Z rows with the leaf sweep, and leaves them unchanged.

    float64 tensors -> RSRS_F64, complex128 -> RSRS_C128 (ld in elements).
    Multi-GPU (nranks > 1): this rank's rows only (Tree.partition()) and the
    NcclComm of this rank in `comm`.
    noise_factor > 0: noise-aware tolerance schedule (f1); triangular=True: the triangular output form for
    real symmetric positive definite A (f4; needs symmetric=True).
    symmetric=True: the f2 shortcut -- float64: real symmetric A (Psi = Omega, Z = Y); complex128: complex
    symmetric A = A^T (Psi = conj(Omega), Z = conj(Y)); Z and Psi may be None."""
    rows = tree.N
    if nranks > 1:
        first, _ = tree.partition(nranks, gather_level, top_level)
        rows = int(first[rank + 1] - first[rank])
    if symmetric:
        Z, Psi = Y, Omega
    _check_tensor("Y", Y, rows, min_cols=p)
    ld = Y.stride(0)
    code = _dtype_code(Y)
    for nm, t in (("Z", Z), ("Omega", Omega), ("Psi", Psi)):
        _check_tensor(nm, t, rows, min_cols=p, dtype=Y.dtype)
        if t.stride(0) != ld:
            raise ValueError("Y, Z, Omega, Psi must share the leading dimension")
        if t.is_cuda != Y.is_cuda:
            raise ValueError("Y, Z, Omega, Psi must all be CUDA tensors or all pinned host tensors")
    if dtype is not None and dtype != code:
        raise ValueError("dtype does not match the tensors")
    dtype = code
    symmode = 0 if not symmetric else (2 if code == RSRS_C128 else 1)
    o = Opts(eps, level_growth, id_scale, oversample, top_level, int(rank), int(nranks),
             None if comm is None else comm.handle, _stream_ptr(stream), int(profile), int(gather_level),
             symmode, int(direct_gram), int(push_updates), int(estimate_coupling), float(noise_factor),
             int(triangular))
    h = _vp()
    _check(_lib.rsrs_factor(tree.handle, dtype, int(p), _ptr(Y), _ptr(Z), _ptr(Omega), _ptr(Psi), int(ld),
                            ctypes.byref(o), ctypes.byref(h)))
    return Factorization(h, tree, Y.dtype)


class NcclComm:
    """The library's NCCL communicator (rsrs_comm_init).  Rank 0 draws the unique
    id; `bcast(bytes) -> bytes` ships it to the other ranks (e.g. torch.distributed)."""

    def __init__(self, nranks: int, rank: int, bcast):
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(_lib.rsrs_comm_unique_id(uid))
        raw = bcast(uid.raw if rank == 0 else None)
        uid = ctypes.create_string_buffer(bytes(raw), 128)
        h = _vp()
        _check(_lib.rsrs_comm_init(nranks, rank, uid, ctypes.byref(h)))
        self._h, self.nranks, self.rank = h, nranks, rank

    @property
    def handle(self):
        return self._h

    def selftest(self):
        """All-reduces and a ring exchange through the library's NCCL transport."""
        _check(_lib.rsrs_comm_selftest(self._h, self.nranks, self.rank))

    def destroy(self):
        if self._h is not None and self._h.value:
            _lib.rsrs_comm_destroy(self._h)
            self._h = None


def factor_emulated(tree: Tree, G: int, Y, Z, Omega, Psi, p: int, eps: float = 1e-6, level_growth: float = 1.0,
                    id_scale: float = 1.0, oversample: int = 10, top_level: int = 2, gather_level: int = -1,
                    symmetric: bool = False, push_updates: bool = False) -> list:
    """G-rank run of the multi-GPU sweep emulated on this GPU (one host thread per rank);
    full tree-ordered Y, Z, Omega, Psi (overwritten).  Returns the G rank factorizations."""
    if symmetric:
        Z, Psi = Y, Omega
    for nm, t in (("Y", Y), ("Z", Z), ("Omega", Omega), ("Psi", Psi)):
        _check_tensor(nm, t, tree.N, min_cols=p, dtype=Y.dtype)
        if t.stride(0) != Y.stride(0):
            raise ValueError("Y, Z, Omega, Psi must share the leading dimension")
    ld = Y.stride(0)
    code = _dtype_code(Y)
    symmode = 0 if not symmetric else (2 if code == RSRS_C128 else 1)
    o = Opts(eps, level_growth, id_scale, oversample, top_level, 0, G, None, None, 0, int(gather_level),
             symmode, 0, int(push_updates), 0)
    hs = (_vp * G)()
    _check(_lib.rsrs_factor_emulated(tree.handle, code, int(p), int(G), _ptr(Y), _ptr(Z), _ptr(Omega), _ptr(Psi),
                                     int(ld), ctypes.byref(o), hs))
    return [Factorization(_vp(hs[q]), tree, Y.dtype) for q in range(G)]


def _emul_sweep(fn, fs, B):
    G = len(fs)
    _check_tensor("B", B, fs[0].N, dtype=fs[0].dtype, allow_1d=True, aligned_rows=False)
    hs = (_vp * G)(*[f._h.value for f in fs])
    nrhs = 1 if B.dim() == 1 else B.shape[1]
    ld = 1 if B.dim() == 1 else B.stride(0)
    _check(fn(hs, G, _ptr(B), ld, nrhs))
    return B


def solve_emulated(fs: list, B):
    """B <- K^-1 B through the G emulated ranks' distributed solve (full B, original order)."""
    return _emul_sweep(_lib.rsrs_solve_emulated, fs, B)


def apply_emulated(fs: list, X):
    return _emul_sweep(_lib.rsrs_apply_emulated, fs, X)


# ----------------------------------------------------------------------------
# harness operator (libsampler.so, include/rsrs_sampler.h) -- not the factor path
# ----------------------------------------------------------------------------
_sampler = None
KERNEL_KIND = {"log2d": 0, "lap3d": 1, "helm2d": 2}


def _sampler_lib():
    global _sampler
    if _sampler is None:
        if not os.path.exists(SAMPLER_PATH):
            raise ImportError(f"{SAMPLER_PATH} is missing (make -C paper_2311_01451_b200/csrc)")
        s = ctypes.CDLL(SAMPLER_PATH)
        s.rsrs_sample_matvec.argtypes = [_i32, _vp, _i64, _d, _vp, _i64, _vp, _i64, _i64, _i32, _vp]
        s.rsrs_sample_matvec.restype = ctypes.c_int
        s.rsrs_sampler_last_error.restype = ctypes.c_char_p
        s.rsrs_sample_matvec_c128.argtypes = [_vp, _i64, _d, _d, _vp, _i64, _vp, _i64, _i64, _i32, _vp]
        s.rsrs_sample_matvec_c128.restype = ctypes.c_int
        s.rsrs_sample_matvec_rows.argtypes = [_i32, _vp, _i64, _i64, _i64, _d, _d, _vp, _i64, _vp, _i64, _i64, _i32,
                                              _vp]
        s.rsrs_sample_matvec_rows.restype = ctypes.c_int
        _sampler = s
    return _sampler


_T11_CACHE = {}


def _t11_apply(pts3, X, Y, slab_b: int = 10):
    """Y = T11 X for the SURVEY 8(f) f3 workload: the sparse Schur complement
    T11 = A11 - A12 A22^-1 A21 of a 3D Poisson slab decomposition, applied exactly in its
    eigenbasis, T11 = S2 diag(mu) S2 with S2 = S (x) S the orthonormal DST-I of the n x n
    interface plane (mu: workloads.t11_symbol, a closed form of the slab's tridiagonal solves).
    Harness operator (the black box RSRS samples), on cuBLAS matmuls through torch -- not the
    factorization path.  Rows of X / Y follow pts3 (any order: a point's plane index is recovered
    from its cell-centre coordinates)."""
    import torch

    import workloads as W
    N = pts3.shape[0]
    n = int(round(N ** 0.5))
    key = (n, slab_b, str(X.device))
    if key not in _T11_CACHE:
        S = torch.from_numpy(W.dst_matrix(n)).to(X.device)
        mu = torch.from_numpy(W.t11_symbol(n, slab_b)).to(X.device)
        _T11_CACHE[key] = (S, mu)
    S, mu = _T11_CACHE[key]
    orig = (torch.floor(pts3[:, 1] * n).long() * n + torch.floor(pts3[:, 0] * n).long()).clamp_(0, N - 1)
    k = 1 if X.dim() == 1 else X.shape[1]
    Xo = torch.empty((N, k), dtype=X.dtype, device=X.device)
    Xo[orig] = X.reshape(N, k)
    V = Xo.view(n, n, k)
    V = torch.einsum("ik,klc->ilc", S, V)
    V = torch.einsum("jl,ilc->ijc", S, V) * mu[:, :, None]
    V = torch.einsum("ik,klc->ilc", S, V)
    V = torch.einsum("jl,ilc->ijc", S, V)
    Y.reshape(N, k).copy_(V.reshape(N, k)[orig])
    return Y


def sample_matvec(kind: str, pts3, weight: float, X, Y, adjoint: bool = False, stream=None, kappa: float = 25.0,
                  slab_b: int = 10):
    """Y = A X with the on-the-fly kernel operator (device tensors; pts3 N x 3).

    helm2d is complex (X, Y complex128); the others are real (float64); t11 is the f3 Schur
    complement (symmetric, so adjoint is the same operator)."""
    if kind == "t11":
        return _t11_apply(pts3, X, Y, slab_b)
    s = _sampler_lib()
    N = pts3.shape[0]
    ncol = 1 if X.dim() == 1 else X.shape[1]
    ldx = 1 if X.dim() == 1 else X.stride(0)
    ldy = 1 if Y.dim() == 1 else Y.stride(0)
    if kind == "helm2d":
        st = s.rsrs_sample_matvec_c128(_ptr(pts3), N, float(weight), float(kappa), _ptr(X), ldx, _ptr(Y), ldy,
                                       ncol, int(adjoint), _stream_ptr(stream))
    else:
        st = s.rsrs_sample_matvec(KERNEL_KIND[kind], _ptr(pts3), N, float(weight), _ptr(X), ldx, _ptr(Y), ldy,
                                  ncol, int(adjoint), _stream_ptr(stream))
    if st != 0:
        raise RSRSError(st, s.rsrs_sampler_last_error().decode())
    return Y


def sample_matvec_rows(kind: str, pts3, weight: float, X, Y, row0: int, adjoint: bool = False, stream=None,
                       kappa: float = 25.0):
    """Rows [row0, row0 + Y.shape[0]) of A X (multi-GPU sampling of a rank's own rows)."""
    if kind == "t11":
        import torch
        full = torch.empty((pts3.shape[0],) + tuple(Y.shape[1:]), dtype=Y.dtype, device=Y.device)
        _t11_apply(pts3, X, full)
        Y.copy_(full[row0:row0 + Y.shape[0]])
        return Y
    s = _sampler_lib()
    N = pts3.shape[0]
    nrows = Y.shape[0]
    ncol = 1 if X.dim() == 1 else X.shape[1]
    ldx = 1 if X.dim() == 1 else X.stride(0)
    ldy = 1 if Y.dim() == 1 else Y.stride(0)
    st = s.rsrs_sample_matvec_rows(KERNEL_KIND[kind], _ptr(pts3), N, int(row0), int(nrows), float(weight),
                                   float(kappa), _ptr(X), ldx, _ptr(Y), ldy, ncol, int(adjoint), _stream_ptr(stream))
    if st != 0:
        raise RSRSError(st, s.rsrs_sampler_last_error().decode())
    return Y
