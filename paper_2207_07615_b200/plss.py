"""Thin ctypes binding of libplss (include/plss.h): argument marshalling only.

Every step of the PLSS path runs in libplss's sm_100a kernels; torch provides device memory
(the matrix copies and the workspace), streams and, for the distributed path, the process group
that broadcasts the NCCL unique id. There is no CPU fallback: if libplss.so is missing or no CUDA
device is present, the calls raise.

Names mirror the C ABI: plss_workspace_bytes, plss_create, plss_create_dist, plss_get_unique_id,
plss_solve, plss_start, plss_step, plss_finish, plss_spmv, plss_spmvT, plss_query, plss_destroy.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libplss.so")
REC = 8
OUTCOMES = {0: "converged", 1: "maxit", 2: "y_vanished", 3: "stagnation", -1: "running"}

# C ABI symbols declared in include/plss.h (checked by tests/test_abi.py)
SYMBOLS = ["plss_workspace_bytes", "plss_create", "plss_get_unique_id", "plss_create_dist",
           "plss_solve", "plss_start", "plss_step", "plss_finish", "plss_spmv", "plss_spmvT",
           "plss_profile", "plss_query", "plss_destroy", "plss_status_str", "plss_last_error",
           "plss_set_wi", "plss_column_norms", "plss_rp_workspace_bytes", "plss_rp_solve", "plss_rp_start",
           "plss_rp_step", "plss_rp_finish", "plss_rp_sketch", "plss_spmmT", "plss_rp_profile",
           "plss_kz_workspace_bytes", "plss_kz_solve", "plss_kz_start", "plss_kz_step", "plss_kz_finish",
           "plss_kz_profile", "plss_eg_workspace_bytes", "plss_eg_solve", "plss_eg_start", "plss_eg_step",
           "plss_eg_finish", "plss_eg_profile", "plss_true_residual", "plss_peer_reduce_emulate",
           "plss_create_dist_cols", "plss_debug_cta_times", "plss_query_segment"]


class PlssError(RuntimeError):
    pass


class plss_matrix(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p),
                ("col_ptr", ctypes.c_void_p), ("row_idx", ctypes.c_void_p), ("val_t", ctypes.c_void_p),
                ("validate", ctypes.c_int32)]


class plss_options(ctypes.Structure):
    _fields_ = [("slabs", ctypes.c_int32), ("graph_chunk", ctypes.c_int32),
                ("maxit_cap", ctypes.c_int32), ("flags", ctypes.c_int32)]


_lib = None


def load_library(path: str = None):
    """Load libplss.so (raises if it was not built). torch is imported first so that the NCCL
    it bundles is the one libplss resolves. PLSS_LIB selects a tuning-variant build."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PLSS_LIB") or LIB_PATH
    import torch  # noqa: F401  (loads torch's libnccl.so.2 / CUDA runtime)
    if not os.path.exists(path):
        raise PlssError(f"{path} is missing: run `python -m paper_2207_07615_b200.build` "
                        "(no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    st = ctypes.c_int
    lib.plss_workspace_bytes.argtypes = [ctypes.POINTER(plss_matrix), ctypes.POINTER(plss_options)]
    lib.plss_workspace_bytes.restype = ctypes.c_size_t
    lib.plss_create.argtypes = [ctypes.POINTER(plss_matrix), ctypes.POINTER(plss_options), P,
                                ctypes.c_size_t, P, ctypes.POINTER(P)]
    lib.plss_create.restype = st
    lib.plss_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.plss_get_unique_id.restype = st
    lib.plss_create_dist.argtypes = [ctypes.POINTER(plss_matrix), I64, I64, ctypes.c_char_p, I32, I32,
                                     ctypes.POINTER(plss_options), P, ctypes.c_size_t, P,
                                     ctypes.POINTER(P)]
    lib.plss_create_dist.restype = st
    lib.plss_solve.argtypes = [P, P, P, D, I32, I32, I32, P, ctypes.POINTER(I32), P, P,
                               ctypes.POINTER(ctypes.c_int)]
    lib.plss_solve.restype = st
    lib.plss_start.argtypes = [P, P, P, D, I32, I32, I32]
    lib.plss_start.restype = st
    lib.plss_step.argtypes = [P, I32]
    lib.plss_step.restype = st
    lib.plss_finish.argtypes = [P, P, ctypes.POINTER(I32), P, P, ctypes.POINTER(ctypes.c_int)]
    lib.plss_finish.restype = st
    lib.plss_spmv.argtypes = [P, P, P]
    lib.plss_spmv.restype = st
    lib.plss_spmvT.argtypes = [P, P, P]
    lib.plss_spmvT.restype = st
    lib.plss_profile.argtypes = [P, I32, P]
    lib.plss_profile.restype = st
    lib.plss_query.argtypes = [P] + [ctypes.POINTER(I32)] * 7
    lib.plss_query.restype = st
    lib.plss_set_wi.argtypes = [P, P]
    lib.plss_set_wi.restype = st
    lib.plss_column_norms.argtypes = [P, P]
    lib.plss_column_norms.restype = st
    U64 = ctypes.c_uint64
    lib.plss_rp_workspace_bytes.argtypes = [P, I32]
    lib.plss_rp_workspace_bytes.restype = ctypes.c_size_t
    lib.plss_rp_start.argtypes = [P, I32, U64, D, P, ctypes.c_size_t, P, P, D, I32, I32]
    lib.plss_rp_start.restype = st
    lib.plss_rp_step.argtypes = [P, I32]
    lib.plss_rp_step.restype = st
    lib.plss_rp_finish.argtypes = [P, P, ctypes.POINTER(I32), P, P, ctypes.POINTER(ctypes.c_int)]
    lib.plss_rp_finish.restype = st
    lib.plss_rp_solve.argtypes = [P, I32, U64, D, P, ctypes.c_size_t, P, P, D, I32, I32, P, ctypes.POINTER(I32),
                                  P, P, ctypes.POINTER(ctypes.c_int)]
    lib.plss_rp_solve.restype = st
    lib.plss_rp_sketch.argtypes = [P, I32, U64, D, I32, I32, P]
    lib.plss_rp_sketch.restype = st
    lib.plss_rp_profile.argtypes = [P, I32, P]
    lib.plss_rp_profile.restype = st
    lib.plss_spmmT.argtypes = [P, I32, I32, P, P]
    lib.plss_spmmT.restype = st
    lib.plss_kz_workspace_bytes.argtypes = [P, I32]
    lib.plss_kz_workspace_bytes.restype = ctypes.c_size_t
    lib.plss_kz_start.argtypes = [P, I32, P, ctypes.c_size_t, P, P, P, D, I32, I32]
    lib.plss_kz_start.restype = st
    lib.plss_kz_step.argtypes = [P, I32]
    lib.plss_kz_step.restype = st
    lib.plss_kz_finish.argtypes = [P, P, ctypes.POINTER(I32), P, P, ctypes.POINTER(ctypes.c_int)]
    lib.plss_kz_finish.restype = st
    lib.plss_kz_solve.argtypes = [P, I32, P, ctypes.c_size_t, P, P, P, D, I32, I32, P, ctypes.POINTER(I32), P, P,
                                  ctypes.POINTER(ctypes.c_int)]
    lib.plss_kz_solve.restype = st
    lib.plss_kz_profile.argtypes = [P, I32, P]
    lib.plss_kz_profile.restype = st
    lib.plss_eg_workspace_bytes.argtypes = [P, I32]
    lib.plss_eg_workspace_bytes.restype = ctypes.c_size_t
    lib.plss_eg_start.argtypes = [P, I32, I32, I32, P, ctypes.c_size_t, P, U64, P, P, D, I32, I32]
    lib.plss_eg_start.restype = st
    lib.plss_eg_step.argtypes = [P, I32]
    lib.plss_eg_step.restype = st
    lib.plss_eg_finish.argtypes = [P, P, ctypes.POINTER(I32), P, P, ctypes.POINTER(ctypes.c_int)]
    lib.plss_eg_finish.restype = st
    lib.plss_eg_solve.argtypes = [P, I32, I32, I32, P, ctypes.c_size_t, P, U64, P, P, D, I32, I32, P,
                                  ctypes.POINTER(I32), P, P, ctypes.POINTER(ctypes.c_int)]
    lib.plss_eg_solve.restype = st
    lib.plss_eg_profile.argtypes = [P, I32, P]
    lib.plss_eg_profile.restype = st
    lib.plss_true_residual.argtypes = [P, P, P, P]
    lib.plss_true_residual.restype = st
    lib.plss_create_dist_cols.argtypes = lib.plss_create_dist.argtypes
    lib.plss_create_dist_cols.restype = st
    lib.plss_peer_reduce_emulate.argtypes = [I32, P, P, P, I32, P, P]
    lib.plss_peer_reduce_emulate.restype = st
    lib.plss_query_segment.argtypes = [P, I32, I32, P]
    lib.plss_query_segment.restype = st
    lib.plss_debug_cta_times.argtypes = [P, I32, I32, P, ctypes.POINTER(I32)]
    lib.plss_debug_cta_times.restype = st
    lib.plss_query_segment.argtypes = [P, I32, I32, P]
    lib.plss_query_segment.restype = st
    lib.plss_debug_cta_times.argtypes = [P, I32, I32, P, ctypes.POINTER(I32)]
    lib.plss_debug_cta_times.restype = st
    lib.plss_destroy.argtypes = [P]
    lib.plss_destroy.restype = None
    lib.plss_status_str.argtypes = [st]
    lib.plss_status_str.restype = ctypes.c_char_p
    lib.plss_last_error.argtypes = [P]
    lib.plss_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(status: int, ctx_ptr=None):
    if status != 0:
        lib = load_library()
        msg = lib.plss_last_error(ctx_ptr)
        raise PlssError(f"{lib.plss_status_str(status).decode()}: {(msg or b'').decode()}")


def _ptr(a) -> Optional[int]:
    """Device or host address of a torch tensor / numpy array (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _vec(ctx, a, n: int, name: str, host_ok: bool = True) -> Optional[int]:
    """Checked address of a float64 vector argument of length >= n (None passes through): a numpy
    array or CPU tensor (host; where the entry point accepts host memory) or a CUDA tensor on the
    ctx's device, C-contiguous and 8-byte aligned (the SpMVs take an x at any 8-byte phase; vectors
    the solve keeps are copied into the workspace).
    Raises PlssError before anything reaches the library (the C side cannot check a
    foreign pointer's dtype, length or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not host_ok:
            raise PlssError(f"{name}: a CUDA tensor is required")
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise PlssError(f"{name}: float64 C-contiguous array required (got {a.dtype})")
        if a.size < n:
            raise PlssError(f"{name}: {a.size} elements, {n} required")
        return a.ctypes.data
    import torch
    if not isinstance(a, torch.Tensor):
        raise PlssError(f"{name}: numpy array or torch tensor required (got {type(a).__name__})")
    if a.dtype != torch.float64 or not a.is_contiguous():
        raise PlssError(f"{name}: contiguous float64 tensor required (got {a.dtype})")
    if a.numel() < n:
        raise PlssError(f"{name}: {a.numel()} elements, {n} required")
    if a.is_cuda:
        dev = ctx.A.row_ptr.device
        if a.device != dev:
            raise PlssError(f"{name}: on {a.device}, the ctx is on {dev}")
        if a.data_ptr() % 8:
            raise PlssError(f"{name}: device vectors must be 8-byte aligned")
    elif not host_ok:
        raise PlssError(f"{name}: a CUDA tensor is required")
    return a.data_ptr()


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


@dataclass
class Matrix:
    """Device CSR + CSC copies of A (torch tensors, int32 / float64), borrowed by a ctx."""
    m: int
    n: int
    row_ptr: "object"
    col_idx: "object"
    val: "object"
    col_ptr: "object"
    row_idx: "object"
    val_t: "object"

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @classmethod
    def from_arrays(cls, m, n, row_ptr, col_idx, val, col_ptr, row_idx, val_t, device="cuda"):
        import torch

        def t(a, dt):
            if isinstance(a, torch.Tensor):
                return a.to(device=device, dtype=dt).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)
        return cls(int(m), int(n), t(row_ptr, torch.int32), t(col_idx, torch.int32),
                   t(val, torch.float64), t(col_ptr, torch.int32), t(row_idx, torch.int32),
                   t(val_t, torch.float64))

    def c_struct(self, validate=False) -> plss_matrix:
        return plss_matrix(self.m, self.n, self.nnz, _ptr(self.row_ptr), _ptr(self.col_idx),
                           _ptr(self.val), _ptr(self.col_ptr), _ptr(self.row_idx), _ptr(self.val_t),
                           1 if validate else 0)


def _opts(slabs=0, graph_chunk=0, maxit_cap=0, sell=True, window=True, rsag=False, peer=False):
    return plss_options(int(slabs), int(graph_chunk), int(maxit_cap),
                        (0 if sell else 1) | (0 if window else 2) | (4 if rsag else 0) | (8 if peer else 0))


def plss_workspace_bytes(A: Matrix, slabs=0, graph_chunk=0, maxit_cap=0, sell=True, window=True) -> int:
    lib = load_library()
    ms = A.c_struct()
    o = _opts(slabs, graph_chunk, maxit_cap, sell, window)
    nbytes = lib.plss_workspace_bytes(ctypes.byref(ms), ctypes.byref(o))
    if nbytes == 0:
        raise PlssError("invalid matrix sizes")
    return int(nbytes)


class Ctx:
    """Owns the ctx handle, the torch workspace and references to the borrowed matrix."""

    def __init__(self, handle, A: Matrix, workspace, stream, maxit_cap):
        self.handle = handle
        self.A = A
        self.workspace = workspace
        self.stream = stream
        self.maxit_cap = maxit_cap
        self._maxit = 0

    @property
    def m(self):
        return self.A.m

    @property
    def n(self):
        return self.A.n

    def __del__(self):
        try:
            plss_destroy(self)
        except Exception:
            pass


def _alloc_workspace(nbytes: int, device):
    import torch
    return torch.empty(nbytes + 256, dtype=torch.uint8, device=device)


def _aligned(ws) -> int:
    p = ws.data_ptr()
    return (p + 255) // 256 * 256


def plss_create(A: Matrix, slabs=0, graph_chunk=0, maxit_cap=20000, stream=None, validate=False,
                sell=True, window=True) -> Ctx:
    lib = load_library()
    nbytes = plss_workspace_bytes(A, slabs, graph_chunk, maxit_cap, sell, window)
    ws = _alloc_workspace(nbytes, A.row_ptr.device)
    h = ctypes.c_void_p()
    ms = A.c_struct(validate)
    o = _opts(slabs, graph_chunk, maxit_cap, sell, window)
    _check(lib.plss_create(ctypes.byref(ms), ctypes.byref(o), _aligned(ws), nbytes, _stream_ptr(stream),
                           ctypes.byref(h)))
    return Ctx(h, A, ws, stream, maxit_cap)


def plss_get_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.plss_get_unique_id(buf))
    return buf.raw


def plss_create_dist(A_local: Matrix, row_offset: int, m_global: int, uid: bytes, rank: int, nranks: int,
                     slabs=0, graph_chunk=0, maxit_cap=20000, stream=None, validate=False, sell=True,
                     window=True, rsag=False, peer=False) -> Ctx:
    """rsag: the reduce-scatter / all-gather step (include/plss.h, options.flags bit2); peer: the
    peer-memory all-reduce step (options.flags bit3)."""
    lib = load_library()
    nbytes = plss_workspace_bytes(A_local, slabs, graph_chunk, maxit_cap, sell, window)
    ws = _alloc_workspace(nbytes, A_local.row_ptr.device)
    h = ctypes.c_void_p()
    ms = A_local.c_struct(validate)
    o = _opts(slabs, graph_chunk, maxit_cap, sell, window, rsag, peer)
    _check(lib.plss_create_dist(ctypes.byref(ms), int(row_offset), int(m_global), uid, int(rank), int(nranks),
                                ctypes.byref(o), _aligned(ws), nbytes, _stream_ptr(stream), ctypes.byref(h)))
    return Ctx(h, A_local, ws, stream, maxit_cap)


def plss_create_dist_cols(A_local: Matrix, col_offset: int, n_global: int, uid: bytes, rank: int, nranks: int,
                          slabs=0, graph_chunk=0, maxit_cap=20000, stream=None, validate=False, sell=True,
                          window=True) -> Ctx:
    """Column-block distributed ctx (include/plss.h): A_local = the m x n_local block of columns
    [col_offset, col_offset + n_local), local column indices in its CSR; x / x0 are shards."""
    lib = load_library()
    nbytes = plss_workspace_bytes(A_local, slabs, graph_chunk, maxit_cap, sell, window)
    ws = _alloc_workspace(nbytes, A_local.row_ptr.device)
    h = ctypes.c_void_p()
    ms = A_local.c_struct(validate)
    o = _opts(slabs, graph_chunk, maxit_cap, sell, window)
    _check(lib.plss_create_dist_cols(ctypes.byref(ms), int(col_offset), int(n_global), uid, int(rank), int(nranks),
                                     ctypes.byref(o), _aligned(ws), nbytes, _stream_ptr(stream), ctypes.byref(h)))
    return Ctx(h, A_local, ws, stream, maxit_cap)


def plss_start(ctx: Ctx, b, x0=None, tol=1e-8, tol_mode=0, maxit=100, flags=0):
    lib = load_library()
    ctx._keep = (b, x0)
    ctx._maxit = int(maxit)
    _check(lib.plss_start(ctx.handle, _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode), int(maxit), int(flags)),
           ctx.handle)


def plss_step(ctx: Ctx, k: int):
    _check(load_library().plss_step(ctx.handle, int(k)), ctx.handle)


def plss_finish(ctx: Ctx, x=None, want_hist=True, want_diag=False):
    """Returns dict(iters, outcome, hist, diag); x (host or device buffer) receives the iterate."""
    lib = load_library()
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(ctx._maxit + 1) if want_hist else None
    diag = np.zeros((ctx._maxit + 1, REC)) if want_diag else None
    _check(lib.plss_finish(ctx.handle, _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it), _ptr(hist), _ptr(diag), ctypes.byref(oc)),
           ctx.handle)
    return _result(it.value, oc.value, hist, diag, x)


def _result(iters, oc, hist, diag, x):
    out = {"iters": iters, "outcome": OUTCOMES.get(oc, str(oc)), "outcome_code": oc, "x": x}
    if hist is not None:
        nh = iters if oc == 1 else iters + 1
        out["hist_full"] = hist
        out["hist"] = hist[:max(1, min(nh, hist.shape[0]))].copy()
    if diag is not None:
        out["diag"] = diag
    return out


def plss_solve(ctx: Ctx, b, x0=None, tol=1e-8, tol_mode=0, maxit=100, flags=0, x=None,
               want_hist=True, want_diag=False):
    """Full solve. b / x0 / x may be device tensors or host arrays (numpy / CPU tensors).
    If x is None a device tensor is allocated. Returns dict(x, iters, outcome, hist[, diag])."""
    import torch
    lib = load_library()
    if x is None:
        x = torch.empty(ctx.n, dtype=torch.float64, device=ctx.A.row_ptr.device)
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(maxit + 1) if want_hist else None
    diag = np.zeros((maxit + 1, REC)) if want_diag else None
    ctx._maxit = int(maxit)
    _check(lib.plss_solve(ctx.handle, _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode),
                          int(maxit), int(flags), _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it), _ptr(hist), _ptr(diag), ctypes.byref(oc)), ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if flags & 1:
        res["hist"] = hist[:it.value].copy()
    return res


def plss_set_wi(ctx: Ctx, wi=None):
    """PLSS W: WI = diag(wi) for later solves (None: WI = I)."""
    ctx._wi = wi
    _check(load_library().plss_set_wi(ctx.handle, _vec(ctx, wi, ctx.n, 'wi')), ctx.handle)


def plss_column_norms(ctx: Ctx, out=None):
    """c_j = ||A_{:,j}|| (zero columns 1) as a device tensor (or into `out`)."""
    import torch
    if out is None:
        out = torch.empty(ctx.n, dtype=torch.float64, device=ctx.A.row_ptr.device)
    _check(load_library().plss_column_norms(ctx.handle, _vec(ctx, out, ctx.n, 'out')), ctx.handle)
    return out


def plss_true_residual(ctx: Ctx, b, x) -> dict:
    """||b - A x|| and ||b|| (and their ratio) for an iterate x (host or device)."""
    out = np.zeros(2)
    _check(load_library().plss_true_residual(ctx.handle, _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x, ctx.n, 'x'), _ptr(out)), ctx.handle)
    return {"abs": float(out[0]), "norm_b": float(out[1]),
            "rel": float(out[0] / out[1]) if out[1] > 0 else float(out[0])}


def plss_peer_reduce_emulate(parts, reds, flags, bounds, stream=None):
    """One step of the peer-memory all-reduce over len(parts) virtual ranks on one device
    (include/plss.h): parts / reds float64 device tensors, flags int32 device tensors of 256 words
    (zeroed before the first step, then kept), bounds the nch + 1 chunk offsets."""
    G = len(parts)
    if not (len(reds) == len(flags) == G):
        raise PlssError("parts, reds and flags need one buffer per virtual rank")
    arr = lambda ts: (ctypes.c_void_p * G)(*[t.data_ptr() for t in ts])  # noqa: E731
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    _check(load_library().plss_peer_reduce_emulate(int(G), arr(parts), arr(reds), arr(flags), int(len(b) - 1),
                                                   b.ctypes.data, _stream_ptr(stream)))
    return reds


def plss_query_segment(ctx: Ctx, which: int, slab: int = 0) -> dict:
    """The format chosen for K1 (which = 1) / K2 (which = 2) of a row slab (include/plss.h)."""
    info = np.zeros(14, dtype=np.int32)
    _check(load_library().plss_query_segment(ctx.handle, int(which), int(slab), info.ctypes.data), ctx.handle)
    keys = ("fmt", "sig", "gsort", "nslices", "nlong", "stat", "grid", "rows", "nchunks", "psi3", "xdefer",
            "s1beg", "s1end", "lin")
    return {k: int(v) for k, v in zip(keys, info)}


def plss_debug_cta_times(ctx: Ctx, which: int, slab: int = 0):
    """Diagnostics (PLSS_DBG_CTA=1 at create): per-CTA {start ns, end ns, entries, units} of the
    last K1 (which = 1) / K2 (which = 2) launch of a slab, as an int64 array [grid, 4]."""
    out = np.zeros(4 * 2048, dtype=np.uint64)
    g = ctypes.c_int32(0)
    _check(load_library().plss_debug_cta_times(ctx.handle, int(which), int(slab), out.ctypes.data, ctypes.byref(g)),
           ctx.handle)
    return out[:4 * g.value].reshape(g.value, 4).astype(np.int64)


def plss_spmv(ctx: Ctx, x, y):
    _check(load_library().plss_spmv(ctx.handle, _vec(ctx, x, ctx.n, 'x', host_ok=False),
                                    _vec(ctx, y, ctx.m, 'y', host_ok=False)), ctx.handle)
    return y


def plss_spmvT(ctx: Ctx, u, v):
    _check(load_library().plss_spmvT(ctx.handle, _vec(ctx, u, ctx.m, 'u', host_ok=False),
                                     _vec(ctx, v, ctx.n, 'v', host_ok=False)), ctx.handle)
    return v


def plss_profile(ctx: Ctx, k: int) -> dict:
    """Average device ms per loop step of each kernel class (CUDA events, non-graph launches)."""
    ms = np.zeros(5)
    _check(load_library().plss_profile(ctx.handle, int(k), _ptr(ms)), ctx.handle)
    return dict(zip(["k1", "k2", "allreduce", "dots", "k3"], ms.tolist()))


def plss_query(ctx: Ctx) -> dict:
    vals = [ctypes.c_int32(0) for _ in range(7)]
    _check(load_library().plss_query(ctx.handle, *[ctypes.byref(v) for v in vals]), ctx.handle)
    keys = ["launches_per_step", "slabs", "tile_nnz", "grid_k1", "grid_k2", "sell_segments", "window_segments"]
    return {k: v.value for k, v in zip(keys, vals)}


def _rp_workspace(ctx: Ctx, r: int):
    """Device workspace of randomized projection with sketch size r, cached on the ctx."""
    nbytes = int(load_library().plss_rp_workspace_bytes(ctx.handle, int(r)))
    if nbytes == 0:
        raise PlssError("plss_rp_workspace_bytes: invalid r (1..64) or distributed ctx")
    ws = getattr(ctx, "_rp_ws", None)
    if ws is None or ws.numel() < nbytes + 256:
        ctx._rp_ws = None
        ws = ctx._rp_ws = _alloc_workspace(nbytes, ctx.A.row_ptr.device)
    return _aligned(ws), nbytes


def plss_rp_start(ctx: Ctx, b, r=10, seed=0, density=1.0, x0=None, tol=1e-8, tol_mode=0, maxit=100):
    """Randomized projection (eq:pkLong, fresh Gaussian S_k): start (see include/plss.h)."""
    lib = load_library()
    wp, nb = _rp_workspace(ctx, r)
    ctx._keep = (b, x0)
    ctx._maxit = int(maxit)
    _check(lib.plss_rp_start(ctx.handle, int(r), int(seed) & 0xFFFFFFFFFFFFFFFF, float(density), wp, nb, _vec(ctx, b, ctx.m, 'b'),
                             _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode), int(maxit)), ctx.handle)


def plss_rp_step(ctx: Ctx, k: int):
    _check(load_library().plss_rp_step(ctx.handle, int(k)), ctx.handle)


def plss_rp_finish(ctx: Ctx, x=None, want_hist=True, want_diag=False):
    lib = load_library()
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(ctx._maxit + 1) if want_hist else None
    diag = np.zeros((ctx._maxit + 1, REC)) if want_diag else None
    _check(lib.plss_rp_finish(ctx.handle, _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it), _ptr(hist), _ptr(diag), ctypes.byref(oc)),
           ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if hist is not None:
        res["hist"] = hist[:it.value + 1].copy()
    return res


def plss_rp_solve(ctx: Ctx, b, r=10, seed=0, density=1.0, x0=None, tol=1e-8, tol_mode=0, maxit=100, x=None,
                  want_hist=True, want_diag=False):
    """Full randomized-projection solve. Returns dict(x, iters, outcome, hist[0..iters][, diag])."""
    import torch
    lib = load_library()
    if x is None:
        x = torch.empty(ctx.n, dtype=torch.float64, device=ctx.A.row_ptr.device)
    wp, nb = _rp_workspace(ctx, r)
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(maxit + 1) if want_hist else None
    diag = np.zeros((maxit + 1, REC)) if want_diag else None
    ctx._maxit = int(maxit)
    _check(lib.plss_rp_solve(ctx.handle, int(r), int(seed) & 0xFFFFFFFFFFFFFFFF, float(density), wp, nb, _vec(ctx, b, ctx.m, 'b'),
                             _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode), int(maxit), _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it),
                             _ptr(hist), _ptr(diag), ctypes.byref(oc)), ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if hist is not None:
        res["hist"] = hist[:it.value + 1].copy()
    return res


def plss_rp_profile(ctx: Ctx, k: int) -> dict:
    """Average device ms per randomized-projection step of each kernel (CUDA events)."""
    ms = np.zeros(6)
    _check(load_library().plss_rp_profile(ctx.handle, int(k), _ptr(ms)), ctx.handle)
    return dict(zip(["gen", "spmm", "gram", "solve", "update", "k1"], ms.tolist()))


def rp_ld(r: int) -> int:
    """Row stride (floats) of S inside randomized-projection solves: whole 32-byte sectors."""
    return (int(r) + 7) // 8 * 8


def plss_rp_sketch(ctx: Ctx, r, seed, k, density=1.0, ld=None, out=None):
    """S_k (device float32, m x ld; columns >= r are 0) of the randomized-projection generator."""
    import torch
    ld = rp_ld(r) if ld is None else int(ld)
    if out is None:
        out = torch.empty((ctx.m, ld), dtype=torch.float32, device=ctx.A.row_ptr.device)
    _check(load_library().plss_rp_sketch(ctx.handle, int(r), int(seed) & 0xFFFFFFFFFFFFFFFF, float(density),
                                         int(k), ld, _ptr(out)), ctx.handle)
    return out


def plss_spmmT(ctx: Ctx, S, r=None, Y=None):
    """Y = A^T S[:, :r] (S: device float32 m x ld row-major) -> device float64 n x r."""
    import torch
    ld = int(S.shape[1])
    r = ld if r is None else int(r)
    if Y is None:
        Y = torch.empty((ctx.n, r), dtype=torch.float64, device=S.device)
    _check(load_library().plss_spmmT(ctx.handle, r, ld, _ptr(S), _ptr(Y)), ctx.handle)
    return Y


def _kz_workspace(ctx: Ctx, kmax: int):
    nbytes = int(load_library().plss_kz_workspace_bytes(ctx.handle, int(kmax)))
    if nbytes == 0:
        raise PlssError("plss_kz_workspace_bytes: invalid kmax or distributed ctx")
    ws = getattr(ctx, "_kz_ws", None)
    if ws is None or ws.numel() < nbytes + 256:
        ctx._kz_ws = None
        ws = ctx._kz_ws = _alloc_workspace(nbytes, ctx.A.row_ptr.device)
    return _aligned(ws), nbytes


def _rows_arg(rows):
    if isinstance(rows, np.ndarray) or not hasattr(rows, "data_ptr"):
        return np.ascontiguousarray(rows, dtype=np.int32)
    import torch
    return rows.to(dtype=torch.int32).contiguous()


def plss_kz_start(ctx: Ctx, b, rows, kmax=None, x0=None, tol=1e-8, tol_mode=0, maxit=100):
    """PLSS Kaczmarz (eq:pkKacz) over the row order `rows` (host or device int32, >= maxit)."""
    lib = load_library()
    kmax = int(maxit if kmax is None else kmax)
    wp, nb = _kz_workspace(ctx, kmax)
    rr = _rows_arg(rows)
    ctx._keep = (b, x0, rr)
    ctx._maxit = int(maxit)
    _check(lib.plss_kz_start(ctx.handle, kmax, wp, nb, _ptr(rr), _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode),
                             int(maxit)), ctx.handle)


def plss_kz_step(ctx: Ctx, k: int):
    _check(load_library().plss_kz_step(ctx.handle, int(k)), ctx.handle)


def plss_kz_finish(ctx: Ctx, x=None, want_hist=True, want_diag=False):
    lib = load_library()
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(ctx._maxit + 1) if want_hist else None
    diag = np.zeros((ctx._maxit + 1, REC)) if want_diag else None
    _check(lib.plss_kz_finish(ctx.handle, _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it), _ptr(hist), _ptr(diag), ctypes.byref(oc)),
           ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if hist is not None:
        res["hist"] = hist[:it.value + 1].copy()
    return res


def plss_kz_solve(ctx: Ctx, b, rows, kmax=None, x0=None, tol=1e-8, tol_mode=0, maxit=100, x=None,
                  want_hist=True, want_diag=False):
    """Full PLSS Kaczmarz solve. Returns dict(x, iters, outcome, hist[0..iters][, diag])."""
    import torch
    lib = load_library()
    if x is None:
        x = torch.empty(ctx.n, dtype=torch.float64, device=ctx.A.row_ptr.device)
    kmax = int(maxit if kmax is None else kmax)
    wp, nb = _kz_workspace(ctx, kmax)
    rr = _rows_arg(rows)
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(maxit + 1) if want_hist else None
    diag = np.zeros((maxit + 1, REC)) if want_diag else None
    ctx._maxit = int(maxit)
    _check(lib.plss_kz_solve(ctx.handle, kmax, wp, nb, _ptr(rr), _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode),
                             int(maxit), _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it), _ptr(hist), _ptr(diag), ctypes.byref(oc)),
           ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if hist is not None:
        res["hist"] = hist[:it.value + 1].copy()
    return res


def plss_kz_profile(ctx: Ctx, k: int) -> dict:
    ms = np.zeros(4)
    _check(load_library().plss_kz_profile(ctx.handle, int(k), _ptr(ms)), ctx.handle)
    return dict(zip(["prep", "gemv", "spmv", "resid"], ms.tolist()))


EG_SKETCH = {"residual": 0, "identity": 1, "gaussian": 2}
EG_FACTOR = {"triangular": 0, "qr": 1}


def _eg_workspace(ctx: Ctx, kmax: int):
    nbytes = int(load_library().plss_eg_workspace_bytes(ctx.handle, int(kmax)))
    if nbytes == 0:
        raise PlssError("plss_eg_workspace_bytes: invalid kmax or distributed ctx")
    ws = getattr(ctx, "_eg_ws", None)
    if ws is None or ws.numel() < nbytes + 256:
        ctx._eg_ws = None
        ws = ctx._eg_ws = _alloc_workspace(nbytes, ctx.A.row_ptr.device)
    return _aligned(ws), nbytes


def plss_eg_start(ctx: Ctx, b, sketch="residual", kmax=None, rows=None, seed=0, x0=None, tol=1e-8, tol_mode=0,
                  maxit=100, factor="triangular"):
    """Growing-sketch engine (Thm 2.1 / Cor 2.2, or the QR variant of section 2.3: factor="qr") with
    residual / identity / gaussian sketch columns."""
    lib = load_library()
    kmax = int(maxit if kmax is None else kmax)
    wp, nb = _eg_workspace(ctx, kmax)
    rr = _rows_arg(rows) if rows is not None else None
    ctx._keep = (b, x0, rr)
    ctx._maxit = int(maxit)
    _check(lib.plss_eg_start(ctx.handle, EG_SKETCH[sketch], EG_FACTOR[factor], kmax, wp, nb, _ptr(rr), int(seed) & 0xFFFFFFFFFFFFFFFF,
                             _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode), int(maxit)), ctx.handle)


def plss_eg_step(ctx: Ctx, k: int):
    _check(load_library().plss_eg_step(ctx.handle, int(k)), ctx.handle)


def plss_eg_finish(ctx: Ctx, x=None, want_hist=True, want_diag=False):
    lib = load_library()
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(ctx._maxit + 1) if want_hist else None
    diag = np.zeros((ctx._maxit + 1, REC)) if want_diag else None
    _check(lib.plss_eg_finish(ctx.handle, _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it), _ptr(hist), _ptr(diag), ctypes.byref(oc)),
           ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if hist is not None:
        res["hist"] = hist[:it.value + 1].copy()
    return res


def plss_eg_solve(ctx: Ctx, b, sketch="residual", kmax=None, rows=None, seed=0, x0=None, tol=1e-8, tol_mode=0,
                  maxit=100, x=None, want_hist=True, want_diag=False, factor="triangular"):
    """Full engine solve. Returns dict(x, iters, outcome, hist[0..iters][, diag])."""
    import torch
    lib = load_library()
    if x is None:
        x = torch.empty(ctx.n, dtype=torch.float64, device=ctx.A.row_ptr.device)
    kmax = int(maxit if kmax is None else kmax)
    wp, nb = _eg_workspace(ctx, kmax)
    rr = _rows_arg(rows) if rows is not None else None
    it = ctypes.c_int32(0)
    oc = ctypes.c_int(0)
    hist = np.zeros(maxit + 1) if want_hist else None
    diag = np.zeros((maxit + 1, REC)) if want_diag else None
    ctx._maxit = int(maxit)
    _check(lib.plss_eg_solve(ctx.handle, EG_SKETCH[sketch], EG_FACTOR[factor], kmax, wp, nb, _ptr(rr), int(seed) & 0xFFFFFFFFFFFFFFFF,
                             _vec(ctx, b, ctx.m, 'b'), _vec(ctx, x0, ctx.n, 'x0'), float(tol), int(tol_mode), int(maxit), _vec(ctx, x, ctx.n, 'x'), ctypes.byref(it),
                             _ptr(hist), _ptr(diag), ctypes.byref(oc)), ctx.handle)
    res = _result(it.value, oc.value, hist, diag, x)
    if hist is not None:
        res["hist"] = hist[:it.value + 1].copy()
    return res


def plss_eg_profile(ctx: Ctx, k: int) -> dict:
    ms = np.zeros(5)
    _check(load_library().plss_eg_profile(ctx.handle, int(k), _ptr(ms)), ctx.handle)
    return dict(zip(["sketch", "gemvT", "tri", "gemv", "k1"], ms.tolist()))   # QR: "tri" = reflector + T


def plss_destroy(ctx: Ctx):
    if ctx.handle:
        load_library().plss_destroy(ctx.handle)
        ctx.handle = None
