"""PLSS CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package. The product path (paper_2207_07615_b200/) never imports it and never falls
back to it.

* `plss_oracle.c`   -- Algorithm 1 in plain binary64 C, sequential sums;
                       WI = I (PLSS) or a diagonal WI (PLSS W, L714-765), `column_norms`.
* `exact.py`        -- the same algorithm in exact rational arithmetic (fractions.Fraction).
* `dense.py`        -- brute-force pins: pseudo-inverse min-norm solution (Thm 3.1 / Cor 3.3),
                       the closed-form update eq:pkLong (L151-167) with the residual sketch
                       eq:S (L611-626), Craig's method by Golub-Kahan bidiagonalization (Thm 6.1,
                       L833-929).

Parity status of each function is listed in DESIGN.md ("Oracle and its pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "plss_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

REC = 8  # per-iteration record: hist, rho, phi, psi, theta, tau, beta, gamma
FREEZE_H = 64 * np.finfo(np.float64).eps  # SURVEY 8c-5 freeze threshold (~1.4e-14)
OUTCOMES = {0: "converged", 1: "maxit", 2: "y_vanished", 3: "stagnation"}


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               _SRC, "-o", _LIB_PATH + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.oracle_spmv.argtypes = [ctypes.c_int64, P, P, P, P, P]
        lib.oracle_spmvT.argtypes = [ctypes.c_int64, P, P, P, P, P]
        lib.oracle_plss.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P, P, P, P, P, P,
                                    ctypes.c_double, ctypes.c_int, ctypes.c_int32, ctypes.c_int,
                                    ctypes.c_double, P, P, P, P]
        lib.oracle_column_norms.argtypes = [ctypes.c_int64, P, P, P]
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_get_threads.restype = ctypes.c_int
        lib.oracle_plss.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class threads:
    """Context manager: run the oracle on `t` host threads (oracle_set_threads; t = 1 is the
    sequential oracle). `t = None` or 0: all host cores (os.cpu_count())."""

    def __init__(self, t=None):
        self.t = int(t) if t else (os.cpu_count() or 1)

    def __enter__(self):
        lib = _load()
        self.prev = lib.oracle_get_threads()
        lib.oracle_set_threads(self.t)
        return self

    def __exit__(self, *a):
        _load().oracle_set_threads(self.prev)


def spmv(m, row_ptr, col_idx, val, x):
    """y = A x over CSR (sequential ascending-column sums)."""
    lib = _load()
    rp, ci, v, xx = _i32(row_ptr), _i32(col_idx), _f64(val), _f64(x)
    y = np.empty(m, dtype=np.float64)
    lib.oracle_spmv(m, _p(rp), _p(ci), _p(v), _p(xx), _p(y))
    return y


def spmvT(n, col_ptr, row_idx, val_t, u):
    """v = A^T u over the CSC copy (sequential ascending-row sums)."""
    lib = _load()
    cp, ri, v, uu = _i32(col_ptr), _i32(row_idx), _f64(val_t), _f64(u)
    out = np.empty(n, dtype=np.float64)
    lib.oracle_spmvT(n, _p(cp), _p(ri), _p(v), _p(uu), _p(out))
    return out


def column_norms(n, col_ptr, val_t):
    """c_j = ||A_{:,j}|| (ascending sum of squares, sqrt; zero columns 1): PLSS W's WI diagonal."""
    lib = _load()
    cp, vt = _i32(col_ptr), _f64(val_t)
    c = np.empty(n, dtype=np.float64)
    lib.oracle_column_norms(n, _p(cp), _p(vt), _p(c))
    return c


def plss(m, n, row_ptr, col_idx, val, col_ptr, row_idx, val_t, b, x0=None, tol=1e-8,
         tol_mode=0, maxit=100, freeze=False, freeze_h=FREEZE_H, keep_updates=False, wi=None):
    """Algorithm 1 (WI = I, or WI = diag(wi): PLSS W). Returns dict(x, iters, outcome,
    rec[(maxit+1), 8], hist[, P]).

    keep_updates: also return P[iters, n], the updates p_1..p_iters (small cases only)."""
    lib = _load()
    rp, ci, v = _i32(row_ptr), _i32(col_idx), _f64(val)
    cp, ri, vt = _i32(col_ptr), _i32(row_idx), _f64(val_t)
    bb = _f64(b)
    xx0 = _f64(x0) if x0 is not None else None
    ww = _f64(wi) if wi is not None else None
    x = np.empty(n, dtype=np.float64)
    it = ctypes.c_int32(0)
    rec = np.zeros((maxit + 1, REC), dtype=np.float64)
    P = np.zeros((maxit, n), dtype=np.float64) if keep_updates else None
    out = lib.oracle_plss(m, n, _p(rp), _p(ci), _p(v), _p(cp), _p(ri), _p(vt), _p(bb), _p(xx0), _p(ww),
                          float(tol), int(tol_mode), int(maxit), int(bool(freeze)), float(freeze_h),
                          _p(x), ctypes.byref(it), _p(rec), _p(P))
    iters = it.value
    # hist_k is recorded at the start of loop step k; a run that ends by the iteration cap (or
    # runs the fixed count in freeze mode) never evaluates hist_{iters}.
    nh = iters if (out == 1 or freeze) else iters + 1
    res = {"x": x, "iters": iters, "outcome": OUTCOMES[out], "outcome_code": out, "rec": rec,
           "hist": rec[:max(nh, 1), 0].copy()}
    if keep_updates:
        res["P"] = P[:iters]
    return res


def plss_system(s, x0=None, **kw):
    """Run the oracle on a plss_gen.System with its own tol / mode / cap unless overridden."""
    args = dict(tol=s.tol, tol_mode=s.tol_mode, maxit=s.maxit, freeze=s.freeze)
    args.update(kw)
    return plss(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t, s.b,
                x0=x0, **args)
