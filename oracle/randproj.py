"""Randomized projection ("Rand. Proj."), the paper's comparison method -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this module. It shares no code with the CUDA path (paper_2207_07615_b200/); the two sides
implement the same counter-based sketch generator independently (reading R17).

The method: eq:pkLong with W = I,

    p_k = A^T S_k (S_k^T A A^T S_k)^+ S_k^T (b - A x_{k-1}),      x_k = x_{k-1} + p_k   (eq:xko)

where S_k in R^{m x r} is drawn afresh every iteration: random standard normal (Experiment I,
L985-991, r = 10; Fig. 2, r = 10/20/40) or sparse normal (`sprandn`, Experiment III,
L1164-1170, r = 5 or 50). "If S_k is not in the range of A, the inverse ... is replaced by the
pseudo-inverse" (L166-167). Each iteration "recomputes Y_k = A^T S_k, Y_k^T Y_k and a solve with
the latter matrix" (L989-991). As in PLSS (eq:recRes, L663-666) the residual is carried
recursively, r_k = r_{k-1} - A p_k (reading R19).

Functions
* `sketch(seed, k, m, r, density)` -- S_k (m x r), the generator of reading R17. Entries are
  IEEE binary32 normals (stored here as float64 values): the paper fixes only "random standard
  normal" (L989-990), and eq:pkLong is the exact projection for whatever S_k is used, so the
  sketch needs no fp64 precision while the projection itself is computed in fp64.
    word(ctr)   = mix64(key + (ctr + 1) * G),  key = mix64(seed), G = 0x9E3779B97F4A7C15,
                  mix64 = the splitmix64 finalizer (xor-shift 30 / *0xBF58476D1CE4E5B9 /
                  xor-shift 27 / *0x94D049BB133111EB / xor-shift 31), all mod 2^64;
    pair (i, q) of row i holds columns 2q, 2q+1 (h = ceil(r/2) pairs per row);
    ctr         = ((k*2^32 + i)*h + q) * 256 + w   (word w < 4; a row's entries depend on
                  (seed, k, i, r) only, not on m: row blocks draw the same S);
    uniforms    (binary32) from ONE word per pair (ctr with w = 0):
                  u1 = 1 - (word >> 40) * 2^-24 in (0, 1],  u2 = ((word >> 16) & (2^24-1)) * 2^-24 in [0, 1);
    Box-Muller (binary32): R = sqrt(-2 ln u1), theta = 2 pi u2,
                  S[i, 2q] = R cos(theta), S[i, 2q+1] = R sin(theta);
    ln          = `ln_unit32`: frexp, one atanh series, only IEEE +,-,*,/ in binary32 (no FMA);
    sin / cos   = `sincos_2pi32`: exact octant reduction of 8 u2, Taylor polynomials of sin and cos
                  on [0, pi/4] (binary32 Horner, no FMA), octant symmetries;
    sparse S    (density < 1): entry (i, 2q+e) is kept iff (word(w = 2+e) >> 11) * 2^-53 < density
                  (compared in binary64).
  With every operation correctly rounded and in a fixed order, the CUDA side reproduces S
  bitwise (tests/test_gpu_randproj.py).
* `randproj(...)` -- the iteration above, dense pseudo-inverse, sequential stop test on the
  recursive residual (same test as PLSS: sqrt(rho_k)/||b|| <= tol or rho_k == 0).

Parity pins (tests/test_oracle_randproj.py): p_k is the minimum-norm solution of the sketched
constraint (eq:itProb-eq:cons with B = I, checked by LAPACK least squares); Pythagoras
||e_{k-1}||^2 = ||e_k||^2 + ||p_k||^2 (p_k is an orthogonal projection of the error); r = m
square S reaches A^+ b in one step (pseudo-inverse branch: S^T A A^T S is singular for m > n);
the sampler's moments / KS statistic against N(0, 1) and the sparse density.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_F32 = np.float32
LN2_32 = _F32(0.6931471805599453)               # RN32(ln 2) = 0x3F317218
SQRT_HALF_32 = _F32(0.7071067811865476)         # RN32(sqrt(1/2)) = 0x3F3504F3
_ATANH_COEF_32 = [_F32(1.0) / _F32(2 * j + 1) for j in range(5, -1, -1)]   # RN32(1/11), ..., 1
PI4_32 = _F32(np.pi / 4)                         # RN32(pi/4) = 0x3F490FDB
# Taylor coefficients RN32(+-1/(2j+1)!) (sin) and RN32(+-1/(2j)!) (cos), highest degree first
_SIN_COEF_32 = [_F32(1.0) / _F32(362880.0), _F32(-1.0) / _F32(5040.0), _F32(1.0) / _F32(120.0),
                _F32(-1.0) / _F32(6.0), _F32(1.0)]
_COS_COEF_32 = [_F32(-1.0) / _F32(3628800.0), _F32(1.0) / _F32(40320.0), _F32(-1.0) / _F32(720.0),
                _F32(1.0) / _F32(24.0), _F32(-0.5), _F32(1.0)]


def mix64(z):
    """splitmix64 finalizer on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def _word(key, ctr):
    return mix64(key + (ctr + np.uint64(1)) * _G)


def _unit(w):
    """53-bit uniform in [0, 1)."""
    return (w >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def ln_unit32(s):
    """ln(s) for binary32 s in (0, 1), every operation in binary32: s = m 2^e with m in
    [sqrt(1/2), sqrt(2)), f = (m-1)/(m+1), ln m = 2 f (1 + f^2/3 + ... + f^10/11) by Horner,
    ln s = e ln2 + ln m. |f| <= 0.1716, so the truncated series is exact to ~2e-9 relative."""
    s = np.asarray(s, dtype=_F32)
    mant, e = np.frexp(s)                      # exact; mant float32 in [0.5, 1)
    small = mant < SQRT_HALF_32
    mant = np.where(small, mant * _F32(2.0), mant).astype(_F32)
    e = np.where(small, e - 1, e).astype(_F32)
    f = (mant - _F32(1.0)) / (mant + _F32(1.0))
    f2 = f * f
    t = np.full_like(f, _ATANH_COEF_32[0])
    for c in _ATANH_COEF_32[1:]:
        t = t * f2 + c
    return e * LN2_32 + (_F32(2.0) * f) * t


def sincos_2pi32(u2):
    """(sin, cos)(2 pi u2) in binary32 for u2 in [0, 1) with 24-bit granularity: x = 8 u2 (exact),
    octant o = floor(x), f = x - o (exact), f <- 1 - f on odd octants (exact), phi = f RN32(pi/4),
    Taylor sin phi (to phi^9) and cos phi (to phi^10) by Horner in phi^2, octant symmetries."""
    u2 = np.asarray(u2, dtype=_F32)
    x = u2 * _F32(8.0)
    o = np.floor(x).astype(np.int64)
    f = x - o.astype(_F32)
    odd = (o & 1) == 1
    f = np.where(odd, _F32(1.0) - f, f).astype(_F32)
    phi = f * PI4_32
    p2 = phi * phi
    ts = np.full_like(p2, _SIN_COEF_32[0])
    for c in _SIN_COEF_32[1:]:
        ts = ts * p2 + c
    sn = phi * ts
    tc = np.full_like(p2, _COS_COEF_32[0])
    for c in _COS_COEF_32[1:]:
        tc = tc * p2 + c
    cs = tc
    # octant o: (sin theta, cos theta) from (sn, cs) of phi
    sin_t = np.select([o == 0, o == 1, o == 2, o == 3, o == 4, o == 5, o == 6],
                      [sn, cs, cs, sn, -sn, -cs, -cs], -sn).astype(_F32)
    cos_t = np.select([o == 0, o == 1, o == 2, o == 3, o == 4, o == 5, o == 6],
                      [cs, sn, -sn, -cs, -cs, -sn, sn], cs).astype(_F32)
    return sin_t, cos_t


def sketch(seed: int, k: int, m: int, r: int, density: float = 1.0) -> np.ndarray:
    """S_k in R^{m x r} (row-major), reading R17. k is the 1-based iteration index."""
    return sketch_rows(seed, k, np.arange(m), r, density)


def sketch_rows(seed: int, k: int, rows, r: int, density: float = 1.0) -> np.ndarray:
    """Rows `rows` of S_k (a row depends on (seed, k, i, r) only)."""
    rows = np.asarray(rows, dtype=np.uint64)
    m = rows.size
    h = (r + 1) // 2
    key = mix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    i = np.repeat(rows, h)
    q = np.tile(np.arange(h, dtype=np.uint64), m)
    base = ((np.uint64(k) << np.uint64(32)) + i) * np.uint64(h) + q
    w = _word(key, base * np.uint64(256))
    u1 = _F32(1.0) - (w >> np.uint64(40)).astype(_F32) * _F32(2.0 ** -24)
    u2 = ((w >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(_F32) * _F32(2.0 ** -24)
    rad = np.sqrt(_F32(-2.0) * ln_unit32(u1))
    sn, cs = sincos_2pi32(u2)
    z0 = (rad * cs).astype(_F32)
    z1 = (rad * sn).astype(_F32)
    if density < 1.0:
        c = base * np.uint64(256)
        z0 = np.where(_unit(_word(key, c + np.uint64(2))) < density, z0, _F32(0.0))
        z1 = np.where(_unit(_word(key, c + np.uint64(3))) < density, z1, _F32(0.0))
    assert z0.dtype == _F32 and z1.dtype == _F32
    S = np.empty((m, 2 * h))
    S[:, 0::2] = z0.reshape(m, h)
    S[:, 1::2] = z1.reshape(m, h)
    return np.ascontiguousarray(S[:, :r])


def randproj(A, b, r: int, seed: int, maxit: int, tol: float = 0.0, tol_mode: int = 0, x0=None,
             density: float = 1.0, keep: bool = False):
    """Rand. Proj. iterations (eq:pkLong, W = I, pseudo-inverse). A: scipy sparse or dense (m x n).

    Returns dict(x, iters, outcome, hist[0..], rank[1..]) and, with keep, the per-iteration S_k,
    p_k (small cases only)."""
    A = sp.csr_matrix(A) if not sp.issparse(A) else A.tocsr()
    m, n = A.shape
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    res = b - A @ x                             # r_0 = b - A x_0
    nb = float(np.linalg.norm(b)) if tol_mode == 0 else 1.0
    nb = nb if nb > 0 else 1.0
    rho = float(res @ res)
    hist = [np.sqrt(rho) / nb]
    ranks, Ss, ps = [], [], []
    outcome = "maxit"
    k = 0
    if rho == 0.0 or hist[0] <= tol:
        outcome = "converged"
    else:
        for k in range(1, maxit + 1):
            S = sketch(seed, k, m, r, density)
            Y = np.asarray(A.T @ S)             # Y_k = A^T S_k (L989-990)
            M = Y.T @ Y                          # S_k^T A A^T S_k
            v = S.T @ res                        # S_k^T (b - A x_{k-1})
            z = np.linalg.pinv(M) @ v            # (.)^+ (L166-167)
            p = Y @ z
            x = x + p                            # eq:xko
            res = res - A @ p                    # r_k = r_{k-1} - A p_k (reading R19)
            rho = float(res @ res)
            hist.append(np.sqrt(rho) / nb)
            ranks.append(int(np.linalg.matrix_rank(M)))
            if keep:
                Ss.append(S)
                ps.append(p)
            if rho == 0.0 or hist[-1] <= tol:
                outcome = "converged"
                break
        else:
            k = maxit
    out = {"x": x, "iters": k, "outcome": outcome, "hist": np.array(hist), "rank": np.array(ranks)}
    if keep:
        out["S"], out["P"] = Ss, ps
    return out
