"""Randomized projection ("Rand. Proj."), the paper's comparison method -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this module. It shares no code with the CUDA path (paper_2207_07615_b200/); the two sides
implement the same counter-based sketch generator independently (reading R7).

The method: eq:pkLong with W = I,

    p_k = A^T S_k (S_k^T A A^T S_k)^+ S_k^T (b - A x_{k-1}),      x_k = x_{k-1} + p_k   (eq:xko)

where S_k in R^{m x r} is drawn afresh every iteration: random standard normal (Experiment I,
L985-991, r = 10; Fig. 2, r = 10/20/40) or sparse normal (`sprandn`, Experiment III,
L1164-1170, r = 5 or 50). "If S_k is not in the range of A, the inverse ... is replaced by the
pseudo-inverse" (L166-167). Each iteration "recomputes Y_k = A^T S_k, Y_k^T Y_k and a solve with
the latter matrix" (L989-991). As in PLSS (eq:recRes, L663-666) the residual is carried
recursively, r_k = r_{k-1} - A p_k (reading R7).

Functions
* `sketch(seed, k, m, r, density)` -- S_k (m x r), the generator of reading R7:
    word(ctr)   = mix64(key + (ctr + 1) * G),  key = mix64(seed), G = 0x9E3779B97F4A7C15,
                  mix64 = the splitmix64 finalizer (xor-shift 30 / *0xBF58476D1CE4E5B9 /
                  xor-shift 27 / *0x94D049BB133111EB / xor-shift 31), all mod 2^64;
    pair (i, q) of row i holds columns 2q, 2q+1 (h = ceil(r/2) pairs per row);
    ctr         = (((k*2^32 + i)*h + q) * 64 + a) * 4 + w   (attempt a < 64, word w < 4; a row's
                  entries depend on (seed, k, i, r) only, not on m: row blocks draw the same S);
    uniforms    u = 2*((word >> 11) * 2^-53) - 1 (w = 0), v likewise (w = 1), in [-1, 1);
    Marsaglia's polar method: the first attempt with 0 < s = u*u + v*v < 1 gives
                  f = sqrt(-2 ln(s) / s), S[i, 2q] = u f, S[i, 2q+1] = v f (no attempt: 0, 0);
    ln          = `ln_unit` below: frexp, one atanh series, only IEEE +,-,*,/ (no FMA);
    sparse S    (density < 1): entry (i, 2q+e) is kept iff (word(w = 2+e) >> 11) * 2^-53 < density.
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
_ATTEMPTS = 64
_LN2 = 0.6931471805599453                       # RN(ln 2)
_SQRT_HALF = 0.7071067811865476
_ATANH_COEF = [1.0 / (2 * j + 1) for j in range(11, -1, -1)]   # 1/23, 1/21, ..., 1/3, 1


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


def ln_unit(s):
    """ln(s) for s in (0, 1): s = m 2^e with m in [sqrt(1/2), sqrt(2)), f = (m-1)/(m+1),
    ln m = 2 f (1 + f^2/3 + f^4/5 + ... + f^22/23) by Horner, ln s = e ln2 + ln m.
    |f| <= 0.1716, so the truncated series is exact to ~1e-17 relative."""
    s = np.asarray(s, dtype=np.float64)
    mant, e = np.frexp(s)                      # s = mant 2^e, mant in [0.5, 1)
    small = mant < _SQRT_HALF
    mant = np.where(small, mant * 2.0, mant)
    e = np.where(small, e - 1, e).astype(np.float64)
    f = (mant - 1.0) / (mant + 1.0)
    f2 = f * f
    t = np.full_like(f, _ATANH_COEF[0])
    for c in _ATANH_COEF[1:]:
        t = t * f2 + c
    return e * _LN2 + (2.0 * f) * t


def sketch(seed: int, k: int, m: int, r: int, density: float = 1.0) -> np.ndarray:
    """S_k in R^{m x r} (row-major), reading R7. k is the 1-based iteration index."""
    h = (r + 1) // 2
    key = mix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    i = np.repeat(np.arange(m, dtype=np.uint64), h)
    q = np.tile(np.arange(h, dtype=np.uint64), m)
    base = ((np.uint64(k) << np.uint64(32)) + i) * np.uint64(h) + q
    z0 = np.zeros(m * h)
    z1 = np.zeros(m * h)
    todo = np.arange(m * h)
    for a in range(_ATTEMPTS):
        if todo.size == 0:
            break
        c = (base[todo] * np.uint64(_ATTEMPTS) + np.uint64(a)) * np.uint64(4)
        u = 2.0 * _unit(_word(key, c)) - 1.0
        v = 2.0 * _unit(_word(key, c + np.uint64(1))) - 1.0
        s = u * u + v * v
        ok = (s > 0.0) & (s < 1.0)
        so = s[ok]
        f = np.sqrt((-2.0 * ln_unit(so)) / so)
        z0[todo[ok]] = u[ok] * f
        z1[todo[ok]] = v[ok] * f
        todo = todo[~ok]
    if density < 1.0:
        c = base * np.uint64(_ATTEMPTS * 4)
        z0 = np.where(_unit(_word(key, c + np.uint64(2))) < density, z0, 0.0)
        z1 = np.where(_unit(_word(key, c + np.uint64(3))) < density, z1, 0.0)
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
            res = res - A @ p                    # r_k = r_{k-1} - A p_k (reading R7)
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
