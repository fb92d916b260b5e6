"""Exact-rational Algorithm 1 -- TEST INFRASTRUCTURE ONLY.

Algorithm 1 with WI = I or a rational diagonal WI, in fractions.Fraction
arithmetic. Algorithm 1's
tau = sqrt(theta*phi)/rho only enters through (tau-1)(tau+1) = theta*phi/rho^2 - 1, so
beta = 1/((tau-1)(tau+1)) = rho^2/(theta*phi - rho^2) is rational (Thm 4.1 proof, PAPER.md
L697-707) and gamma = (theta/rho)*beta (L809). No square root is ever needed; the stop test is
exact: r = 0.
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence


def _F(v):
    return v if isinstance(v, Fraction) else Fraction(v)


def matvec(A: Sequence[Sequence[Fraction]], x: Sequence[Fraction]) -> List[Fraction]:
    return [sum((a * xi for a, xi in zip(row, x)), Fraction(0)) for row in A]


def matvecT(A: Sequence[Sequence[Fraction]], u: Sequence[Fraction]) -> List[Fraction]:
    n = len(A[0]) if A else 0
    return [sum((A[i][j] * u[i] for i in range(len(A))), Fraction(0)) for j in range(n)]


def dotq(a, b) -> Fraction:
    return sum((ai * bi for ai, bi in zip(a, b)), Fraction(0))


def plss_exact(A, b, x0=None, maxit=None, wi=None):
    """Run Algorithm 1 exactly until r = 0 (or maxit updates). wi: the diagonal of WI (rational;
    None = identity): WIy = y ./ wi, phi = y^T WIy, p = beta p + gamma WIy, theta = p^T (WI p)
    (PLSS W).

    Returns dict with x, iters, converged, and per-step lists: rho (rho_0..), p (p_1..),
    r (r_0..), y (y_1..), beta, gamma, psi (y_k^T p_{k-1}, k >= 2).
    """
    A = [[_F(a) for a in row] for row in A]
    m = len(A)
    n = len(A[0]) if m else 0
    b = [_F(v) for v in b]
    x = [_F(v) for v in x0] if x0 is not None else [Fraction(0)] * n
    w = [_F(v) for v in wi] if wi is not None else [Fraction(1)] * n
    wdiv = lambda y: [yi / wj for yi, wj in zip(y, w)]           # WI \ y  (L788, L805)
    wdot = lambda p: sum((pi * wj * pi for pi, wj in zip(p, w)), Fraction(0))   # p^T (WI p)
    maxit = maxit if maxit is not None else 4 * max(m, n, 1)
    r = [bi - ai for bi, ai in zip(b, matvec(A, x))]          # r0 = b - A x0   (L786)
    out = {"rho": [], "p": [], "r": [list(r)], "y": [], "beta": [], "gamma": [], "psi": [],
           "theta": [], "phi": []}
    rho = dotq(r, r)                                           # (L788)
    out["rho"].append(rho)
    if rho == 0:
        return dict(out, x=x, iters=0, converged=True)
    y = matvecT(A, r)                                          # y1 = A^T r0  (L786)
    wy = wdiv(y)
    phi = dotq(y, wy)                                          # (L789)
    if phi == 0:
        return dict(out, x=x, iters=0, converged=False)
    p = [rho / phi * yi for yi in wy]                          # p1 = (rho/phi) WIy  (L795)
    theta = wdot(p)                                            # (L796)
    x = [xi + pi for xi, pi in zip(x, p)]                      # (L797)
    out["y"].append(y); out["p"].append(p); out["phi"].append(phi); out["theta"].append(theta)
    iters = 1
    while iters < maxit:
        Ap = matvec(A, p)
        r = [ri - api for ri, api in zip(r, Ap)]               # r = r - A p  (L801)
        rho = dotq(r, r)                                       # (L804)
        out["r"].append(list(r)); out["rho"].append(rho)
        if rho == 0:
            return dict(out, x=x, iters=iters, converged=True)
        y = matvecT(A, r)                                      # (L802)
        wy = wdiv(y)                                           # (L805)
        phi = dotq(y, wy)                                      # (L806)
        out["psi"].append(dotq(y, p))
        denom = theta * phi - rho * rho                        # rho^2((tau-1)(tau+1))
        if denom == 0 or phi == 0:
            return dict(out, x=x, iters=iters, converged=False)
        beta = rho * rho / denom                               # (L807-808)
        gamma = (theta / rho) * beta                           # (L809)
        p = [beta * pi + gamma * yi for pi, yi in zip(p, wy)]  # (L811)
        theta = wdot(p)                                        # (L812)
        x = [xi + pi for xi, pi in zip(x, p)]                  # (L813)
        out["y"].append(y); out["p"].append(p); out["beta"].append(beta)
        out["gamma"].append(gamma); out["phi"].append(phi); out["theta"].append(theta)
        iters += 1
    Ap = matvec(A, p)
    r = [ri - api for ri, api in zip(r, Ap)]
    out["r"].append(list(r)); out["rho"].append(dotq(r, r))
    return dict(out, x=x, iters=iters, converged=out["rho"][-1] == 0)


def rank_exact(A) -> int:
    """Rank by exact Gaussian elimination (test helper)."""
    M = [[_F(a) for a in row] for row in A]
    rows, cols = len(M), len(M[0]) if M else 0
    rk = 0
    for c in range(cols):
        piv = next((i for i in range(rk, rows) if M[i][c] != 0), None)
        if piv is None:
            continue
        M[rk], M[piv] = M[piv], M[rk]
        for i in range(rows):
            if i != rk and M[i][c] != 0:
                f = M[i][c] / M[rk][c]
                M[i] = [a - f * bb for a, bb in zip(M[i], M[rk])]
        rk += 1
    return rk


def solve_exact(M, v):
    """Solve a nonsingular square system exactly (Gauss-Jordan)."""
    k = len(M)
    aug = [[_F(a) for a in row] + [_F(vi)] for row, vi in zip(M, v)]
    for c in range(k):
        piv = next(i for i in range(c, k) if aug[i][c] != 0)
        aug[c], aug[piv] = aug[piv], aug[c]
        pv = aug[c][c]
        aug[c] = [a / pv for a in aug[c]]
        for i in range(k):
            if i != c and aug[i][c] != 0:
                f = aug[i][c]
                aug[i] = [a - f * bb for a, bb in zip(aug[i], aug[c])]
    return [aug[i][k] for i in range(k)]
