"""PLSS Kaczmarz (section 7) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this module. It shares no code with the CUDA path (paper_2207_07615_b200/).

The sketch is a growing set of identity columns S_k = [e_{i_1} ... e_{i_k}] in a random order
(L933-936; the row order is an INPUT, `rows`). With y_k = A^T e_{i_k} = a_{i_k} (L950-951) and the
orthogonal updates P_{k-1} = [p_1 ... p_{k-1}], Theta_{k-1} = diag(p_j^T p_j), eq:pkKacz
(L952-956):

    d_{k-1}   = Theta_{k-1}^{-1/2} P_{k-1}^T a_{i_k}
    gamma_{k-1} = e_{i_k}^T (b - A x_{k-1}) / ((||a_{i_k}|| - ||d_{k-1}||)(||a_{i_k}|| + ||d_{k-1}||))
    p_k       = gamma_{k-1} (a_{i_k} - P_{k-1} Theta_{k-1}^{-1} P_{k-1}^T a_{i_k})

P_{k-1}^T a_{i_k} is read from the stored [A p_1 ... A p_{k-1}] (row i_k of that m x (k-1) array,
L961-966: (A p_j)_i = a_i^T p_j); A p_k is computed once per step and appended; the residual is
carried as r_k = r_{k-1} - A p_k (reading R19's recursive residual; e_{i_k}^T (b - A x_{k-1}) is
r_{k-1}[i_k]). Readings (R20, R21): a row with ||a||^2 - ||d||^2 <= 1e-14 ||a||^2 (in
the span of the history, or empty) or already satisfied (r_{k-1}[i_k] = 0: p_k = 0, and a zero
column would make Theta singular) is skipped (p_k = 0, nothing appended); after `kmax` stored
updates the history is cleared and the next updates start a new history at the current x.

Parity pins (tests/test_oracle_kaczmarz.py): the worked diag(2,1) example (SPEC.md L326-349:
p_1 = (1,0), p_2 = (0,1), x = (1,1)); the first step is classical Kaczmarz (P_0 = 0, L956-958);
iterates equal eq:pkLong with the identity-column sketch through a dense pseudo-inverse
(oracle/dense.py route, not this recursion); mutually orthogonal updates; visited rows have zero
residual (S_k^T r_k = 0); one-sweep termination at the minimum-norm solution on full-row-rank
systems; repeated rows are skipped.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

SKIP_REL = 1e-14


def kz_solve(A, b, rows, maxit, tol=0.0, tol_mode=0, x0=None, kmax=None, keep=False):
    """PLSS Kaczmarz. A: scipy sparse or dense (m x n); rows: row order (length >= maxit).

    Returns dict(x, iters, outcome, hist[0..iters], skipped, rec) and with keep the updates P."""
    A = sp.csr_matrix(A) if not sp.issparse(A) else A.tocsr()
    m, n = A.shape
    b = np.asarray(b, dtype=np.float64)
    rows = np.asarray(rows, dtype=np.int64)
    kmax = maxit if kmax is None else int(kmax)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - A @ x                                       # r_0
    nb = float(np.linalg.norm(b)) if tol_mode == 0 else 1.0
    nb = nb if nb > 0 else 1.0
    rho = float(r @ r)
    hist = [np.sqrt(rho) / nb]
    P, AP, theta = [], [], []                           # history: p_j, A p_j, p_j^T p_j
    allP = []
    skipped = 0
    outcome = "maxit"
    k = 0
    if rho == 0.0 or hist[0] <= tol:
        outcome = "converged"
    else:
        for k in range(1, maxit + 1):
            i = int(rows[k - 1])
            lo, hi = A.indptr[i], A.indptr[i + 1]
            cols, vals = A.indices[lo:hi], A.data[lo:hi]
            a = np.zeros(n)
            a[cols] = vals                              # a_{i_k} = A^T e_{i_k}
            aa = float(vals @ vals)
            g = np.array([apj[i] for apj in AP])        # P^T a_i from the stored A p_j (L961-966)
            th = np.array(theta)
            dd = float(np.sum(g * g / th)) if len(g) else 0.0      # ||d||^2
            na, nd = np.sqrt(aa), np.sqrt(dd)
            denom = (na - nd) * (na + nd)
            if aa == 0.0 or denom <= SKIP_REL * aa or r[i] == 0.0:
                skipped += 1                            # reading R20
                p = None
            else:
                gamma = r[i] / denom                    # e_i^T (b - A x_{k-1}) / (...)
                w = g / th if len(g) else np.zeros(0)   # Theta^{-1} P^T a_i
                corr = np.stack(P, axis=1) @ w if P else np.zeros(n)
                p = gamma * (a - corr)                  # eq:pkKacz
                Ap = A @ p
                x = x + p
                r = r - Ap
                P.append(p)
                AP.append(Ap)
                theta.append(float(p @ p))
                if keep:
                    allP.append(p)
                if len(P) == kmax:                      # reading R21: history reset
                    P, AP, theta = [], [], []
            rho = float(r @ r)
            hist.append(np.sqrt(rho) / nb)
            if rho == 0.0 or hist[-1] <= tol:
                outcome = "converged"
                break
        else:
            k = maxit
    out = {"x": x, "iters": k, "outcome": outcome, "hist": np.array(hist), "skipped": skipped}
    if keep:
        out["P"] = allP
    return out


def classical_kaczmarz_step(A, b, x, i):
    """x + ((b_i - a_i^T x) / ||a_i||^2) a_i (the P_{k-1} = 0 case, L956-958)."""
    A = sp.csr_matrix(A) if not sp.issparse(A) else A.tocsr()
    a = np.asarray(A.getrow(i).todense()).ravel()
    return x + ((b[i] - a @ x) / (a @ a)) * a
