"""Growing-sketch engine with the triangular factorization (section 2.4, Thm 2.1 and
Cor 2.2, L284-441) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this module. It shares no code with the CUDA path (paper_2207_07615_b200/).

For any sketch column s_k (eq:genS, L200-207) with y_k = A^T s_k (eq:yk, L236-244) and the stored
Y_{k-1} = [y_1 .. y_{k-1}], R_{k-1} = [t_1 .. t_{k-1}] (upper triangular, t_j = [t_hat_j; -1; 0]),
D_{k-1} = diag(1/delta_j), the engine computes (Thm 2.1 eq:Nkrec; Cor 2.2 eq:compute-pk-alpha1):

    g       = Y_{k-1}^T y_k
    t_hat_k = R_{k-1} D_{k-1} R_{k-1}^T g          (= N_{k-1} Y_{k-1}^T y_k, "2 multiplications with
                                                   triangular matrices only", L432-435)
    delta_k = y_k^T y_k - g^T t_hat_k
    p_k     = (s_k^T r_{k-1} / delta_k) (y_k - Y_{k-1} t_hat_k)
    append y_k to Y, t_k to R, 1/delta_k to D;  x_k = x_{k-1} + p_k;  r_k = r_{k-1} - A p_k

N_k = (Y_k^T Y_k)^{-1} is never formed and no system is solved. Sketch columns (`sketch`):
  "residual"  s_k = r_{k-1} (eq:S, L611-626): Thm 4.1 says the updates are PLSS's;
  "identity"  s_k = e_{rows[k-1]} (section 7): PLSS Kaczmarz's updates;
  "gaussian"  s_k = column 0 of randproj.sketch(seed, k, m, 1) (binary32 normals, reading R17).
Readings (R22): delta_k <= 1e-14 y_k^T y_k (y_k numerically in range(Y_{k-1})), y_k = 0
or s_k^T r_{k-1} = 0 skip the step (p_k = 0, nothing appended); after kmax stored columns the
history is cleared (as R21). The residual is recursive (R19).

`qr_engine` is the QR variant (section 2.3, eq:ykeqQR / eq:pkQR, L247-282): Y_k = Q_k T_k by a
Householder QR (LAPACK through numpy, recomputed each step: the definition, not the update) and
p_k = (s_k^T r_{k-1} / r_kk) q_k with q_k, r_kk the last column of Q_k and last diagonal of T_k;
the skip rule compares r_kk^2 (= delta_k) with 1e-14 y_k^T y_k.

Parity pins (tests/test_oracle_engine.py): R D R^T equals inv(Y^T Y) (Thm 2.1); iterates equal
eq:pkLong with the same sketch through a dense pseudo-inverse (both engines); residual sketch ==
the PLSS oracle (Thm 4.1); identity sketch == the PLSS Kaczmarz oracle; orthogonal updates.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import randproj

SKIP_REL = 1e-14


def sketch_column(kind, k, m, r, rows=None, seed=0):
    """s_k for the given sketch kind (k is 1-based; r = r_{k-1})."""
    if kind == "residual":
        return r.copy()
    if kind == "identity":
        s = np.zeros(m)
        s[int(rows[k - 1])] = 1.0
        return s
    if kind == "gaussian":
        return randproj.sketch(seed, k, m, 1)[:, 0]
    raise ValueError(kind)


def tri_engine(A, b, sketch="residual", maxit=100, tol=0.0, tol_mode=0, x0=None, rows=None, seed=0,
               kmax=None, keep=False):
    A = sp.csr_matrix(A) if not sp.issparse(A) else A.tocsr()
    m, n = A.shape
    b = np.asarray(b, dtype=np.float64)
    kmax = maxit if kmax is None else int(kmax)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - A @ x
    nb = float(np.linalg.norm(b)) if tol_mode == 0 else 1.0
    nb = nb if nb > 0 else 1.0
    rho = float(r @ r)
    hist = [np.sqrt(rho) / nb]
    Y, T, dinv = [], [], []            # y_j, t_hat_j (length j-1), 1/delta_j
    allP, deltas = [], []
    skipped = 0
    outcome = "maxit"
    k = 0
    if rho == 0.0 or hist[0] <= tol:
        outcome = "converged"
    else:
        for k in range(1, maxit + 1):
            s = sketch_column(sketch, k, m, r, rows, seed)
            y = A.T @ s                                    # y_k = A^T s_k (eq:yk)
            rs = float(s @ r)                              # s_k^T r_{k-1}
            yy = float(y @ y)
            h = len(Y)
            if h:
                Yk = np.stack(Y, axis=1)
                g = Yk.T @ y
                R = np.zeros((h, h))                        # R_{k-1} = [t_1 .. t_h]
                for j, tj in enumerate(T):
                    R[:j, j] = tj
                    R[j, j] = -1.0
                that = R @ (np.array(dinv) * (R.T @ g))     # R D R^T g
                delta = yy - float(g @ that)
            else:
                Yk, that, delta = None, np.zeros(0), yy
            if yy == 0.0 or delta <= SKIP_REL * yy or rs == 0.0:
                skipped += 1                               # reading R22
            else:
                d = y - (Yk @ that if h else 0.0)
                p = (rs / delta) * d                       # Cor 2.2
                x = x + p
                r = r - A @ p
                Y.append(y)
                T.append(that)
                dinv.append(1.0 / delta)
                deltas.append(delta)
                if keep:
                    allP.append(p)
                if len(Y) == kmax:
                    Y, T, dinv = [], [], []
            rho = float(r @ r)
            hist.append(np.sqrt(rho) / nb)
            if rho == 0.0 or hist[-1] <= tol:
                outcome = "converged"
                break
        else:
            k = maxit
    out = {"x": x, "iters": k, "outcome": outcome, "hist": np.array(hist), "skipped": skipped,
           "delta": np.array(deltas)}
    if keep:
        out["P"] = allP
    return out


def qr_engine(A, b, sketch="residual", maxit=100, tol=0.0, tol_mode=0, x0=None, rows=None, seed=0,
              kmax=None, keep=False):
    """eq:pkQR: p_k = (s_k^T r_{k-1} / r_kk) q_k from the Householder QR of Y_k (section 2.3)."""
    A = sp.csr_matrix(A) if not sp.issparse(A) else A.tocsr()
    m, n = A.shape
    b = np.asarray(b, dtype=np.float64)
    kmax = maxit if kmax is None else int(kmax)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - A @ x
    nb = float(np.linalg.norm(b)) if tol_mode == 0 else 1.0
    nb = nb if nb > 0 else 1.0
    rho = float(r @ r)
    hist = [np.sqrt(rho) / nb]
    Y, allP = [], []
    skipped = 0
    outcome = "maxit"
    k = 0
    if rho == 0.0 or hist[0] <= tol:
        outcome = "converged"
    else:
        for k in range(1, maxit + 1):
            s = sketch_column(sketch, k, m, r, rows, seed)
            y = A.T @ s
            rs = float(s @ r)
            yy = float(y @ y)
            if len(Y) < n and yy > 0.0:
                Q, T = np.linalg.qr(np.stack(Y + [y], axis=1))     # Householder (LAPACK geqrf)
                rkk = float(T[-1, -1])
            else:
                rkk = 0.0
            if yy == 0.0 or rkk * rkk <= SKIP_REL * yy or rs == 0.0:
                skipped += 1                                       # reading R22
            else:
                p = (rs / rkk) * Q[:, -1]                          # eq:pkQR
                x = x + p
                r = r - A @ p
                Y.append(y)
                if keep:
                    allP.append(p)
                if len(Y) == kmax:
                    Y = []
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


def rdrt_inverse(Ys):
    """N_k = R_k D_k R_k^T built by the recursion of Thm 2.1 from the columns Ys (for the pin)."""
    T, dinv = [], []
    for k, y in enumerate(Ys):
        if k:
            Yk = np.stack(Ys[:k], axis=1)
            g = Yk.T @ y
            R = np.zeros((k, k))
            for j, tj in enumerate(T):
                R[:j, j] = tj
                R[j, j] = -1.0
            that = R @ (np.array(dinv) * (R.T @ g))
            delta = float(y @ y) - float(g @ that)
        else:
            that, delta = np.zeros(0), float(y @ y)
        T.append(that)
        dinv.append(1.0 / delta)
    K = len(Ys)
    R = np.zeros((K, K))
    for j, tj in enumerate(T):
        R[:j, j] = tj
        R[j, j] = -1.0
    return R @ np.diag(dinv) @ R.T
