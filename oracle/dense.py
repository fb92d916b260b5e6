"""Dense brute-force pins for the PLSS oracle -- TEST INFRASTRUCTURE ONLY.

These are independent of Algorithm 1's short recursion and of each other:

* `min_norm_solution`  -- A^+ b via numpy.linalg.pinv: the limit x_n = A^+ b of Thm 3.1
                           and of Cor 3.3 (L583-609) from x0 = 0.
* `pk_long_iterates`   -- the closed-form update eq:pkLong (L151-167), W = I, with the residual
                          sketch S_k = [r_0 ... r_{k-1}] of eq:S (L611-626), pseudo-inverse form.
                          Thm 4.1 (L628-712) states the short recursion reproduces these updates.
* `craig_updates`      -- Craig's method via Golub-Kahan bidiagonalization (eq:bidiag1/2,
                          eq:craigRes, L833-854; zeta_k = -(beta_k/alpha_k) zeta_{k-1}, zeta_0 = -1,
                          L875). Thm 6.1 (L858-929): its updates equal the PLSS updates when W = I.
"""
from __future__ import annotations

import numpy as np


def min_norm_solution(A, b):
    return np.linalg.pinv(np.asarray(A, dtype=np.float64)) @ np.asarray(b, dtype=np.float64)


def pk_long_iterates(A, b, K, x0=None):
    """Iterate x_k = x_{k-1} + p_k, p_k = A^T S_k (S_k^T A A^T S_k)^+ S_k^T r_{k-1}, S_k = [r_0..r_{k-1}].

    Returns (updates [p_1..p_K], iterates [x_1..x_K]).
    """
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros(A.shape[1]) if x0 is None else np.array(x0, dtype=np.float64)
    S = []
    ps, xs = [], []
    for _ in range(K):
        r = b - A @ x                       # r_{k-1} := b - A x_{k-1}
        S.append(r)
        Sk = np.stack(S, axis=1)            # eq:S
        Y = A.T @ Sk                        # Y_k = A^T S_k (eq:yk)
        p = Y @ (np.linalg.pinv(Y.T @ Y) @ (Sk.T @ r))
        x = x + p                           # eq:xko
        ps.append(p)
        xs.append(x.copy())
    return ps, xs


def craig_updates(A, b, K):
    """Craig's updates zeta_k v_k by Golub-Kahan bidiagonalization from x0 = 0 (Paige-Saunders)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    beta = np.linalg.norm(b)                # beta_1 u_1 = b
    u = b / beta
    w = A.T @ u
    alpha = np.linalg.norm(w)               # alpha_1 v_1 = A^T u_1
    v = w / alpha
    zeta_prev = -1.0                        # zeta_0 = -1
    ups = []
    for _ in range(K):
        zeta = -(beta / alpha) * zeta_prev  # zeta_k = -(beta_k/alpha_k) zeta_{k-1}
        ups.append(zeta * v)                # p_k^C = zeta_k v_k
        # next bidiagonalization step: beta_{k+1} u_{k+1} = A v_k - alpha_k u_k, ...
        t = A @ v - alpha * u
        beta = np.linalg.norm(t)
        if beta == 0:
            break
        u = t / beta
        w = A.T @ u - beta * v
        alpha = np.linalg.norm(w)
        if alpha == 0:
            break
        v = w / alpha
        zeta_prev = zeta
    return ups
