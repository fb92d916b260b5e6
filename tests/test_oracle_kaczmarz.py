"""Pins of the PLSS Kaczmarz oracle (oracle/kaczmarz.py) against what the paper fixes, by routes
independent of its recursion:

* the worked example A = diag(2,1), b = (2,1), rows (0, 1): p_1 = (1,0), p_2 = (0,1), x = (1,1)
  (derived from eq:pkKacz by hand; tests/golden/kaczmarz_diag21.json);
* the first step is the classical Kaczmarz step (P_0 = 0);
* the iterates equal eq:pkLong (L151-167) with the identity-column sketch S_k = [e_{i_1}..e_{i_k}]
  evaluated through a dense pseudo-inverse (L933-950: "the updates with this sketch are (cf.
  eq:pkLong)");
* orthogonal updates; visited rows have zero residual (eq:orthSr with identity columns);
  one-sweep termination at the minimum-norm solution A^+ b on full-row-rank systems (Cor 3.2/3.3);
* a repeated row (in the span of the history) is skipped (reading R20); history reset (R21)
  keeps each segment a valid run.
"""
import json
import os

import numpy as np
import scipy.sparse as sp

from oracle import dense
from oracle import kaczmarz as kz

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "kaczmarz_diag21.json")


def _system(seed=0, m=15, n=25, dens=0.4):
    rng = np.random.default_rng(seed)
    A = sp.random(m, n, density=dens, random_state=rng, data_rvs=rng.standard_normal).tocsr()
    A = (A + sp.csr_matrix((np.ones(m), (np.arange(m), rng.choice(n, m, replace=False))), shape=(m, n))).tocsr()
    b = A @ rng.standard_normal(n)
    return A, b


def test_worked_example_diag21():
    g = json.load(open(GOLDEN))
    A = np.array(g["A"], dtype=float)
    b = np.array(g["b"], dtype=float)
    out = kz.kz_solve(A, b, g["rows"], maxit=2, keep=True)
    for p, pe in zip(out["P"], g["p"]):
        np.testing.assert_array_equal(p, pe)
    np.testing.assert_array_equal(out["x"], g["x"])
    assert out["outcome"] == "converged" and out["iters"] == 2


def test_first_step_is_classical_kaczmarz():
    A, b = _system()
    for i in (0, 3, 7):
        out = kz.kz_solve(A, b, [i], maxit=1)
        ref = kz.classical_kaczmarz_step(A, b, np.zeros(A.shape[1]), i)
        np.testing.assert_allclose(out["x"], ref, rtol=0, atol=1e-14 * np.linalg.norm(ref))


def _pk_long_identity(A, b, rows, K):
    """x_k by eq:pkLong with S_k = [e_{i_1} .. e_{i_k}] and a dense pseudo-inverse."""
    Ad = A.toarray()
    m, n = Ad.shape
    x = np.zeros(n)
    xs = []
    for k in range(1, K + 1):
        S = np.zeros((m, k))
        S[rows[:k], np.arange(k)] = 1.0
        r = b - Ad @ x
        Y = Ad.T @ S
        x = x + Y @ (np.linalg.pinv(Y.T @ Y) @ (S.T @ r))
        xs.append(x.copy())
    return xs


def test_equals_pk_long_with_identity_sketch():
    for seed in range(5):
        A, b = _system(seed, m=12, n=20)
        rows = np.random.default_rng(seed).permutation(12)
        ref = _pk_long_identity(A, b, rows, 12)
        x = np.zeros(20)
        out = kz.kz_solve(A, b, rows, maxit=12, keep=True)
        for p, xr in zip(out["P"], ref):
            x = x + p
            np.testing.assert_allclose(x, xr, rtol=0, atol=1e-8 * max(1.0, np.linalg.norm(xr)))


def test_orthogonal_updates_and_visited_rows():
    A, b = _system(1, m=15, n=25)
    rows = np.random.default_rng(1).permutation(15)
    out = kz.kz_solve(A, b, rows, maxit=10, keep=True)
    P = np.stack(out["P"], axis=1)
    G = P.T @ P
    nrm = np.sqrt(np.diag(G))
    off = np.abs(G - np.diag(np.diag(G))) / np.outer(nrm, nrm)
    assert off.max() <= 1e-10
    r = b - A @ out["x"]
    assert np.max(np.abs(r[rows[:10]])) <= 1e-10 * np.linalg.norm(b)


def test_one_sweep_min_norm_termination():
    for seed in range(10):
        A, b = _system(seed, m=15, n=25)
        rows = np.random.default_rng(100 + seed).permutation(15)
        out = kz.kz_solve(A, b, rows, maxit=15, tol=1e-8)
        assert out["outcome"] == "converged" and out["iters"] <= 15
        np.testing.assert_allclose(out["x"], dense.min_norm_solution(A.toarray(), b), rtol=0, atol=1e-8)


def test_repeated_row_skipped_and_history_reset():
    A, b = _system(2, m=10, n=30)
    rows = [0, 1, 0, 2, 1, 3]
    out = kz.kz_solve(A, b, rows, maxit=6, keep=True)
    assert out["skipped"] == 2 and len(out["P"]) == 4
    # a history cap of 1 keeps every step a classical-Kaczmarz-like step from the current x
    rows = np.random.default_rng(3).permutation(10)
    capped = kz.kz_solve(A, b, np.concatenate([rows, rows, rows]), maxit=30, kmax=1)
    x = np.zeros(30)
    for i in np.concatenate([rows, rows, rows])[:30]:
        x = kz.classical_kaczmarz_step(A, b, x, int(i))
    np.testing.assert_allclose(capped["x"], x, rtol=0, atol=1e-10 * np.linalg.norm(x))


def test_identity_matrix_and_zero_rhs():
    A = sp.identity(6, format="csr")
    b = np.arange(1.0, 7.0)
    out = kz.kz_solve(A, b, np.arange(6)[::-1], maxit=6, tol=1e-14)
    np.testing.assert_array_equal(out["x"], b)
    out = kz.kz_solve(A, np.zeros(6), np.arange(6), maxit=6)
    assert out["iters"] == 0 and out["outcome"] == "converged"
