"""Pins of the triangular growing-sketch engine oracle (oracle/engine.py; Thm 2.1,
Cor 2.2) by routes independent of its recursion:

* R_k D_k R_k^T equals inv(Y_k^T Y_k) (Thm 2.1, eq:rdrt-decomposition-of-the-inverse);
* the iterates equal eq:pkLong (L151-167) with the same growing sketch S_k through a dense
  pseudo-inverse, for residual, identity and Gaussian sketch columns;
* residual sketches reproduce the PLSS oracle's iterates (Thm 4.1: the short recursion and the
  general update coincide); identity sketches reproduce the PLSS Kaczmarz oracle (section 7);
* orthogonal updates (section 2.5); a repeated identity column is skipped (reading R22).
"""
import numpy as np
import scipy.sparse as sp

import oracle
from oracle import engine
from oracle import kaczmarz as okz

import plss_gen


def _system(seed=0, m=30, n=20, dens=0.3):
    rng = np.random.default_rng(seed)
    A = sp.random(m, n, density=dens, random_state=rng, data_rvs=rng.standard_normal).tocsr()
    A = (A + sp.csr_matrix((np.ones(n), (rng.choice(m, n, replace=n > m), np.arange(n))), shape=(m, n))).tocsr()
    b = A @ rng.standard_normal(n)
    return A, b


def test_rdrt_equals_inverse_gram():
    rng = np.random.default_rng(0)
    Y = [rng.standard_normal(12) for _ in range(7)]
    N = engine.rdrt_inverse(Y)
    Yk = np.stack(Y, axis=1)
    np.testing.assert_allclose(N, np.linalg.inv(Yk.T @ Yk), rtol=1e-10, atol=1e-12)


def _pk_long_sketch(A, b, kind, K, rows=None, seed=0):
    Ad = A.toarray()
    m, n = Ad.shape
    x = np.zeros(n)
    cols, xs = [], []
    for k in range(1, K + 1):
        r = b - Ad @ x
        cols.append(engine.sketch_column(kind, k, m, r, rows, seed))
        S = np.stack(cols, axis=1)
        Y = Ad.T @ S
        x = x + Y @ (np.linalg.pinv(Y.T @ Y) @ (S.T @ r))
        xs.append(x.copy())
    return xs


def test_equals_pk_long_all_sketches():
    for kind in ("residual", "identity", "gaussian"):
        for seed in range(3):
            A, b = _system(seed)
            rows = np.random.default_rng(seed).permutation(A.shape[0])
            K = 8
            ref = _pk_long_sketch(A, b, kind, K, rows, seed)
            out = engine.tri_engine(A, b, sketch=kind, maxit=K, rows=rows, seed=seed, keep=True)
            assert out["skipped"] == 0
            x = np.zeros(A.shape[1])
            for p, xr in zip(out["P"], ref):
                x = x + p
                np.testing.assert_allclose(x, xr, rtol=0, atol=1e-8 * max(1.0, np.linalg.norm(xr)))


def test_qr_engine_equals_pk_long_and_triangular():
    for kind in ("residual", "identity", "gaussian"):
        A, b = _system(7)
        rows = np.random.default_rng(2).permutation(A.shape[0])
        K = 10
        ref = _pk_long_sketch(A, b, kind, K, rows, 3)
        q = engine.qr_engine(A, b, sketch=kind, maxit=K, rows=rows, seed=3, keep=True)
        t = engine.tri_engine(A, b, sketch=kind, maxit=K, rows=rows, seed=3)
        x = np.zeros(A.shape[1])
        for p, xr in zip(q["P"], ref):
            x = x + p
            np.testing.assert_allclose(x, xr, rtol=0, atol=1e-8 * max(1.0, np.linalg.norm(xr)))
        np.testing.assert_allclose(q["hist"], t["hist"], rtol=1e-8, atol=1e-15)


def test_residual_sketch_is_plss():
    s = plss_gen.make_config("C1")
    ref = oracle.plss_system(s, maxit=40, tol=0.0)
    out = engine.tri_engine(s.scipy_csr(), s.b, sketch="residual", maxit=40)
    k = 30
    np.testing.assert_allclose(out["hist"][:k], ref["hist"][:k], rtol=1e-8)


def test_identity_sketch_is_kaczmarz():
    A, b = _system(4, m=25, n=40)
    rows = np.random.default_rng(9).permutation(25)
    a = engine.tri_engine(A, b, sketch="identity", maxit=25, rows=rows)
    k = okz.kz_solve(A, b, rows, maxit=25)
    np.testing.assert_allclose(a["x"], k["x"], rtol=0, atol=1e-9 * np.linalg.norm(k["x"]))
    np.testing.assert_allclose(a["hist"], k["hist"], rtol=1e-7, atol=1e-14)


def test_orthogonal_updates_and_skip():
    A, b = _system(5, m=40, n=25)
    out = engine.tri_engine(A, b, sketch="gaussian", maxit=12, seed=4, keep=True)
    P = np.stack(out["P"], axis=1)
    G = P.T @ P
    nrm = np.sqrt(np.diag(G))
    assert np.max(np.abs(G - np.diag(np.diag(G))) / np.outer(nrm, nrm)) <= 1e-10
    rows = [0, 1, 0, 2]
    out = engine.tri_engine(A, b, sketch="identity", maxit=4, rows=rows)
    assert out["skipped"] == 1
