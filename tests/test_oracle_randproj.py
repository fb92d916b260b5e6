"""Pins of the randomized-projection oracle (oracle/randproj.py) against what the paper and the
mathematics fix, independent of the oracle's own route (pinv of the r x r Gram matrix):

* eq:itProb-eq:cons (B = I): p_k is the MINIMUM-NORM p with
  S_k^T A (x_{k-1} + p) = S_k^T b -- checked with LAPACK's SVD least squares (gelsd) on S_k^T A.
* p_k = P_k e_{k-1} with P_k the orthogonal projector onto range(A^T S_k), e = x* - x for a
  consistent system, so ||e_{k-1}||^2 = ||e_k||^2 + ||p_k||^2 and the error never grows.
* r = m (a square, almost surely invertible S): range(A^T S) = range(A^T), one step reaches the
  minimum-norm solution A^+ b from x0 = 0 -- and for m > n the Gram matrix S^T A A^T S is
  singular, so this exercises the pseudo-inverse branch (L166-167).
* The sampler (Box-Muller in binary32): ln_unit32 and sincos_2pi32 against libm, moments and
  Kolmogorov-Smirnov statistic of S against N(0, 1), independence of iterations / seeds, the
  sparse density.
"""
import math

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse as sp
import scipy.stats

from oracle import dense
from oracle import randproj as rp


def _system(seed=0, m=60, n=25, dens=0.3):
    rng = np.random.default_rng(seed)
    A = sp.random(m, n, density=dens, random_state=rng, data_rvs=rng.standard_normal).tocsr()
    A = A + sp.csr_matrix((np.ones(n), (rng.choice(m, n, replace=False), np.arange(n))), shape=(m, n))
    xs = rng.standard_normal(n)
    return A.tocsr(), xs, A @ xs


def test_sincos_2pi32_matches_libm():
    assert rp.PI4_32.view(np.uint32) == 0x3F490FDB
    u2 = np.concatenate([np.arange(0, 1 << 24, 997), np.arange(8) << 21, (np.arange(8) << 21) + 1,
                         (np.arange(1, 9) << 21) - 1]).astype(np.float32) * np.float32(2.0 ** -24)
    sn, cs = rp.sincos_2pi32(u2)
    assert sn.dtype == np.float32 and cs.dtype == np.float32
    th = 2 * np.pi * u2.astype(np.float64)
    assert np.max(np.abs(sn - np.sin(th))) <= 3e-7 and np.max(np.abs(cs - np.cos(th))) <= 3e-7
    assert np.max(np.abs(sn.astype(np.float64) ** 2 + cs.astype(np.float64) ** 2 - 1)) <= 1e-6


def test_ln_unit32_matches_libm_and_constants():
    assert rp.LN2_32.view(np.uint32) == 0x3F317218 and rp.SQRT_HALF_32.view(np.uint32) == 0x3F3504F3
    assert abs(float(rp.LN2_32) - math.log(2)) <= np.spacing(np.float32(0.69)) / 2
    rng = np.random.default_rng(1)
    s = np.concatenate([rng.random(20000).astype(np.float32), np.float32([2.0 ** -46, 0.5, 0.70710677,
                                                                         0.7071068, 1 - 2.0 ** -24])])
    s = s[s > 0]
    got = rp.ln_unit32(s)
    assert got.dtype == np.float32
    ref = np.array([math.log(float(v)) for v in s])
    ulps = np.abs(got.astype(np.float64) - ref) / np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert ulps.max() <= 3


def test_sketch_entries_are_binary32():
    S = rp.sketch(4, 3, 3000, 7, density=0.5)
    np.testing.assert_array_equal(S.astype(np.float32).astype(np.float64), S)


def test_sketch_is_standard_normal():
    S = rp.sketch(seed=7, k=1, m=100_000, r=3)
    z = S.ravel()
    assert abs(z.mean()) < 5 / math.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0 / z.size)
    assert abs(scipy.stats.kurtosis(z)) < 0.05
    assert scipy.stats.kstest(z, "norm").pvalue > 1e-3
    # columns from the two halves of a pair and from different pairs are uncorrelated
    c = np.corrcoef(S.T)
    assert np.max(np.abs(c - np.eye(3))) < 5 / math.sqrt(S.shape[0])


def test_sketch_fresh_per_iteration_and_seed():
    a = rp.sketch(1, 1, 5000, 4)
    b = rp.sketch(1, 2, 5000, 4)
    c = rp.sketch(2, 1, 5000, 4)
    np.testing.assert_array_equal(a, rp.sketch(1, 1, 5000, 4))      # deterministic
    for u in (b, c):
        assert abs(np.corrcoef(a.ravel(), u.ravel())[0, 1]) < 5 / math.sqrt(a.size)
    # a row's entries depend only on (seed, k, i, r): any m gives the same leading rows
    np.testing.assert_array_equal(rp.sketch(1, 1, 100, 4), a[:100])


def test_sketch_sparse_density():
    S = rp.sketch(3, 1, 200_000, 5, density=0.01)
    frac = np.count_nonzero(S) / S.size
    assert abs(frac - 0.01) < 5 * math.sqrt(0.01 * 0.99 / S.size)
    nz = S[S != 0]
    assert scipy.stats.kstest(nz, "norm").pvalue > 1e-3
    dense_S = rp.sketch(3, 1, 200_000, 5)
    np.testing.assert_array_equal(S[S != 0], dense_S[S != 0])        # the mask only zeroes


def test_update_is_min_norm_sketched_solution():
    A, xs, b = _system()
    out = rp.randproj(A, b, r=6, seed=5, maxit=8, keep=True)
    Ad = A.toarray()
    x = np.zeros(A.shape[1])
    for S, p in zip(out["S"], out["P"]):
        C = S.T @ Ad
        ref, *_ = scipy.linalg.lstsq(C, S.T @ (b - Ad @ x), lapack_driver="gelsd")
        np.testing.assert_allclose(p, ref, rtol=0, atol=1e-10 * np.linalg.norm(ref))
        np.testing.assert_allclose(C @ (x + p), S.T @ b, rtol=0, atol=1e-9 * np.linalg.norm(S.T @ b))
        x = x + p


def test_error_pythagoras_and_monotone():
    A, xs, b = _system(seed=1, m=80, n=30)
    out = rp.randproj(A, b, r=4, seed=9, maxit=40, keep=True)
    x = np.zeros(A.shape[1])
    e_prev = np.linalg.norm(xs - x)
    for p in out["P"]:
        x = x + p
        e = np.linalg.norm(xs - x)
        assert abs(e_prev ** 2 - (e ** 2 + p @ p)) <= 1e-10 * e_prev ** 2
        assert e <= e_prev * (1 + 1e-12)
        e_prev = e
    assert e_prev < 0.5 * np.linalg.norm(xs)       # it does converge, slowly (rate rho < 1)
    np.testing.assert_allclose(out["x"], x, rtol=0, atol=1e-12 * np.linalg.norm(x))


def test_full_sketch_one_step_pinv_branch():
    A, xs, b = _system(seed=2, m=30, n=12)
    out = rp.randproj(A, b, r=A.shape[0], seed=3, maxit=1)
    assert out["rank"][0] == A.shape[1] < A.shape[0]                 # S^T A A^T S singular
    np.testing.assert_allclose(out["x"], dense.min_norm_solution(A.toarray(), b), rtol=0, atol=1e-10)
    assert out["hist"][1] <= 1e-12


def test_underdetermined_converges_to_min_norm():
    rng = np.random.default_rng(4)
    A = sp.random(20, 50, density=0.4, random_state=rng, data_rvs=rng.standard_normal).tocsr()
    b = A @ rng.standard_normal(50)
    out = rp.randproj(A, b, r=8, seed=1, maxit=400, tol=1e-12)
    assert out["outcome"] == "converged"
    np.testing.assert_allclose(out["x"], dense.min_norm_solution(A.toarray(), b), rtol=0, atol=1e-9)


def test_stop_test_and_zero_rhs():
    A, xs, b = _system()
    out = rp.randproj(A, np.zeros(A.shape[0]), r=3, seed=1, maxit=5)
    assert out["iters"] == 0 and out["outcome"] == "converged" and not out["x"].any()
    out = rp.randproj(A, b, r=5, seed=1, maxit=5)
    assert out["iters"] == 5 and out["outcome"] == "maxit" and out["hist"].size == 6
    out2 = rp.randproj(A, b, r=5, seed=1, maxit=50, tol=out["hist"][3] * (1 + 1e-12))
    assert out2["outcome"] == "converged" and out2["iters"] <= 3
