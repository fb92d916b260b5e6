"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU needed).

Each test names the passage it checks. The oracle under test is oracle/plss_oracle.c (fp64,
Algorithm 1) and oracle/exact.py (rational Algorithm 1). The pins are
independent of both: a hand-derived worked example (tests/golden), the closed-form update
eq:pkLong (L151-167) with the residual sketch eq:S (L611-626), Craig's method (Thm 6.1,
L858-929), the pseudo-inverse (Thm 3.1, Cor 3.3 L583-609), orthogonality
(eq:orthogonal-updates L457-460, eq:orthSr L221-229), psi = -rho (L671-672), special cases.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import dense, exact
import plss_gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _q(v):
    return Fraction(v[0], v[1])


def _run_dense(A, b, **kw):
    s = plss_gen.from_dense(A, b, keep_zeros=False)
    args = dict(tol=1e-14, tol_mode=0, maxit=max(1, 4 * min(s.m, s.n)))
    args.update(kw)
    return s, oracle.plss(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t,
                          s.b, **args)


# ---------------------------------------------------------------------------------------------
# worked example
# ---------------------------------------------------------------------------------------------

def _golden():
    with open(os.path.join(GOLDEN, "worked_diag21.json")) as f:
        return json.load(f)


def test_worked_example_exact_rational():
    g = _golden()
    out = exact.plss_exact(g["A"], g["b"])
    assert out["converged"] and out["iters"] == g["iters"]
    assert out["rho"][0] == _q(g["rho0"]) and out["rho"][1] == _q(g["rho1"]) and out["rho"][2] == 0
    assert out["y"][0] == [_q(v) for v in g["y1"]]
    assert out["phi"][0] == _q(g["phi1"])
    assert out["p"][0] == [_q(v) for v in g["p1"]]
    assert out["theta"][0] == _q(g["theta1"])
    assert out["r"][1] == [_q(v) for v in g["r1"]]
    assert out["beta"][0] == _q(g["beta1"]) and out["gamma"][0] == _q(g["gamma1"])
    assert out["psi"][0] == _q(g["psi2"])
    assert out["p"][1] == [_q(v) for v in g["p2"]]
    assert out["x"] == [_q(v) for v in g["x2"]]


def test_worked_example_fp64_oracle():
    g = _golden()
    s, out = _run_dense(np.array(g["A"], float), np.array(g["b"], float), tol=1e-14,
                        keep_updates=True)
    assert out["outcome"] == "converged" and out["iters"] == g["iters"]
    np.testing.assert_allclose(out["x"], [float(_q(v)) for v in g["x2"]], atol=1e-14, rtol=0)
    np.testing.assert_allclose(out["P"][0], [float(_q(v)) for v in g["p1"]], atol=1e-14, rtol=0)
    np.testing.assert_allclose(out["P"][1], [float(_q(v)) for v in g["p2"]], atol=1e-14, rtol=0)
    rec = out["rec"]
    assert abs(rec[0, 1] - 5.0) <= 1e-14                      # rho0
    assert abs(rec[0, 2] - 17.0) <= 1e-14                     # phi1
    assert abs(rec[0, 4] - 25 / 17) <= 1e-14                  # theta1
    assert abs(rec[1, 6] - 9 / 25) <= 1e-14                   # beta
    assert abs(rec[1, 7] - 17 / 20) <= 1e-14                  # gamma (Alg. 1, not L639-643)
    assert abs(rec[1, 3] - (-180 / 289)) <= 1e-14             # psi2 = -rho1
    np.testing.assert_allclose(out["hist"], [float(_q(v)) for v in g["hist"]], atol=1e-14, rtol=0)
    assert abs(float(out["P"][0] @ out["P"][1])) <= 1e-14     # p2^T p1 = 0


# ---------------------------------------------------------------------------------------------
# exact finite termination (Thm 3.1, Cor 3.3)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("shape,seed", [((6, 4), 1), ((4, 6), 2), ((7, 7), 3), ((9, 5), 4),
                                        ((5, 9), 5), ((3, 3), 6)])
def test_exact_terminates_in_rank_steps(shape, seed):
    rng = np.random.default_rng(seed)
    m, n = shape
    A = rng.integers(-4, 5, size=shape).tolist()
    xs = rng.integers(-3, 4, size=n).tolist()
    b = exact.matvec([[Fraction(a) for a in row] for row in A], [Fraction(v) for v in xs])
    rk = exact.rank_exact(A)
    out = exact.plss_exact(A, b)
    assert out["converged"]
    assert out["iters"] <= rk
    # generic b: termination in exactly rank(A) steps (Krylov dimension)
    assert out["iters"] == rk
    # orthogonal updates and residuals, exactly (eq:orthogonal-updates, eq:orthSr)
    P, R = out["p"], out["r"]
    for i in range(len(P)):
        for j in range(i):
            assert exact.dotq(P[i], P[j]) == 0
    for i in range(len(R)):
        for j in range(i):
            assert exact.dotq(R[i], R[j]) == 0
    # psi_k = y_k^T p_{k-1} = -rho_{k-1}
    for k, psi in enumerate(out["psi"]):
        assert psi == -out["rho"][k + 1]
    # x = A^+ b: A x = b and x in range(A^T) (min-norm, Cor 3.3)
    Aq = [[Fraction(a) for a in row] for row in A]
    assert exact.matvec(Aq, out["x"]) == b
    At = [list(col) for col in zip(*A)]
    aug = [row + [xv] for row, xv in zip(At, out["x"])]
    assert exact.rank_exact(aug) == rk


def test_exact_rank_one():
    A = [[1, 2], [2, 4]]
    b = [3, 6]
    out = exact.plss_exact(A, b)
    assert out["converged"] and out["iters"] == 1
    assert out["x"] == [Fraction(3, 5), Fraction(6, 5)]     # A^+ b for the rank-1 matrix


# ---------------------------------------------------------------------------------------------
# fp64 oracle vs the exact oracle on the same (exactly representable) inputs
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("shape,seed", [((8, 5), 10), ((5, 8), 11), ((12, 8), 12), ((8, 12), 13)])
def test_fp64_tracks_exact(shape, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal(shape)
    xs = rng.standard_normal(shape[1])
    # consistent b in exact arithmetic; the fp64 oracle gets its nearest doubles
    bq = exact.matvec([[Fraction(a) for a in row] for row in A.tolist()],
                      [Fraction(v) for v in xs.tolist()])
    b = np.array([float(v) for v in bq])
    ex = exact.plss_exact(A.tolist(), bq)
    assert ex["converged"] and ex["iters"] == min(shape)
    nb = float(np.sqrt(float(ex["rho"][0])))
    s, out = _run_dense(A, b, tol=1e-12, maxit=min(shape) + 3)
    # finite termination within rank(A) steps in fp64 for min(m,n) <= 16
    assert out["outcome"] == "converged" and out["iters"] <= min(shape)
    h_exact = [float(np.sqrt(float(r))) / nb for r in ex["rho"]]
    k = min(len(h_exact), len(out["hist"])) - 1
    np.testing.assert_allclose(out["hist"][:k], h_exact[:k], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(out["x"], [float(v) for v in ex["x"]], rtol=1e-9, atol=1e-10)


# ---------------------------------------------------------------------------------------------
# closed form eq:pkLong with the residual sketch (Thm 4.1) and Craig (Thm 6.1)
# ---------------------------------------------------------------------------------------------

def _systems(count=50):
    rng = np.random.default_rng(1234)
    shapes = [(30, 20), (20, 30), (12, 8)]
    for t in range(count):
        m, n = shapes[t % 3]
        A = rng.standard_normal((m, n))
        yield A, A @ rng.standard_normal(n)


def test_recursion_equals_closed_form_pkLong():
    worst = 0.0
    for A, b in _systems():
        s, out = _run_dense(A, b, tol=0.0, maxit=8, keep_updates=True)
        ps, xs = dense.pk_long_iterates(A, b, 8)
        for k in range(8):
            worst = max(worst, np.linalg.norm(np.sum(out["P"][:k + 1], axis=0) - xs[k]) /
                        np.linalg.norm(xs[k]))
            worst = max(worst, np.linalg.norm(out["P"][k] - ps[k]) / np.linalg.norm(ps[k]))
    assert worst <= 1e-8, worst


def test_recursion_equals_craig():
    worst = 0.0
    for A, b in _systems():
        s, out = _run_dense(A, b, tol=0.0, maxit=8, keep_updates=True)
        ups = dense.craig_updates(A, b, 8)
        for k in range(len(ups)):
            worst = max(worst, np.linalg.norm(out["P"][k] - ups[k]) / np.linalg.norm(ups[k]))
    assert worst <= 1e-8, worst


def test_printed_theorem_gamma_is_off_by_rho():
    """Reading R1: the printed gamma of Thm 4.1 (L639-643) equals theta/(theta*phi - rho^2), a factor
    rho short of Algorithm 1's gamma = (theta/rho) beta = theta*rho/(theta*phi - rho^2)."""
    g = _golden()
    rho, theta, phi = _q(g["rho1"]), _q(g["theta1"]), Fraction(288, 289)
    alg1 = (theta / rho) * (rho * rho / (theta * phi - rho * rho))
    printed = 1 / (phi * (1 - rho * rho / (theta * phi)))   # ||y||^2 (1 - r^2/(p y))(1 + ...)
    assert alg1 == _q(g["gamma1"])
    assert printed * rho == alg1


# ---------------------------------------------------------------------------------------------
# minimum-norm limit vs the pseudo-inverse (Thm 3.1, Cor 3.3)
# ---------------------------------------------------------------------------------------------

def test_min_norm_underdetermined_pinv():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((20, 35))
    b = A @ rng.standard_normal(35)
    s, out = _run_dense(A, b, tol=1e-12, maxit=100)
    assert out["outcome"] == "converged" and out["iters"] <= 20 + 3   # fp64 overshoot <= 3
    xp = dense.min_norm_solution(A, b)
    assert np.linalg.norm(out["x"] - xp) / np.linalg.norm(xp) <= 1e-10


def test_c1_converges_to_pinv():
    s = plss_gen.make_config("C1")
    out = oracle.plss_system(s)
    assert out["outcome"] == "converged"
    assert out["iters"] <= 100                                # BASELINE C1: <= 100 iterations
    A = np.zeros((s.m, s.n))
    A[np.repeat(np.arange(s.m), np.diff(s.row_ptr)), s.col_idx] = s.val
    xp = dense.min_norm_solution(A, s.b)
    assert np.linalg.norm(out["x"] - xp) / np.linalg.norm(xp) <= 1e-9
    # psi = -rho identity while orthogonality holds
    rec = out["rec"]
    for k in range(1, 20):
        assert abs(rec[k, 3] / rec[k, 1] + 1) <= 1e-12


# ---------------------------------------------------------------------------------------------
# special cases (Krylov dimension = number of distinct |a_ii| on supp(b))
# ---------------------------------------------------------------------------------------------

def test_identity_one_step():
    b = np.array([1.0, -2.0, 0.5, 3.0])
    s, out = _run_dense(np.eye(4), b, tol=1e-15)
    assert out["iters"] == 1 and out["outcome"] == "converged"
    np.testing.assert_array_equal(out["x"], b)


def test_scaled_identity_one_step():
    b = np.array([2.0, 4.0, -6.0, 8.0])
    s, out = _run_dense(2 * np.eye(4), b, tol=1e-15)
    assert out["iters"] == 1
    np.testing.assert_allclose(out["x"], b / 2, rtol=0, atol=1e-15)


def test_diagonal_distinct_values_steps():
    d = np.array([1.0, 1.0, 2.0, 2.0, 3.0, -3.0, 5.0])
    A = np.diag(d)
    s, out = _run_dense(A, A @ np.ones(7), tol=1e-12)
    assert out["outcome"] == "converged" and out["iters"] == 4   # |a_ii| in {1, 2, 3, 5}
    np.testing.assert_allclose(out["x"], np.ones(7), rtol=0, atol=1e-12)


def test_zero_rhs_and_exact_start():
    A = np.array([[2.0, 1.0], [1.0, 3.0], [0.0, 1.0]])
    s, out = _run_dense(A, np.zeros(3))
    assert out["iters"] == 0 and out["outcome"] == "converged"
    xs = np.array([1.0, -1.0])
    b = A @ xs
    s = plss_gen.from_dense(A, b)
    out = oracle.plss(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t, s.b,
                      x0=xs, tol=1e-14, maxit=10)
    assert out["iters"] == 0 and out["outcome"] == "converged"
    np.testing.assert_array_equal(out["x"], xs)


def test_y_vanished_for_b_orthogonal_to_range():
    A = np.array([[1.0], [0.0]])
    s = plss_gen.from_dense(A, np.array([0.0, 1.0]), keep_zeros=True)
    out = oracle.plss(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t, s.b,
                      tol=1e-12, maxit=10)
    assert out["outcome"] == "y_vanished" and out["iters"] == 0


# ---------------------------------------------------------------------------------------------
# orthogonality windows and Pythagoras ||x_k - x0||^2 = sum theta_i
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(8, 5), (5, 8)])
def test_update_orthogonality_small(shape):
    rng = np.random.default_rng(99)
    worst = 0.0
    for _ in range(30):
        A = rng.standard_normal(shape)
        b = A @ rng.standard_normal(shape[1])
        s, out = _run_dense(A, b, tol=1e-10, keep_updates=True)
        assert out["iters"] <= min(shape)      # 100% of seeds at tol 1e-10
        P = out["P"]
        nrm = np.linalg.norm(P, axis=1)
        C = np.abs(P @ P.T) / np.outer(nrm, nrm)
        np.fill_diagonal(C, 0)
        worst = max(worst, C.max())
        theta = out["rec"][:out["iters"], 4]
        assert abs(np.sum(theta) - out["x"] @ out["x"]) <= 1e-10 * (out["x"] @ out["x"])
    assert worst <= 1e-10, worst


def test_c1_first_20_updates_orthogonal():
    s = plss_gen.make_config("C1")
    out = oracle.plss_system(s, keep_updates=True)
    P = out["P"][:20]
    nrm = np.linalg.norm(P, axis=1)
    C = np.abs(P @ P.T) / np.outer(nrm, nrm)
    np.fill_diagonal(C, 0)
    assert C.max() <= 1e-10


# ---------------------------------------------------------------------------------------------
# spmv / spmvT
# ---------------------------------------------------------------------------------------------

def _ragged(seed=5, m=300, n=200):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) * (rng.random((m, n)) < 0.05)
    A[3, :] = rng.standard_normal(n)  # one (nearly) dense row
    A[::7] = 0.0            # empty rows
    A[:, ::11] = 0.0        # empty columns
    return A


def test_spmv_matches_dense_and_adjoint():
    A = _ragged()
    s = plss_gen.from_dense(A, np.zeros(A.shape[0]))
    rng = np.random.default_rng(6)
    x = rng.standard_normal(s.n)
    u = rng.standard_normal(s.m)
    y = oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)
    v = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
    ref_y, ref_v = A @ x, A.T @ u
    assert np.max(np.abs(y - ref_y)) <= 1e-14 * np.max(np.abs(A) @ np.abs(x))
    assert np.max(np.abs(v - ref_v)) <= 1e-14 * np.max(np.abs(A.T) @ np.abs(u))
    assert abs(u @ y - v @ x) <= 1e-12 * abs(u @ y)
    # empty rows/cols give exact zeros
    assert np.all(y[::7] == 0.0) and np.all(v[::11] == 0.0)


# ---------------------------------------------------------------------------------------------
# scaled configs: C3 solution is 1 (SPD, b = A 1); C4 min-norm keeps empty columns at 0
# ---------------------------------------------------------------------------------------------

def test_c3_scaled_converges_to_ones():
    s = plss_gen.make_config("C3", N=64)
    out = oracle.plss_system(s, maxit=5000)
    assert out["outcome"] == "converged"
    assert np.max(np.abs(out["x"] - 1.0)) <= 1e-6


def test_c4_scaled_empty_columns_stay_zero():
    s = plss_gen.make_config("C4s")
    out = oracle.plss_system(s, maxit=300, tol=1e-6)
    empty = np.diff(s.col_ptr) == 0
    assert empty.sum() > 0
    assert np.all(out["x"][empty] == 0.0)          # x_k in range(A^T) (Cor 3.3)
    h = out["hist"]
    assert h[-1] < h[0]


def test_freeze_mode_keeps_x_fixed():
    s = plss_gen.make_config("C5xs")
    out = oracle.plss_system(s, maxit=60)       # tol = 0: only the freeze threshold stops progress
    assert out["iters"] == 60 and out["outcome"] == "maxit"
    rec = out["rec"]
    frozen = np.nonzero(rec[:60, 0] <= oracle.FREEZE_H)[0]
    assert frozen.size > 0
    k = frozen[0]
    assert np.all(rec[k + 1:60, 6] == 0.0) and np.all(rec[k + 1:60, 7] == 0.0)
    assert np.all(rec[k + 1:60, 0] == rec[k + 1, 0])  # residual frozen


def test_parity_floor_row_permutation():
    """Two valid oracles differing only by a row permutation agree to ~1e-14 in the pre-asymptotic
    window: the floor the GPU parity tolerances are checked against."""
    s = plss_gen.make_config("C2s")
    base = oracle.plss_system(s, maxit=50, tol=0.0)
    perm = np.random.default_rng(3).permutation(s.m)
    A = s.scipy_csr()[perm]
    A.sort_indices()
    t = plss_gen._finish("perm", s.m, s.n, A.indptr, A.indices, A.data, None, 0.0, 0, 50,
                         b=s.b[perm])
    other = oracle.plss_system(t, maxit=50, tol=0.0)
    d = np.abs(base["hist"] - other["hist"]) / base["hist"]
    assert d.max() <= 1e-11


# ---------------------------------------------------------------------------------------------
# PLSS W (diagonal WI, PAPER.md L714-765 / Algorithm 1 with B^T B): NEXT-1
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("shape,seed", [((7, 4), 0), ((5, 8), 1), ((6, 6), 2), ((9, 5), 3)])
def test_plssw_exact_terminates_at_min_wi_norm_solution(shape, seed):
    """With WI = diag(w) > 0 the iteration is plain PLSS on A_W = A R_W^T (W = R_W^T R_W = WI^-1,
    L716-721): it terminates in rank(A) steps, the updates are WI-orthogonal, psi_k = -rho_{k-1}
    still holds (y^T p is invariant under the transformation), and from x0 = 0 the limit is the
    minimum WI-norm solution x = W A^T (A W A^T)^+ b."""
    rng = np.random.default_rng(seed + 100)
    m, n = shape
    A = rng.integers(-4, 5, size=shape).tolist()
    w = [Fraction(int(v)) for v in rng.integers(1, 10, size=n)]
    xs = rng.integers(-3, 4, size=n).tolist()
    Aq = [[Fraction(a) for a in row] for row in A]
    b = exact.matvec(Aq, [Fraction(v) for v in xs])
    rk = exact.rank_exact(A)
    out = exact.plss_exact(A, b, wi=w)
    assert out["converged"] and out["iters"] == rk
    P = out["p"]
    for i in range(len(P)):
        for j in range(i):
            assert sum((pi * wk * pj for pi, wk, pj in zip(P[i], w, P[j])), Fraction(0)) == 0
    for k, psi in enumerate(out["psi"]):
        assert psi == -out["rho"][k + 1]
    x = out["x"]
    assert exact.matvec(Aq, x) == b
    # x = W A^T z for some z: x ./ (1/w) = WI x lies in range(A^T)
    wx = [xi * wi for xi, wi in zip(x, w)]
    At = [list(col) for col in zip(*Aq)]
    assert exact.rank_exact([row + [v] for row, v in zip(At, wx)]) == rk


def test_plssw_unit_weights_are_plss_bitwise():
    for name in ("C1", "C2s"):
        s = plss_gen.make_config(name)
        a = oracle.plss_system(s)
        b = oracle.plss_system(s, wi=np.ones(s.n))
        np.testing.assert_array_equal(a["x"], b["x"])
        np.testing.assert_array_equal(a["rec"], b["rec"])


@pytest.mark.parametrize("shape,seed", [((12, 6), 4), ((8, 14), 5)])
def test_plssw_fp64_tracks_exact(shape, seed):
    rng = np.random.default_rng(seed)
    m, n = shape
    A = rng.integers(-4, 5, size=shape)
    w = rng.integers(1, 10, size=n)
    xs = rng.integers(-3, 4, size=n)
    b = A @ xs
    ex = exact.plss_exact(A.tolist(), [Fraction(int(v)) for v in b], wi=[Fraction(int(v)) for v in w])
    s = plss_gen.from_dense(A.astype(float), b.astype(float), tol=1e-13, maxit=min(m, n) + 4)
    fp = oracle.plss_system(s, wi=w.astype(float))
    assert fp["outcome"] == "converged"
    xe = np.array([float(v) for v in ex["x"]])
    assert np.linalg.norm(fp["x"] - xe) <= 1e-10 * np.linalg.norm(xe)
    for k in range(1, min(len(ex["rho"]), len(fp["hist"])) - 1):
        rho_e = float(ex["rho"][k])
        assert abs(fp["rec"][k, 1] - rho_e) <= 1e-9 * max(rho_e, float(ex["rho"][0]) * 1e-12)


def test_plssw_equals_plss_on_column_scaled_matrix():
    """The paper's derivation (eq:pkTransrec -> eq:pkShortW): PLSS W on A with WI = diag(c) is PLSS
    on A_W = A diag(c)^-1/2 with x = diag(c)^-1/2 x_W; the residuals, hence hist, coincide."""
    s = plss_gen.make_config("C2s")
    c = oracle.column_norms(s.n, s.col_ptr, s.val_t)
    d = 1.0 / np.sqrt(c)
    sw = plss_gen._finish("C2s-scaled", s.m, s.n, s.row_ptr, s.col_idx, s.val * d[s.col_idx], None,
                          s.tol, s.tol_mode, s.maxit, b=s.b)
    a = oracle.plss_system(s, wi=c, maxit=60)
    b = oracle.plss_system(sw, maxit=60)
    k = min(len(a["hist"]), len(b["hist"]), 40)
    np.testing.assert_allclose(a["hist"][:k], b["hist"][:k], rtol=1e-9, atol=0)
    xw = d * b["x"]
    assert np.linalg.norm(a["x"] - xw) <= 1e-8 * np.linalg.norm(xw)


def test_column_norms():
    s = plss_gen.make_config("C4xs")                 # has empty columns
    c = oracle.column_norms(s.n, s.col_ptr, s.val_t)
    dense_norms = np.sqrt(np.bincount(s.col_idx, weights=s.val ** 2, minlength=s.n))
    empty = np.diff(s.col_ptr) == 0
    assert empty.any() and np.all(c[empty] == 1.0)
    np.testing.assert_allclose(c[~empty], dense_norms[~empty], rtol=1e-14)


# ---------------------------------------------------------------------------------------------
# STAGNATION guard (tau - 1 <= 1e-14; tau >= 1 by Cauchy-Schwarz)
# ---------------------------------------------------------------------------------------------

def test_stagnation_exact_tau_one():
    """A = [1; 1], b = e_1 (inconsistent: b is not in range(A)). By hand: r0 = b, rho0 = 1,
    y1 = A^T r0 = 1, phi1 = 1, p1 = 1, theta1 = 1, x1 = 1; r1 = r0 - A p1 = (0, -1), rho1 = 1,
    y2 = -1, phi2 = 1, so tau = sqrt(theta1 phi2) / rho1 = 1 exactly: the exact-rational oracle's
    denominator theta phi - rho^2 is 0 at that step, and the fp64 oracle reports STAGNATION with
    one update applied (x = 1), the breakdown as an outcome, not an error."""
    A = np.array([[1.0], [1.0]])
    b = np.array([1.0, 0.0])
    ex = exact.plss_exact([[Fraction(1)], [Fraction(1)]], [Fraction(1), Fraction(0)], maxit=10)
    assert ex["iters"] == 1 and not ex["converged"]
    assert ex["theta"][0] * ex["phi"][-1] - ex["rho"][-1] ** 2 == 0
    s = plss_gen.from_dense(A, b, tol=1e-12, maxit=10)
    r = oracle.plss_system(s)
    assert r["outcome"] == "stagnation" and r["iters"] == 1
    assert r["x"].tolist() == [1.0]
    assert r["rec"][1, 0] == 1.0 and r["rec"][1, 1] == 1.0      # hist_1 = ||r1|| / ||b|| = 1
    # freeze mode: the guard freezes the iterate (beta = gamma = 0) and the outcome is kept
    f = oracle.plss_system(s, maxit=6, freeze=True, tol=0.0)
    assert f["outcome"] == "stagnation" and f["iters"] == 6 and f["x"].tolist() == [1.0]


def test_stagnation_does_not_fire_on_consistent_systems():
    """The guard must not fire before convergence on consistent systems (SURVEY 8c pin table,
    'breakdown guard safety'): min(tau - 1) over C1's run stays far from 1e-14."""
    s = plss_gen.make_config("C1")
    r = oracle.plss_system(s)
    tau = r["rec"][1:r["iters"], 5]
    assert r["outcome"] == "converged" and tau.min() - 1.0 > 0.1


# ---------------------------------------------------------------------------------------------
# threaded oracle (oracle_set_threads): bitwise element values, fixed-order blocked dots
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("T", [2, 3, 8])
def test_threaded_oracle_spmv_bitwise(T):
    s = plss_gen.make_config("C2s")
    rng = np.random.default_rng(7)
    x, u = rng.standard_normal(s.n), rng.standard_normal(s.m)
    y1 = oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)
    v1 = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
    with oracle.threads(T):
        y = oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)
        v = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
    np.testing.assert_array_equal(y, y1)
    np.testing.assert_array_equal(v, v1)


@pytest.mark.parametrize("name,T,weighted", [("C2s", 4, False), ("C5xs", 8, False), ("C1", 16, False),
                                             ("C2s", 3, True), ("C5xs", 8, True)])
def test_threaded_oracle_tracks_sequential(name, T, weighted):
    """Only the dot products' summation order differs: the histories agree to rounding while the
    process is pre-asymptotic, runs with a fixed T are bitwise repeatable, and T
    larger than a vector leaves empty blocks (C1: n = 100 < T * 8)."""
    s = plss_gen.make_config(name)
    wi = oracle.column_norms(s.n, s.col_ptr, s.val_t) if weighted else None   # PLSS W: the blocked wdot
    a = oracle.plss_system(s, maxit=30, wi=wi)
    with oracle.threads(T):
        b = oracle.plss_system(s, maxit=30, wi=wi)
        c = oracle.plss_system(s, maxit=30, wi=wi)
    np.testing.assert_array_equal(b["rec"], c["rec"])
    k = min(len(a["hist"]), len(b["hist"]), 25)
    assert np.max(np.abs(a["hist"][:k] - b["hist"][:k]) / a["hist"][:k]) <= 1e-12
    assert np.linalg.norm(a["x"] - b["x"]) <= 1e-10 * np.linalg.norm(a["x"])
    assert oracle._load().oracle_get_threads() == 1          # restored on exit
