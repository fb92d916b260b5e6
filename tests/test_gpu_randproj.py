"""GPU parity of randomized projection (include/plss.h plss_rp_*) against the
oracle (oracle/randproj.py), through the C ABI.

* The sketch S_k: bitwise (both sides implement the same counter-based generator from correctly
  rounded operations only, reading R17), dense and sparse, ragged row counts, r odd/even.
* Y = A^T S (plss_spmmT): bitwise the oracle's per-column sequential sums.
* Solves: hist within 1e-9 (relative) over the iterations, final x within 1e-7, equal iteration
  counts, outcomes and Gram ranks; the rank-deficient r > n case (pseudo-inverse branch, reading
  R18) reaches A^+ b in one step.
"""
import numpy as np
import pytest

import oracle
import plss_gen
from oracle import dense
from oracle import randproj as rp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_2207_07615_b200 import build as pbuild
    pbuild.build()
    import paper_2207_07615_b200 as p
    p.load_library()
    assert torch.cuda.is_available()
    return p


def _ctx(pkg, s, **kw):
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    kw.setdefault("maxit_cap", 400)
    return pkg.plss_create(A, **kw)


def _small(seed=0, m=1000, n=300, per_row=6):
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(m), per_row)
    cols = np.concatenate([rng.choice(n, per_row, replace=False) for _ in range(m)])
    import scipy.sparse as sp
    A = sp.csr_matrix((rng.standard_normal(m * per_row), (rows, cols)), shape=(m, n))
    A.sort_indices()
    xs = rng.standard_normal(n)
    return plss_gen._finish("rp-small", m, n, A.indptr, A.indices, A.data, xs, 1e-8, 0, 200)


@pytest.mark.parametrize("r", [1, 5, 10, 33, 64])
@pytest.mark.parametrize("density", [1.0, 0.1])
def test_sketch_bitwise(pkg, r, density):
    s = _small(m=10_007 if r <= 10 else 2_003)
    ctx = _ctx(pkg, s)
    for k, ld in ((1, None), (7, r + (r & 1))):
        S = pkg.plss_rp_sketch(ctx, r, seed=123, k=k, density=density, ld=ld).cpu().numpy()
        assert S.dtype == np.float32 and S.shape[1] >= r
        np.testing.assert_array_equal(S[:, :r].astype(np.float64), rp.sketch(123, k, s.m, r, density))
        assert not S[:, r:].any()
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("case", ["small", "C4xs", "C3_64"])
@pytest.mark.parametrize("r", [1, 3, 8, 17, 50])
def test_spmmT_bitwise(pkg, case, r):
    s = {"small": lambda: _small(1), "C4xs": lambda: plss_gen.make_config("C4xs"),
         "C3_64": lambda: plss_gen.make_config("C3", N=64)}[case]()
    ctx = _ctx(pkg, s)
    S = rp.sketch(5, 1, s.m, r)
    S32 = np.zeros((s.m, pkg.rp_ld(r)), dtype=np.float32)
    S32[:, :r] = S
    Y = pkg.plss_spmmT(ctx, torch.from_numpy(S32).cuda(), r=r).cpu().numpy()
    ref = np.stack([oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, np.ascontiguousarray(S[:, c]))
                    for c in range(r)], axis=1)
    np.testing.assert_array_equal(Y, ref)
    pkg.plss_destroy(ctx)


def _compare(res, ref, k_hist=None):
    assert res["iters"] == ref["iters"], (res["iters"], ref["iters"])
    assert res["outcome"] == ref["outcome"]
    h, hr = res["hist"], ref["hist"]
    k = len(hr) if k_hist is None else min(k_hist, len(hr))
    assert len(h) == len(hr)
    live = hr[:k] > 1e-13
    assert np.max(np.abs(h[:k] - hr[:k])[live] / hr[:k][live]) <= 1e-9
    x, xr = res["x"].cpu().numpy(), ref["x"]
    assert np.linalg.norm(x - xr) <= 1e-7 * np.linalg.norm(xr)
    ranks = res["diag"][1:res["iters"] + 1, 2]
    np.testing.assert_array_equal(ranks, ref["rank"])


CASES = {
    "C1_r10": (lambda: plss_gen.make_config("C1"), dict(r=10, maxit=60)),
    "small_r5_sparse": (lambda: _small(2), dict(r=5, maxit=80, density=0.2)),
    "C2s_r10": (lambda: plss_gen.make_config("C2s"), dict(r=10, maxit=25)),
    "C2s_r5_sparse": (lambda: plss_gen.make_config("C2s"), dict(r=5, maxit=25, density=0.02)),
    "C4xs_r5": (lambda: plss_gen.make_config("C4xs"), dict(r=5, maxit=25)),
    "C3_32_r40": (lambda: plss_gen.make_config("C3", N=32), dict(r=40, maxit=30)),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("slabs", [1, 3])
def test_rp_solve_parity(pkg, case, slabs):
    make, kw = CASES[case]
    s = make()
    ref = rp.randproj(s.scipy_csr(), s.b, r=kw["r"], seed=11, maxit=kw["maxit"], tol=1e-12,
                      density=kw.get("density", 1.0))
    ctx = _ctx(pkg, s, slabs=slabs)
    res = pkg.plss_rp_solve(ctx, torch.from_numpy(s.b).cuda(), r=kw["r"], seed=11, maxit=kw["maxit"], tol=1e-12,
                            density=kw.get("density", 1.0), want_diag=True)
    pkg.plss_destroy(ctx)
    _compare(res, ref)


def test_rp_converges_with_stop_test(pkg):
    s = _small(3, m=400, n=60)
    ref = rp.randproj(s.scipy_csr(), s.b, r=20, seed=2, maxit=300, tol=1e-8)
    assert ref["outcome"] == "converged"
    ctx = _ctx(pkg, s)
    res = pkg.plss_rp_solve(ctx, s.b, r=20, seed=2, maxit=300, tol=1e-8, want_diag=True)   # host b
    _compare(res, ref, k_hist=50)     # north_star's window: later hist values near 1e-8 carry the
                                      # fp64 floor of the recursive residual (~1e-16 ||b|| absolute)
    # the PLSS path still works on the same ctx afterwards (its state is re-initialised)
    out = pkg.plss_solve(ctx, s.b, tol=1e-8, maxit=300)
    assert out["outcome"] == "converged"
    pkg.plss_destroy(ctx)


def test_rp_rank_deficient_pinv_branch(pkg):
    """r > n: Y^T Y (r x r) has rank n; one step gives the minimum-norm solution (L166-167)."""
    s = _small(4, m=40, n=12, per_row=4)
    ctx = _ctx(pkg, s)
    res = pkg.plss_rp_solve(ctx, s.b, r=24, seed=3, maxit=1, tol=0.0, want_diag=True)
    pkg.plss_destroy(ctx)
    assert res["diag"][1, 2] == 12
    xmn = dense.min_norm_solution(s.scipy_csr().toarray(), s.b)
    np.testing.assert_allclose(res["x"].cpu().numpy(), xmn, rtol=0, atol=1e-9 * np.linalg.norm(xmn))


def test_rp_x0_and_zero_rhs(pkg):
    s = _small(5, m=300, n=80)
    ctx = _ctx(pkg, s)
    res = pkg.plss_rp_solve(ctx, np.zeros(s.m), r=4, seed=1, maxit=5)
    assert res["iters"] == 0 and res["outcome"] == "converged"
    x0 = np.random.default_rng(0).standard_normal(s.n)
    ref = rp.randproj(s.scipy_csr(), s.b, r=6, seed=9, maxit=15, x0=x0)
    res = pkg.plss_rp_solve(ctx, s.b, r=6, seed=9, maxit=15, x0=x0, tol=0.0, want_diag=True)
    pkg.plss_destroy(ctx)
    _compare(res, ref)


def test_rp_bad_arguments(pkg):
    s = _small(6, m=100, n=30)
    ctx = _ctx(pkg, s)
    for kw in (dict(r=0), dict(r=65), dict(r=4, density=0.0), dict(r=4, density=1.5)):
        with pytest.raises(pkg.PlssError):
            pkg.plss_rp_solve(ctx, s.b, maxit=3, **kw)
    with pytest.raises(pkg.PlssError):
        pkg.plss_rp_step(ctx, 1)                         # before plss_rp_start
    pkg.plss_destroy(ctx)


def test_rp_start_step_finish_matches_solve(pkg):
    s = plss_gen.make_config("C2s")
    ctx = _ctx(pkg, s)
    b = torch.from_numpy(s.b).cuda()
    a = pkg.plss_rp_solve(ctx, b, r=8, seed=4, maxit=37, tol=0.0)
    pkg.plss_rp_start(ctx, b, r=8, seed=4, maxit=37, tol=0.0)
    pkg.plss_rp_step(ctx, 20)
    pkg.plss_rp_step(ctx, 17)
    c = pkg.plss_rp_finish(ctx, x=torch.empty(s.n, dtype=torch.float64, device="cuda"))
    pkg.plss_destroy(ctx)
    assert a["iters"] == c["iters"] == 37 and c["outcome"] == "maxit"
    np.testing.assert_array_equal(a["x"].cpu().numpy(), c["x"].cpu().numpy())
    np.testing.assert_array_equal(a["hist"], c["hist"])
