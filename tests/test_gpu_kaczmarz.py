"""GPU parity of PLSS Kaczmarz (include/plss.h plss_kz_*) against the oracle
(oracle/kaczmarz.py), through the C ABI: the worked diag(2,1) example exactly, residual history
within 1e-9 over the first 50 steps, final x within 1e-7, equal step counts, outcomes and skipped
rows; one-sweep termination at A^+ b; history reset (kmax); errors.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import plss_gen
from oracle import dense
from oracle import kaczmarz as okz

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "kaczmarz_diag21.json")


@pytest.fixture(scope="module")
def pkg():
    from paper_2207_07615_b200 import build as pbuild
    pbuild.build()
    import paper_2207_07615_b200 as p
    p.load_library()
    assert torch.cuda.is_available()
    return p


def _sys_from_csr(A, b, name="kz"):
    A = sp.csr_matrix(A)
    A.sort_indices()
    return plss_gen._finish(name, A.shape[0], A.shape[1], A.indptr, A.indices, A.data, None, 1e-8, 0, 100, b=b)


def _ctx(pkg, s, **kw):
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    kw.setdefault("maxit_cap", 1000)
    return pkg.plss_create(A, **kw)


def _compare(res, ref, k_hist=50):
    assert res["iters"] == ref["iters"], (res["iters"], ref["iters"])
    assert res["outcome"] == ref["outcome"]
    h, hr = res["hist"], ref["hist"]
    assert len(h) == len(hr)
    k = min(k_hist, len(hr))
    live = hr[:k] > 1e-13
    assert np.max(np.abs(h[:k] - hr[:k])[live] / hr[:k][live]) <= 1e-9
    x, xr = res["x"].cpu().numpy(), ref["x"]
    assert np.linalg.norm(x - xr) <= 1e-7 * max(np.linalg.norm(xr), 1e-300)
    assert int(res["diag"][1:res["iters"] + 1, 2].sum()) == ref["skipped"]


def test_worked_example_diag21(pkg):
    g = json.load(open(GOLDEN))
    s = _sys_from_csr(np.array(g["A"], float), np.array(g["b"], float))
    ctx = _ctx(pkg, s)
    res = pkg.plss_kz_solve(ctx, s.b, np.array(g["rows"]), maxit=2, tol=0.0, want_diag=True)
    pkg.plss_destroy(ctx)
    np.testing.assert_array_equal(res["x"].cpu().numpy(), g["x"])
    assert res["iters"] == 2 and res["outcome"] == "converged"


def _rand_sys(seed, m, n, dens):
    rng = np.random.default_rng(seed)
    A = sp.random(m, n, density=dens, random_state=rng, data_rvs=rng.standard_normal).tocsr()
    A = A + sp.csr_matrix((np.ones(m), (np.arange(m), rng.choice(n, m, replace=m > n))), shape=(m, n))
    return _sys_from_csr(A, A @ rng.standard_normal(n))


CASES = {
    "small_fullrowrank": (lambda: _rand_sys(0, 40, 90, 0.1), 40, None),
    "C2s": (lambda: plss_gen.make_config("C2s"), 300, None),
    "C2s_kmax64": (lambda: plss_gen.make_config("C2s"), 300, 64),
    "C4xs": (lambda: plss_gen.make_config("C4xs"), 300, None),
    "C3_32": (lambda: plss_gen.make_config("C3", N=32), 250, 100),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("slabs", [1, 3])
def test_kz_parity(pkg, case, slabs):
    make, steps, kmax = CASES[case]
    s = make()
    rows = np.random.default_rng(7).permutation(s.m)
    rows = np.concatenate([rows, rows])[:steps]
    ref = okz.kz_solve(s.scipy_csr(), s.b, rows, maxit=steps, tol=1e-12, kmax=kmax)
    ctx = _ctx(pkg, s, slabs=slabs)
    res = pkg.plss_kz_solve(ctx, torch.from_numpy(s.b).cuda(), torch.from_numpy(rows).cuda(), kmax=kmax,
                            maxit=steps, tol=1e-12, want_diag=True)
    pkg.plss_destroy(ctx)
    _compare(res, ref)


def test_one_sweep_min_norm(pkg):
    s = _rand_sys(3, 30, 70, 0.15)
    rows = np.random.default_rng(1).permutation(30)
    ctx = _ctx(pkg, s)
    res = pkg.plss_kz_solve(ctx, s.b, rows, maxit=30, tol=1e-10)
    pkg.plss_destroy(ctx)
    assert res["outcome"] == "converged" and res["iters"] <= 30
    xmn = dense.min_norm_solution(s.scipy_csr().toarray(), s.b)
    np.testing.assert_allclose(res["x"].cpu().numpy(), xmn, rtol=0, atol=1e-8 * np.linalg.norm(xmn))


def test_repeated_rows_skipped(pkg):
    s = _rand_sys(4, 20, 50, 0.2)
    rows = np.array([0, 1, 0, 2, 1, 3, 3, 4])
    ref = okz.kz_solve(s.scipy_csr(), s.b, rows, maxit=8)
    ctx = _ctx(pkg, s)
    res = pkg.plss_kz_solve(ctx, s.b, rows, maxit=8, tol=0.0, want_diag=True)
    pkg.plss_destroy(ctx)
    assert ref["skipped"] == 3
    _compare(res, ref)


def test_start_step_finish_and_errors(pkg):
    s = plss_gen.make_config("C2s")
    rows = np.random.default_rng(2).permutation(s.m)[:90]
    ctx = _ctx(pkg, s)
    a = pkg.plss_kz_solve(ctx, s.b, rows, maxit=90, tol=0.0)
    pkg.plss_kz_start(ctx, s.b, rows, maxit=90, tol=0.0)
    pkg.plss_kz_step(ctx, 50)
    pkg.plss_kz_step(ctx, 40)
    c = pkg.plss_kz_finish(ctx, x=torch.empty(s.n, dtype=torch.float64, device="cuda"))
    assert a["iters"] == c["iters"] == 90 and c["outcome"] == "maxit"
    np.testing.assert_array_equal(a["x"].cpu().numpy(), c["x"].cpu().numpy())
    np.testing.assert_array_equal(a["hist"], c["hist"])
    with pytest.raises(pkg.PlssError):
        pkg.plss_kz_solve(ctx, s.b, np.array([0, s.m]), maxit=2)        # row out of range
    with pytest.raises(pkg.PlssError):
        pkg.plss_kz_solve(ctx, s.b, rows, kmax=0, maxit=2)
    # the PLSS path still works on the ctx afterwards
    out = pkg.plss_solve(ctx, s.b, tol=1e-8, maxit=1000)
    assert out["outcome"] == "converged"
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("case", ["C2s", "C3_32"])
def test_fused_residual_bitwise(pkg, case):
    """Short rows (<= 32 entries): k_kz_resid computes (A p)_l itself instead of the separate plain
    SpMV -- the same sequential ascending sum, so the run is bitwise the unfused one."""
    s = plss_gen.make_config("C3", N=32) if case == "C3_32" else plss_gen.make_config(case)
    rows = np.random.default_rng(4).permutation(s.m)[:120]
    out = []
    for fuse in ("1", "0"):
        old = os.environ.get("PLSS_KZ_FUSE")
        os.environ["PLSS_KZ_FUSE"] = fuse
        try:
            ctx = _ctx(pkg, s, slabs=2)
            r = pkg.plss_kz_solve(ctx, s.b, rows, maxit=120, tol=0.0)
            pkg.plss_destroy(ctx)
        finally:
            if old is None:
                os.environ.pop("PLSS_KZ_FUSE")
            else:
                os.environ["PLSS_KZ_FUSE"] = old
        out.append(r)
    np.testing.assert_array_equal(out[0]["x"].cpu().numpy(), out[1]["x"].cpu().numpy())
    np.testing.assert_array_equal(out[0]["hist"], out[1]["hist"])
