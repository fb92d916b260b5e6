"""GPU parity of the growing-sketch engine (include/plss.h plss_eg_*) against
the oracle (oracle/engine.py: Thm 2.1 / Cor 2.2, and the QR variant of section 2.3 against a LAPACK
Householder QR of Y_k each step) for residual, identity and Gaussian sketch columns:
residual history within 1e-9 over the first 50 steps, final x within 1e-7, equal step counts,
outcomes and skips; the residual sketch also reproduces the PLSS oracle (Thm 4.1) and the identity
sketch the PLSS Kaczmarz GPU path.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import plss_gen
from oracle import engine

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
    kw.setdefault("maxit_cap", 600)
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
    assert int(res["diag"][1:res["iters"] + 1, 3].sum()) == ref["skipped"]


CASES = {
    "C1": (lambda: plss_gen.make_config("C1"), 40, None),
    "C2s": (lambda: plss_gen.make_config("C2s"), 120, None),
    "C2s_kmax32": (lambda: plss_gen.make_config("C2s"), 120, 32),
    "C4xs": (lambda: plss_gen.make_config("C4xs"), 100, None),
    "C3_32": (lambda: plss_gen.make_config("C3", N=32), 100, None),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("sketch", ["residual", "identity", "gaussian"])
@pytest.mark.parametrize("slabs", [1, 3])
@pytest.mark.parametrize("factor", ["triangular", "qr"])
def test_engine_parity(pkg, case, sketch, slabs, factor):
    make, steps, kmax = CASES[case]
    s = make()
    rows = np.resize(np.random.default_rng(7).permutation(s.m), steps)
    run = engine.tri_engine if factor == "triangular" else engine.qr_engine
    ref = run(s.scipy_csr(), s.b, sketch=sketch, maxit=steps, tol=1e-12, rows=rows, seed=5, kmax=kmax)
    ctx = _ctx(pkg, s, slabs=slabs)
    res = pkg.plss_eg_solve(ctx, torch.from_numpy(s.b).cuda(), sketch=sketch, kmax=kmax, rows=rows, seed=5,
                            maxit=steps, tol=1e-12, want_diag=True, factor=factor)
    pkg.plss_destroy(ctx)
    _compare(res, ref)


def test_qr_and_triangular_agree_on_gpu(pkg):
    s = plss_gen.make_config("C2s")
    ctx = _ctx(pkg, s)
    a = pkg.plss_eg_solve(ctx, s.b, sketch="gaussian", seed=9, maxit=80, tol=0.0, factor="triangular")
    q = pkg.plss_eg_solve(ctx, s.b, sketch="gaussian", seed=9, maxit=80, tol=0.0, factor="qr")
    pkg.plss_destroy(ctx)
    np.testing.assert_allclose(q["hist"], a["hist"], rtol=1e-9)


def test_residual_sketch_matches_plss_oracle(pkg):
    """Thm 4.1 on the GPU: the general engine with residual sketches vs the PLSS oracle."""
    s = plss_gen.make_config("C2s")
    ref = oracle.plss_system(s, maxit=60, tol=0.0)
    ctx = _ctx(pkg, s)
    res = pkg.plss_eg_solve(ctx, s.b, sketch="residual", maxit=60, tol=0.0)
    pkg.plss_destroy(ctx)
    k = 40
    np.testing.assert_allclose(res["hist"][:k], ref["hist"][:k], rtol=1e-8)


def test_identity_sketch_matches_kaczmarz_gpu(pkg):
    s = plss_gen.make_config("C2s")
    rows = np.random.default_rng(3).permutation(s.m)[:150]
    ctx = _ctx(pkg, s)
    a = pkg.plss_eg_solve(ctx, s.b, sketch="identity", rows=rows, maxit=150, tol=0.0)
    k = pkg.plss_kz_solve(ctx, s.b, rows, maxit=150, tol=0.0)
    pkg.plss_destroy(ctx)
    np.testing.assert_allclose(a["hist"], k["hist"], rtol=1e-8, atol=1e-15)
    xa, xk = a["x"].cpu().numpy(), k["x"].cpu().numpy()
    assert np.linalg.norm(xa - xk) <= 1e-8 * np.linalg.norm(xk)


def test_engine_errors_and_step_api(pkg):
    s = plss_gen.make_config("C2s")
    ctx = _ctx(pkg, s)
    with pytest.raises(pkg.PlssError):
        pkg.plss_eg_solve(ctx, s.b, sketch="identity", rows=None, maxit=3)
    with pytest.raises(pkg.PlssError):
        pkg.plss_eg_solve(ctx, s.b, sketch="identity", rows=np.array([s.m, 0, 1]), maxit=3)
    a = pkg.plss_eg_solve(ctx, s.b, sketch="gaussian", seed=2, maxit=50, tol=0.0)
    pkg.plss_eg_start(ctx, s.b, sketch="gaussian", seed=2, maxit=50, tol=0.0)
    pkg.plss_eg_step(ctx, 33)
    pkg.plss_eg_step(ctx, 17)
    c = pkg.plss_eg_finish(ctx, x=torch.empty(s.n, dtype=torch.float64, device="cuda"))
    pkg.plss_destroy(ctx)
    assert a["iters"] == c["iters"] == 50
    np.testing.assert_array_equal(a["x"].cpu().numpy(), c["x"].cpu().numpy())
