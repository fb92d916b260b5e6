"""GPU: the paper's other methods (randomized projection, PLSS Kaczmarz, the growing-sketch engine)
on degenerate systems -- zero rows, zero columns, an all-zero matrix with b != 0 (inconsistent:
every step is skipped) -- give the oracles' iteration counts and outcomes, and the true residual
works on them."""
import numpy as np
import pytest
import scipy.sparse as sp

import plss_gen
from oracle import engine as oeg
from oracle import kaczmarz as okz
from oracle import randproj as orp

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


@pytest.mark.parametrize("m,n", [(0, 5), (5, 0), (0, 0), (3, 4)])
def test_degenerate_systems_all_methods(pkg, m, n):
    s = plss_gen._finish("degenerate", m, n, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), None,
                         1e-8, 0, 5, b=np.ones(m))
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    Asp = sp.csr_matrix((m, n))
    ctx = pkg.plss_create(A, maxit_cap=5)
    cases = [("rp", lambda: pkg.plss_rp_solve(ctx, s.b, r=2, seed=1, maxit=3),
              lambda: orp.randproj(Asp, s.b, r=2, seed=1, maxit=3)),
             ("eg-residual", lambda: pkg.plss_eg_solve(ctx, s.b, sketch="residual", maxit=3),
              lambda: oeg.tri_engine(Asp, s.b, sketch="residual", maxit=3)),
             ("eg-gaussian", lambda: pkg.plss_eg_solve(ctx, s.b, sketch="gaussian", seed=1, maxit=3),
              lambda: oeg.tri_engine(Asp, s.b, sketch="gaussian", maxit=3, seed=1))]
    if m > 0:
        rows = np.arange(min(m, 3))
        cases.append(("kz", lambda: pkg.plss_kz_solve(ctx, s.b, rows, maxit=3),
                      lambda: okz.kz_solve(Asp, s.b, rows, maxit=3)))
    else:
        with pytest.raises(pkg.PlssError):                   # no valid row index exists
            pkg.plss_kz_solve(ctx, s.b, np.zeros(1, np.int64), maxit=3)
    for name, gpu, ref in cases:
        g, r = gpu(), ref()
        assert (g["iters"], g["outcome"]) == (r["iters"], r["outcome"]), name
        assert g["x"].cpu().numpy().shape == (n,)
        assert not np.any(g["x"].cpu().numpy())                # nothing to add to x0 = 0
    t = pkg.plss_true_residual(ctx, s.b, np.zeros(n))
    assert t["abs"] == pytest.approx(np.sqrt(m)) and t["norm_b"] == pytest.approx(np.sqrt(m))
    pkg.plss_destroy(ctx)
