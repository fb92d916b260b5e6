"""GPU: the SELL-32 kernel formats: fmt 1 (grid-stride slices), fmt 3
(one CTA per SM over contiguous slice ranges, the K1 default) and fmt 2 (shared-memory windows of
the gathered vector, k_sellw; opt-in through PLSS_WIN1 / PLSS_WIN2).

A format changes WHERE an entry's g value is read (ring in shared memory, L1, L2) and which warp
sums a row, never the summation order, so every SpMV output must be bitwise the oracle's
sequential sum, for any window size, alignment of g, or window jump pattern.
"""
import os

import numpy as np
import pytest

import oracle
import plss_gen

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


def _matrix(pkg, s):
    return pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)


class _env:
    """Set window-size overrides (read by plss_create) for the duration of a block."""

    def __init__(self, **kw):
        self.kw = {k: str(v) for k, v in kw.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kw}
        os.environ.update(self.kw)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _spmv_pair(pkg, ctx, s, x, u, offset=0):
    """y = A x and v = A^T u through the C ABI; offset > 0 places x and u at an 8-byte phase."""
    xb = torch.zeros(s.n + 2, dtype=torch.float64, device="cuda")
    ub = torch.zeros(s.m + 2, dtype=torch.float64, device="cuda")
    xb[offset:offset + s.n] = torch.from_numpy(x).cuda()
    ub[offset:offset + s.m] = torch.from_numpy(u).cuda()
    y = torch.empty(s.m, dtype=torch.float64, device="cuda")
    v = torch.empty(s.n, dtype=torch.float64, device="cuda")
    pkg.plss_spmv(ctx, xb[offset:offset + s.n], y)
    pkg.plss_spmvT(ctx, ub[offset:offset + s.m], v)
    return y.cpu().numpy(), v.cpu().numpy()


def _banded_blocks_permuted(seed=0, m=40_000, n=10_000, half=300, block=512):
    """Banded rows (plus 2 random columns per row) whose 512-row blocks are shuffled: the best
    window jumps from block to block (reset blocks) and some blocks move backwards (clamps)."""
    s = plss_gen.c5_banded(seed=seed, m=m, n=n, band=5, unif=2, half=half, maxit=20)
    rng = np.random.default_rng(seed + 1)
    nb = (m + block - 1) // block
    order = rng.permutation(nb)
    perm = np.concatenate([np.arange(b * block, min(m, (b + 1) * block)) for b in order])
    A = s.scipy_csr()[perm]
    A.sort_indices()
    return plss_gen._finish("banded-perm", m, n, A.indptr, A.indices, A.data, None, 1e-8, 0, 20,
                            b=s.b[perm], freeze=True)


CASES = {
    "C5xs": lambda: plss_gen.make_config("C5xs"),
    "C3_128": lambda: plss_gen.make_config("C3", N=128),
    "banded_perm": _banded_blocks_permuted,
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("win", [(4096, 16384), (256, 512), (1024, 2048)])
@pytest.mark.parametrize("slabs", [1, 3])
def test_window_spmv_bit_exact(pkg, case, win, slabs):
    s = CASES[case]()
    x = np.random.default_rng(2).standard_normal(s.n)
    u = np.random.default_rng(3).standard_normal(s.m)
    ref_y = oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)
    ref_v = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
    with _env(PLSS_WIN1=win[0], PLSS_WIN2=win[1]):
        ctx = pkg.plss_create(_matrix(pkg, s), slabs=slabs, maxit_cap=4, validate=True)
    q = pkg.plss_query(ctx)
    assert q["window_segments"] >= 1, q           # every case here has band locality
    for offset in (0, 1):
        y, v = _spmv_pair(pkg, ctx, s, x, u, offset)
        np.testing.assert_array_equal(y, ref_y)
        np.testing.assert_array_equal(v, ref_v)
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("case", ["C5xs", "banded_perm"])
def test_window_solve_matches_unwindowed_and_is_deterministic(pkg, case):
    """SpMV outputs are bitwise equal with and without windows (above); the dot products use a
    different (fixed) reduction shape, so solves agree to rounding, and two windowed runs agree
    bitwise even though slices are taken in a run-dependent order."""
    s = CASES[case]()
    out = []
    for window in (True, True, False):
        with _env(PLSS_WIN1=4096, PLSS_WIN2=16384):
            ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=s.maxit, window=window)
        q = pkg.plss_query(ctx)
        assert (q["window_segments"] >= 1) == window
        res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, maxit=s.maxit,
                             flags=1 if s.freeze else 0, want_hist=True)
        out.append((res["x"].cpu().numpy(), res["hist"], res["iters"]))
        pkg.plss_destroy(ctx)
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[2][2]
    k = 25
    h0, h2 = out[0][1][:k], out[2][1][:k]
    live = h2 > 1e-12                          # before the recursion reaches rounding level
    assert live.sum() >= 5 and np.max(np.abs(h0 - h2)[live] / h2[live]) <= 1e-11
    assert np.linalg.norm(out[0][0] - out[2][0]) <= 1e-10 * np.linalg.norm(out[2][0])


def test_no_window_without_locality(pkg):
    s = plss_gen.make_config("C2")           # uniform random columns over 100k: no window pays off
    with _env(PLSS_WIN1=4096, PLSS_WIN2=16384):
        ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=4)
    assert pkg.plss_query(ctx)["window_segments"] == 0
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("case", ["C5xs", "C3_128", "banded_perm", "ragged_c4"])
@pytest.mark.parametrize("sellc", [0, 1, 2])
@pytest.mark.parametrize("slabs", [1, 4])
def test_formats_spmv_bit_exact(pkg, case, sellc, slabs):
    """fmt 1 / fmt 3 for K1 and K2 segments (PLSS_SELLC 0: none, 1: K1, 2: both)."""
    s = plss_gen.make_config("C4xs") if case == "ragged_c4" else CASES[case]()
    x = np.random.default_rng(2).standard_normal(s.n)
    u = np.random.default_rng(3).standard_normal(s.m)
    with _env(PLSS_SELLC=sellc):
        ctx = pkg.plss_create(_matrix(pkg, s), slabs=slabs, maxit_cap=4, validate=True)
    y, v = _spmv_pair(pkg, ctx, s, x, u)
    lens = np.diff(s.row_ptr)
    ref_y = oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)
    short = lens <= 128                    # rows on the warp-tree path (CSR tiles) excepted
    np.testing.assert_array_equal(y[short], ref_y[short])
    clen = np.diff(s.col_ptr)
    ref_v = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
    np.testing.assert_array_equal(v[clen <= 128], ref_v[clen <= 128])
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("slabs", [3, 4, 7])
def test_repeated_spmv_bitwise_stable(pkg, slabs):
    """Races in the shared-memory staging of K2's sigma-permuted y (a ring slot reused while a
    straggler slice still owns it) show up as run-to-run differences: repeat and compare."""
    s = CASES["C5xs"]()
    x = np.random.default_rng(2).standard_normal(s.n)
    u = np.random.default_rng(3).standard_normal(s.m)
    ref_y = oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)
    ref_v = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
    ctx = pkg.plss_create(_matrix(pkg, s), slabs=slabs, maxit_cap=4)
    for _ in range(8):
        y, v = _spmv_pair(pkg, ctx, s, x, u)
        np.testing.assert_array_equal(y, ref_y)
        np.testing.assert_array_equal(v, ref_v)
    pkg.plss_destroy(ctx)
