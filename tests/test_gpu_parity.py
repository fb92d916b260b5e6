"""GPU parity: libplss (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star), fixed: relative residual history within 1e-9 over the first
min(50, K_f) iterations (K_f = the window where two valid oracle orderings agree to 1e-11,
SURVEY 8c-11, measured over 5 row permutations in tests/golden/parity_floor.json), final
||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-7, iterations within 2%. A bar is never widened: where
the oracle disagrees with a row-permuted copy of itself by more than a bar (ill-conditioned C4
runs, DESIGN R11), a miss of that bar is reported as an explicit xfail naming the floor.
SpMV outputs of rows with <= LONGROW (128) entries are sequential ascending-index sums on both
sides: bit-exact. Longer rows use a fixed warp tree: within n*eps*sum|a_ij x_j| of the oracle.
"""
import json
import os

import numpy as np
import pytest

import oracle
import plss_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HIST_TOL = 1e-9
X_TOL = 1e-7
IT_TOL = 0.02
LONGROW = 128
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "parity_floor.json")) as _f:
    FLOOR = json.load(_f)             # scripts/parity_floor.py (oracle vs 5 row-permuted oracles)


def _assert_spmv(got, ptr, idx, val, vec, ref):
    """Bit-exact on segments of <= LONGROW entries; tree-sum bound on longer ones."""
    lens = np.diff(ptr)
    short = lens <= LONGROW
    np.testing.assert_array_equal(got[short], ref[short])
    for i in np.nonzero(~short)[0]:
        seg = slice(ptr[i], ptr[i + 1])
        bound = 2.3e-16 * lens[i] * np.sum(np.abs(val[seg] * vec[idx[seg]]))
        assert abs(got[i] - ref[i]) <= bound, (i, got[i], ref[i])


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


def _gpu_solve(pkg, s, slabs=0, x0=None, sell=True, **kw):
    A = _matrix(pkg, s)
    args = dict(tol=s.tol, tol_mode=s.tol_mode, maxit=s.maxit, flags=1 if s.freeze else 0)
    args.update(kw)
    ctx = pkg.plss_create(A, slabs=slabs, maxit_cap=max(args["maxit"], 1), validate=True, sell=sell)
    b = torch.from_numpy(s.b).cuda()
    xx0 = torch.from_numpy(x0).cuda() if x0 is not None else None
    res = pkg.plss_solve(ctx, b, xx0, want_diag=True, **args)
    res["xh"] = res["x"].cpu().numpy()
    pkg.plss_destroy(ctx)
    return res


def _permuted(s, seed=3):
    perm = np.random.default_rng(seed).permutation(s.m)
    A = s.scipy_csr()[perm]
    A.sort_indices()
    return plss_gen._finish("perm", s.m, s.n, A.indptr, A.indices, A.data, None, s.tol, s.tol_mode,
                            s.maxit, b=s.b[perm], freeze=s.freeze)


def _floor(s, ref, x0=None, kmax=50, key=None):
    """The fp64 parity floor: a second valid oracle ordering (row-permuted A, b)
    run with the same settings. Returns K_f (iterations where the two agree to 1e-11 in hist),
    their iteration-count difference and their final-x difference. With `key`, merged with the
    5-permutation distribution of tests/golden/parity_floor.json (smallest K_f, largest
    differences)."""
    other = oracle.plss_system(_permuted(s), x0=x0, maxit=ref["rec"].shape[0] - 1)
    h0, h1 = ref["hist"], other["hist"]
    k = min(len(h0), len(h1), kmax)
    rel = np.abs(h0[:k] - h1[:k]) / np.maximum(h0[:k], 1e-300)
    bad = np.nonzero(rel > 1e-11)[0]
    nx = np.linalg.norm(ref["x"])
    fl = {"kf": int(bad[0]) if bad.size else k, "diters": abs(other["iters"] - ref["iters"]),
          "dx": np.linalg.norm(other["x"] - ref["x"]) / (nx if nx > 0 else 1.0)}
    return _merge_golden(fl, key, ref)


def _merge_golden(fl, key, ref):
    g = FLOOR.get(key) if key else None
    if g is not None and g["iters"] == ref["iters"]:
        fl = {"kf": min(fl["kf"], g["kf_min"]), "diters": max(fl["diters"], g["diters_max"]),
              "dx": max(fl["dx"], g["dx_max"])}
    return fl


def _assert_parity(res, ref, fl, s):
    """The north_star bars, fixed (no widening): same outcome, hist within 1e-9 for k <= min(50,
    K_f), iterations within 2%, x within 1e-7. A bar the oracle itself misses against a row-permuted
    copy (fl) becomes an explicit xfail when the GPU misses it too."""
    assert res["outcome"] == ref["outcome"], (res["outcome"], ref["outcome"])
    k = min(fl["kf"], 50, len(res["hist"]), len(ref["hist"]))
    assert k >= 1
    h_err = np.max(np.abs(res["hist"][:k] - ref["hist"][:k]) / np.maximum(ref["hist"][:k], 1e-300))
    assert h_err <= HIST_TOL, (h_err, k)
    it_bar = max(1, int(np.ceil(IT_TOL * ref["iters"])))
    d_it = abs(res["iters"] - ref["iters"])
    nx = np.linalg.norm(ref["x"])
    x_err = np.linalg.norm(res["xh"] - ref["x"]) / (nx if nx > 0 else 1.0)
    if d_it > it_bar and fl["diters"] > it_bar:
        pytest.xfail(f"iterations {res['iters']} vs {ref['iters']}: the oracle's own row-permutation floor "
                     f"({fl['diters']}) exceeds the 2% bar ({it_bar})")
    assert d_it <= it_bar, (res["iters"], ref["iters"], it_bar)
    if x_err > X_TOL and fl["dx"] > X_TOL:
        pytest.xfail(f"x error {x_err:.2e}: the oracle's own row-permutation floor ({fl['dx']:.2e}) "
                     f"exceeds the 1e-7 bar")
    assert x_err <= X_TOL, (x_err, fl)
    return h_err, x_err


# ---------------------------------------------------------------------------------------------
# SpMV entry points: bit-exact against the oracle's sequential sums
# ---------------------------------------------------------------------------------------------

def _ragged_system(seed=0, m=3000, n=5000):
    """Zipf row lengths, empty rows, empty columns, rows longer than a tile (spill path)."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.zipf(1.8, m), n)
    lens[::17] = 0                          # empty rows
    lens[5] = n                             # a dense row, longer than a tile + spill
    lens[6] = 4096
    lens[7] = 33                            # just above the warp-cooperative threshold
    cols = []
    for L in lens:
        c = np.sort(rng.choice(n, L, replace=False))
        cols.append(c[c % 13 != 0])         # empty columns
    lens = np.array([c.size for c in cols])
    row_ptr = np.zeros(m + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    col_idx = np.concatenate(cols)
    val = rng.standard_normal(col_idx.size)
    return plss_gen._finish("ragged", m, n, row_ptr, col_idx, val, rng.standard_normal(n), 1e-8, 0, 100)


@pytest.mark.parametrize("slabs,sell", [(1, True), (3, True), (1, False), (3, False)])
def test_spmv_spmvT_bit_exact(pkg, slabs, sell):
    s = _ragged_system()
    A = _matrix(pkg, s)
    ctx = pkg.plss_create(A, slabs=slabs, maxit_cap=10, validate=True, sell=sell)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(s.n)
    u = rng.standard_normal(s.m)
    y = torch.empty(s.m, dtype=torch.float64, device="cuda")
    v = torch.empty(s.n, dtype=torch.float64, device="cuda")
    pkg.plss_spmv(ctx, torch.from_numpy(x).cuda(), y)
    pkg.plss_spmvT(ctx, torch.from_numpy(u).cuda(), v)
    _assert_spmv(y.cpu().numpy(), s.row_ptr, s.col_idx, s.val, x,
                 oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x))
    _assert_spmv(v.cpu().numpy(), s.col_ptr, s.row_idx, s.val_t, u,
                 oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u))
    assert (np.diff(s.row_ptr) > LONGROW).sum() >= 3
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("name", ["C1", "C2s", "C4s", "C5xs"])
def test_spmv_configs_bit_exact(pkg, name):
    s = plss_gen.make_config(name)
    for slabs, sell in ((1, True), (4, True), (1, False), (4, False)):
        A = _matrix(pkg, s)
        ctx = pkg.plss_create(A, slabs=slabs, maxit_cap=4, sell=sell)
        q = pkg.plss_query(ctx)
        if not sell:
            assert q["sell_segments"] == 0
        elif name in ("C1", "C2s", "C5xs"):
            # regular rows: SELL-32 for every CSR slab; CSC slabs of short columns may stay on tiles
            assert q["sell_segments"] == 2 if slabs == 1 else q["sell_segments"] >= q["slabs"]
        x = np.random.default_rng(2).standard_normal(s.n)
        u = np.random.default_rng(3).standard_normal(s.m)
        y = torch.empty(s.m, dtype=torch.float64, device="cuda")
        v = torch.empty(s.n, dtype=torch.float64, device="cuda")
        pkg.plss_spmv(ctx, torch.from_numpy(x).cuda(), y)
        pkg.plss_spmvT(ctx, torch.from_numpy(u).cuda(), v)
        _assert_spmv(y.cpu().numpy(), s.row_ptr, s.col_idx, s.val, x,
                     oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x))
        _assert_spmv(v.cpu().numpy(), s.col_ptr, s.row_idx, s.val_t, u,
                     oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u))
        pkg.plss_destroy(ctx)


# ---------------------------------------------------------------------------------------------
# full solves vs the oracle
# ---------------------------------------------------------------------------------------------

def test_worked_example(pkg):
    s = plss_gen.from_dense(np.diag([2.0, 1.0]), np.array([2.0, 1.0]), tol=1e-14, maxit=10)
    res = _gpu_solve(pkg, s)
    assert res["outcome"] == "converged" and res["iters"] == 2
    np.testing.assert_allclose(res["xh"], [1.0, 1.0], atol=1e-14, rtol=0)
    d = res["diag"]
    assert abs(d[0, 7] - 5 / 17) <= 1e-15 and abs(d[1, 6] - 9 / 25) <= 1e-15 and abs(d[1, 7] - 17 / 20) <= 1e-15


@pytest.mark.parametrize("name,slabs,sell,cap", [
    ("C1", 0, True, 0), ("C2s", 0, True, 0), ("C2s", 3, True, 0), ("C2s", 3, False, 0),
    # C4s (20k x 80k, ill-conditioned): its x window (the largest cap at which 5 row-permuted oracles
    # stay within 1e-9 in x: 10, tests/golden/parity_floor.json) with every bar, and 400 capped
    # steps, where the floor is 1.7e-2 in x (only the history window and the invariants bind)
    ("C4s", 0, True, 10), ("C4s", 0, True, 400), ("C4xs", 0, True, 0),
    ("C5xs", 0, True, 0), ("C5xs", 4, True, 0), ("C5xs", 4, False, 0),
    # C5s: 640k x 80k with C5's +-1024 band, the default 10-slab y-staged schedule of the timed C5
    ("C5s", 10, True, 0)])
def test_solve_parity(pkg, name, slabs, sell, cap):
    s = plss_gen.make_config(name)
    if cap:
        s.maxit = cap
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s, slabs=slabs, sell=sell)
    _assert_parity(res, ref, _floor(s, ref, key=name), s)
    if name.startswith("C4"):
        empty = np.diff(s.col_ptr) == 0      # x in range(A^T): empty columns stay exactly 0
        assert empty.any() and np.all(res["xh"][empty] == 0.0)


def test_solve_parity_c3_scaled(pkg):
    s = plss_gen.make_config("C3", N=128)
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    _assert_parity(res, ref, _floor(s, ref, key="C3_128"), s)
    assert np.max(np.abs(res["xh"] - 1.0)) <= 1e-5


def test_solve_parity_c2_full(pkg):
    s = plss_gen.make_config("C2")
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    _assert_parity(res, ref, _floor(s, ref), s)


def test_scalar_records_match_oracle(pkg):
    s = plss_gen.make_config("C1")
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    d, r = res["diag"], ref["rec"]
    for k in range(1, 30):
        for col in (1, 2, 4, 6, 7):   # rho, phi, theta, beta, gamma
            assert abs(d[k, col] - r[k, col]) <= 1e-9 * abs(r[k, col]), (k, col)
        assert abs(d[k, 3] / d[k, 1] + 1) <= 1e-12        # psi = -rho (L671-672)


def test_nonzero_x0(pkg):
    s = plss_gen.make_config("C2s")
    x0 = np.random.default_rng(5).standard_normal(s.n)
    ref = oracle.plss_system(s, x0=x0)
    res = _gpu_solve(pkg, s, x0=x0)
    _assert_parity(res, ref, _floor(s, ref, x0=x0), s)


def test_host_buffers_equal_device_buffers(pkg):
    s = plss_gen.make_config("C2s")
    A = _matrix(pkg, s)
    ctx = pkg.plss_create(A, maxit_cap=s.maxit)
    r_dev = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, maxit=s.maxit)
    xh = np.zeros(s.n)
    r_host = pkg.plss_solve(ctx, s.b.copy(), tol=s.tol, maxit=s.maxit, x=xh)
    assert r_dev["iters"] == r_host["iters"]
    np.testing.assert_array_equal(r_dev["x"].cpu().numpy(), xh)
    pkg.plss_destroy(ctx)


def test_deterministic_run_to_run(pkg):
    s = plss_gen.make_config("C4s")
    a = _gpu_solve(pkg, s, maxit=200)
    b = _gpu_solve(pkg, s, maxit=200)
    np.testing.assert_array_equal(a["xh"], b["xh"])
    np.testing.assert_array_equal(a["hist"], b["hist"])


def test_freeze_mode_fixed_iterations(pkg):
    s = plss_gen.make_config("C5xs")
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    assert res["iters"] == s.maxit == ref["iters"]
    assert res["outcome"] == ref["outcome"] == "maxit"
    assert np.linalg.norm(res["xh"] - ref["x"]) / np.linalg.norm(ref["x"]) <= X_TOL
    d = res["diag"]
    frozen = np.nonzero(d[:s.maxit, 0] <= oracle.FREEZE_H)[0]
    assert frozen.size and np.all(d[frozen[0] + 1:s.maxit, 6] == 0.0)


# ---------------------------------------------------------------------------------------------
# edge and degenerate cases
# ---------------------------------------------------------------------------------------------

def test_zero_rhs_converges_immediately(pkg):
    s = plss_gen.make_config("C2s")
    s.b = np.zeros(s.m)
    res = _gpu_solve(pkg, s)
    assert res["iters"] == 0 and res["outcome"] == "converged"
    assert np.all(res["xh"] == 0.0)


def test_exact_start(pkg):
    s = plss_gen.make_config("C3", N=32)
    res = _gpu_solve(pkg, s, x0=np.ones(s.n))
    ref = oracle.plss_system(s, x0=np.ones(s.n))
    assert res["iters"] == ref["iters"] and res["outcome"] == ref["outcome"]


def test_y_vanished(pkg):
    s = plss_gen.from_dense(np.array([[1.0], [0.0]]), np.array([0.0, 1.0]), keep_zeros=True,
                            tol=1e-12, maxit=10)
    res = _gpu_solve(pkg, s)
    assert res["outcome"] == "y_vanished" and res["iters"] == 0


def test_identity_one_step(pkg):
    b = np.arange(1.0, 301.0)
    s = plss_gen.from_dense(np.eye(300), b, tol=1e-15, maxit=5)
    res = _gpu_solve(pkg, s)
    assert res["iters"] == 1
    np.testing.assert_array_equal(res["xh"], b)


def test_empty_matrix(pkg):
    m, n = 50, 40
    s = plss_gen._finish("empty", m, n, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), None,
                         1e-8, 0, 5, b=np.zeros(m))
    res = _gpu_solve(pkg, s)
    assert res["iters"] == 0 and res["outcome"] == "converged"
    s.b = np.ones(m)
    res = _gpu_solve(pkg, s)
    assert res["outcome"] == "y_vanished"


def test_maxit_one_and_cap(pkg):
    s = plss_gen.make_config("C1")
    res = _gpu_solve(pkg, s, maxit=1)
    ref = oracle.plss_system(s, maxit=1)
    assert res["iters"] == ref["iters"] == 1 and res["outcome"] == ref["outcome"] == "maxit"
    np.testing.assert_allclose(res["xh"], ref["x"], rtol=1e-12)
    A = _matrix(pkg, s)
    ctx = pkg.plss_create(A, maxit_cap=10)
    with pytest.raises(pkg.PlssError):
        pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), maxit=11)
    with pytest.raises(pkg.PlssError):
        pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=-1.0, maxit=5)
    pkg.plss_destroy(ctx)


def test_validation_rejects_bad_matrices(pkg):
    s = plss_gen.make_config("C2s")
    bad = plss_gen.make_config("C2s")
    bad.col_idx = bad.col_idx.copy()
    bad.col_idx[[8, 9]] = bad.col_idx[[9, 8]]           # unsorted row
    with pytest.raises(pkg.PlssError, match="format"):
        pkg.plss_create(_matrix(pkg, bad), validate=True)
    bad = plss_gen.make_config("C2s")
    bad.col_idx = bad.col_idx.copy()
    bad.col_idx[0] = s.n + 5                             # out of range
    with pytest.raises(pkg.PlssError, match="format"):
        pkg.plss_create(_matrix(pkg, bad), validate=True)
    bad = plss_gen.make_config("C2s")
    bad.val_t = bad.val_t.copy()
    bad.val_t[7] += 1.0                                  # CSC is not the transpose
    with pytest.raises(pkg.PlssError, match="format"):
        pkg.plss_create(_matrix(pkg, bad), validate=True)
    bad = plss_gen.make_config("C2s")
    bad.val = bad.val.copy()
    bad.val[3] = np.nan
    with pytest.raises(pkg.PlssError, match="format"):
        pkg.plss_create(_matrix(pkg, bad), validate=True)


def test_slabs_agree(pkg):
    s = plss_gen.make_config("C5xs")
    a = _gpu_solve(pkg, s, slabs=1)
    b = _gpu_solve(pkg, s, slabs=7)
    assert a["iters"] == b["iters"]
    k = 25
    assert np.max(np.abs(a["hist"][:k] - b["hist"][:k]) / a["hist"][:k]) <= 1e-11


# ---------------------------------------------------------------------------------------------
# PLSS W (diagonal WI = diag(||A_{:,j}||), NEXT-1): same kernels, K2's last slab stores WIy and
# weights phi, K3 weights theta
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name,slabs,cap", [("C1", 0, 0), ("C2s", 0, 0), ("C2s", 3, 0), ("C4s", 0, 10),
                                            ("C4xs", 0, 0), ("C5xs", 0, 0), ("C5xs", 4, 0)])
def test_plssw_solve_parity(pkg, name, slabs, cap):
    s = plss_gen.make_config(name)
    if cap:
        s.maxit = cap              # C4s: its x window (tests/golden/parity_floor.json, C4s_W)
    A = _matrix(pkg, s)
    ctx = pkg.plss_create(A, slabs=slabs, maxit_cap=s.maxit, validate=True)
    c = pkg.plss_column_norms(ctx)
    c_ref = oracle.column_norms(s.n, s.col_ptr, s.val_t)
    np.testing.assert_array_equal(c.cpu().numpy(), c_ref)          # same sums, same sqrt
    pkg.plss_set_wi(ctx, c)
    res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, tol_mode=s.tol_mode, maxit=s.maxit,
                         flags=1 if s.freeze else 0, want_diag=True)
    res["xh"] = res["x"].cpu().numpy()
    ref = oracle.plss_system(s, wi=c_ref)
    # parity floor of the weighted oracle (row-permuted ordering)
    other = oracle.plss_system(_permuted(s), wi=c_ref, maxit=ref["rec"].shape[0] - 1)
    k = min(len(ref["hist"]), len(other["hist"]), 50)
    rel = np.abs(ref["hist"][:k] - other["hist"][:k]) / np.maximum(ref["hist"][:k], 1e-300)
    bad = np.nonzero(rel > 1e-11)[0]
    nx = np.linalg.norm(ref["x"])
    fl = {"kf": int(bad[0]) if bad.size else k, "diters": abs(other["iters"] - ref["iters"]),
          "dx": np.linalg.norm(other["x"] - ref["x"]) / (nx if nx > 0 else 1.0)}
    _assert_parity(res, ref, _merge_golden(fl, name + "_W", ref), s)
    # WI-orthogonality identity psi_k = -rho_{k-1}, as for PLSS (invariant under the transform)
    d = res["diag"]
    live = [kk for kk in range(1, min(res["iters"], 20)) if d[kk, 0] > 1e-8]
    for kk in live:
        assert abs(d[kk, 3] / d[kk, 1] + 1.0) <= 1e-8
    # WI = I again reproduces plain PLSS on the same ctx
    pkg.plss_set_wi(ctx, None)
    plain = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, tol_mode=s.tol_mode, maxit=s.maxit,
                           flags=1 if s.freeze else 0)
    ref0 = oracle.plss_system(s)
    assert abs(plain["iters"] - ref0["iters"]) <= max(1, int(np.ceil(IT_TOL * ref0["iters"])))
    pkg.plss_destroy(ctx)


def test_plssw_rejects_bad_weights(pkg):
    s = plss_gen.make_config("C1")
    ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=4)
    w = np.ones(s.n)
    w[3] = 0.0
    with pytest.raises(pkg.PlssError, match="invalid"):
        pkg.plss_set_wi(ctx, w)
    w[3] = np.nan
    with pytest.raises(pkg.PlssError, match="invalid"):
        pkg.plss_set_wi(ctx, w)
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("name", ["C2s", "C4xs", "C1"])
def test_true_residual_at_exit(pkg, name):
    """the solve stops on the recursive residual; plss_true_residual reports
    ||b - A x|| / ||b|| once at exit. Checked against the oracle's own SpMV of the returned x (both
    sums per row are sequential and bitwise equal; only the final norm's order differs), host and
    device arguments, and against the recursive history at convergence."""
    s = plss_gen.make_config(name)
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    ctx = pkg.plss_create(A, maxit_cap=s.maxit)
    res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, maxit=s.maxit)
    x = res["x"].cpu().numpy()
    ref = np.linalg.norm(s.b - oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x))
    for b_arg, x_arg in ((s.b, x), (torch.from_numpy(s.b).cuda(), res["x"])):
        t = pkg.plss_true_residual(ctx, b_arg, x_arg)
        assert abs(t["abs"] - ref) <= 1e-12 * np.linalg.norm(s.b)
        assert abs(t["norm_b"] - np.linalg.norm(s.b)) <= 1e-13 * np.linalg.norm(s.b)
    if res["outcome"] == "converged":                 # recursive and true residual agree at the end
        assert t["rel"] <= 10 * s.tol + 1e-13
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("m,n", [(0, 5), (5, 0), (0, 0)])
def test_degenerate_dimensions(pkg, m, n):
    """Zero rows or columns: the ctx builds, b has no residual to reduce (||b|| = 0 or A^T r = 0),
    the solve reports converged / y_vanished without launching a bad grid, the SpMVs are no-ops."""
    s = plss_gen._finish("degenerate", m, n, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), None,
                         1e-8, 0, 5, b=np.ones(m))
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    assert res["iters"] == ref["iters"] == 0
    assert res["outcome"] == ref["outcome"]
    assert res["xh"].shape == (n,)
    A = _matrix(pkg, s)
    ctx = pkg.plss_create(A, maxit_cap=5, validate=True)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    v = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.plss_spmv(ctx, torch.zeros(n, dtype=torch.float64, device="cuda"), y)
    pkg.plss_spmvT(ctx, torch.zeros(m, dtype=torch.float64, device="cuda"), v)
    pkg.plss_destroy(ctx)


def test_stagnation_outcome(pkg):
    """STAGNATION (tau - 1 <= 1e-14) on the GPU: A = [1; 1], b = e_1 has tau = 1
    exactly at the first loop step (worked by hand in test_oracle_pins.py); the outcome, the one
    applied update and the record match the oracle, normal and freeze mode."""
    s = plss_gen.from_dense(np.array([[1.0], [1.0]]), np.array([1.0, 0.0]), tol=1e-12, maxit=10)
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    assert res["outcome"] == ref["outcome"] == "stagnation" and res["iters"] == ref["iters"] == 1
    assert res["xh"].tolist() == ref["x"].tolist() == [1.0]
    assert res["diag"][1, 0] == ref["rec"][1, 0] == 1.0
    res = _gpu_solve(pkg, s, tol=0.0, maxit=6, flags=1)
    assert res["outcome"] == "stagnation" and res["iters"] == 6 and res["xh"].tolist() == [1.0]


def test_stagnation_inconsistent_random(pkg):
    """An inconsistent 300 x 100 system: the recursive residual stops moving once it reaches
    b's component outside range(A) and the guard fires; outcome and step count equal the
    oracle's (201 steps)."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((300, 100))
    s = plss_gen.from_dense(A, rng.standard_normal(300), tol=1e-12, maxit=400)
    ref = oracle.plss_system(s)
    res = _gpu_solve(pkg, s)
    assert ref["outcome"] == "stagnation"
    assert res["outcome"] == "stagnation"
    assert abs(res["iters"] - ref["iters"]) <= max(1, int(np.ceil(IT_TOL * ref["iters"])))
