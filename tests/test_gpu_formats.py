"""GPU: which format each segment takes (plss_query_segment) and the round-2 formats
against the oracle: static stepping (C5's K1), globally sorted rows with the long ones in
k_longchunks (C4's K1; k_longrows with PLSS_LCHUNK=0), a thread per short column (k_scalar, C4's K2), and the 1024-row sigma windows
of K2 (the SIGMA_WIDE path had no test of its own), each bitwise on its SpMV outputs,
repeatable, and inside a solve (also on a single-rank chunked distributed ctx)."""
import json
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


class _env:
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


def _matrix(pkg, s):
    return pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)


def _spmv_pair(pkg, ctx, s, x, u):
    y = torch.empty(s.m, dtype=torch.float64, device="cuda")
    v = torch.empty(s.n, dtype=torch.float64, device="cuda")
    pkg.plss_spmv(ctx, torch.from_numpy(x).cuda(), y)
    pkg.plss_spmvT(ctx, torch.from_numpy(u).cuda(), v)
    return y.cpu().numpy(), v.cpu().numpy()


def _check(got, ptr, idx, val, vec, ref):
    lens = np.diff(ptr)
    short = lens <= 128
    np.testing.assert_array_equal(got[short], ref[short])
    for i in np.nonzero(~short)[0]:
        seg = slice(ptr[i], ptr[i + 1])
        assert abs(got[i] - ref[i]) <= 2.3e-16 * lens[i] * np.sum(np.abs(val[seg] * vec[idx[seg]]))


def _spmv_bitwise_repeatable(pkg, ctx, s, seed=1):
    rng = np.random.default_rng(seed)
    x, u = rng.standard_normal(s.n), rng.standard_normal(s.m)
    y, v = _spmv_pair(pkg, ctx, s, x, u)
    _check(y, s.row_ptr, s.col_idx, s.val, x, oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x))
    _check(v, s.col_ptr, s.row_idx, s.val_t, u, oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u))
    for _ in range(3):
        y2, v2 = _spmv_pair(pkg, ctx, s, x, u)
        np.testing.assert_array_equal(y2, y)
        np.testing.assert_array_equal(v2, v)


def test_c5_formats_static_k1_sigma_k2(pkg):
    s = plss_gen.make_config("C5xs")
    ctx = pkg.plss_create(_matrix(pkg, s), slabs=4, maxit_cap=8)
    for sl in range(4):
        k1 = pkg.plss_query_segment(ctx, 1, sl)
        k2 = pkg.plss_query_segment(ctx, 2, sl)
        assert k1["fmt"] == 3 and k1["stat"] == 2 and k1["gsort"] == 0     # rows of 12: 6 in flight
        assert k2["fmt"] == 3 and k2["sig"] == 512 and k2["stat"] == 0
    _spmv_bitwise_repeatable(pkg, ctx, s)
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("name", ["C4s", "C4xs"])
def test_c4_formats_longrows_and_scalar(pkg, name):
    s = plss_gen.make_config(name)
    ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=8)
    k1 = pkg.plss_query_segment(ctx, 1, 0)
    k2 = pkg.plss_query_segment(ctx, 2, 0)
    assert k1["fmt"] == 3 and k1["gsort"] == 1 and k1["nlong"] == int((np.diff(s.row_ptr) > 128).sum()) > 0
    # the one-entry rows (sorted last) run in k_sell's batched phase 2: from the first slice whose
    # longest row has one entry; the rows have >= 1 entry, so there is no empty slice
    lens = np.sort(np.diff(s.row_ptr)[np.diff(s.row_ptr) <= 128])[::-1]
    assert k1["s1beg"] == (int(np.argmax(lens <= 1)) + 31) // 32 and k1["s1end"] == k1["nslices"], k1
    assert k2["fmt"] == 5                                   # columns of ~1 entry: a thread per column
    assert k1["lin"] == 0 and pkg.plss_query(ctx)["launches_per_step"] == 4   # k_sell + k_longchunks, k_scalar, K3
    _spmv_bitwise_repeatable(pkg, ctx, s)
    pkg.plss_destroy(ctx)


def test_k2_wide_sigma_windows(pkg):
    """With k_scalar off, C4s's K2 columns (power-law transposed: 35% empty) leave > 15% padding in
    512-row sigma windows and take 1024-row ones (SIGMA_WIDE, y staged in shared memory);
    PLSS_SIGWIDE=0 sends them to the global sort. Both bitwise and repeatable, and the solve agrees
    with the default formats' solve within the parity floor."""
    s = plss_gen.make_config("C4s")
    with _env(PLSS_SCALAR=0):
        ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
    k2 = pkg.plss_query_segment(ctx, 2, 0)
    assert k2["fmt"] == 3 and k2["sig"] == 1024 and k2["gsort"] == 0, k2
    _spmv_bitwise_repeatable(pkg, ctx, s)
    b = torch.from_numpy(s.b).cuda()
    wide = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)
    pkg.plss_destroy(ctx)
    with _env(PLSS_SCALAR=0, PLSS_SIGWIDE=0):
        ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
    k2 = pkg.plss_query_segment(ctx, 2, 0)
    assert k2["fmt"] == 3 and k2["sig"] == 0 and k2["gsort"] == 1, k2
    assert 0 < k2["s1beg"] < k2["s1end"] < k2["nslices"], k2     # one-entry columns, then empty ones
    _spmv_bitwise_repeatable(pkg, ctx, s)
    glob = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)
    pkg.plss_destroy(ctx)
    ref = oracle.plss_system(s, maxit=40)
    k = 12                                                   # C4s's K_f is 16 (tests/golden/parity_floor.json)
    for res in (wide, glob):
        assert np.max(np.abs(res["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9


def test_wide_sigma_chunked_dist_single_rank(pkg):
    """the column chunks of the distributed step (make_chunks) follow the segment's sigma
    window; a single-rank NCCL ctx whose last K2 segment has 1024-row windows solves like the plain
    ctx and bitwise like its own unchunked form."""
    s = plss_gen.make_config("C4s")
    A = _matrix(pkg, s)
    b = torch.from_numpy(s.b).cuda()
    out = {}
    for chunks in (1, 4):
        with _env(PLSS_SCALAR=0, PLSS_DIST_CHUNKS=chunks):
            ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=1, maxit_cap=60)
        assert pkg.plss_query_segment(ctx, 2, 0)["sig"] == 1024
        out[chunks] = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)
        out[chunks]["xh"] = out[chunks]["x"].cpu().numpy()
        pkg.plss_destroy(ctx)
    np.testing.assert_array_equal(out[1]["hist"], out[4]["hist"])
    np.testing.assert_array_equal(out[1]["xh"], out[4]["xh"])
    ref = oracle.plss_system(s, maxit=40)
    assert np.max(np.abs(out[4]["hist"][:12] - ref["hist"][:12]) / ref["hist"][:12]) <= 1e-9


def test_query_segment_rejects_bad_arguments(pkg):
    s = plss_gen.make_config("C1")
    ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=4)
    for which, slab in ((0, 0), (3, 0), (1, 5), (2, -1)):
        with pytest.raises(pkg.PlssError):
            pkg.plss_query_segment(ctx, which, slab)
    pkg.plss_destroy(ctx)


def _long_rows_system(transpose=False, seed=7):
    """Short rows (1 .. 8 entries) plus 70 long ones (> LONGROW = 128 entries: 129 .. 5000, chunk
    boundaries of LCH = 384 straddled, 70 = two full groups of 32 rows and a ragged one) in random
    positions; distinct uniform columns, U(-1, 1) values, b = A x*. transpose: the same matrix
    transposed, so K2's columns are the long ones."""
    rng = np.random.default_rng(seed)
    m, n = 20000, 30000
    lens = rng.integers(1, 9, size=m)
    fixed = [129, 130, 383, 384, 385, 767, 768, 769, 1000, 1152, 4096, 5000]
    extra = rng.integers(129, 3000, size=70 - len(fixed))
    pos = rng.choice(m, size=70, replace=False)
    lens[pos] = np.concatenate([fixed, extra])
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    idx = np.concatenate([np.sort(rng.choice(n, size=L, replace=False)) for L in lens])
    val = rng.uniform(-1, 1, size=ptr[-1])
    if transpose:
        import scipy.sparse as sp
        At = sp.csr_matrix((val, idx, ptr), shape=(m, n)).T.tocsr()
        At.sort_indices()
        m, n, ptr, idx, val = n, m, At.indptr, At.indices, At.data
    xs = rng.standard_normal(n)
    return plss_gen._finish("longrows" + ("T" if transpose else ""), m, n, ptr, idx, val, xs, 1e-10, 0, 40)


@pytest.mark.parametrize("transpose", [False, True])
def test_long_rows_in_chunks(pkg, transpose):
    """k_longchunks (a warp per chunk of LCH entries, rows finished by their last chunk's warp, row
    dot terms in two fixed levels, joint election with the slices' CTAs): K1's long rows (or K2's
    long columns for the transposed matrix) -- chunk count as set up, SpMV bitwise on short rows and
    within the tree-sum bound on long ones, repeatable; the solve bitwise the same whether or not
    k_longchunks runs concurrently with the slices (so whichever launch finalizes, the totals are
    the same: final_sum2's fixed shape), bitwise repeatable, and against the oracle within the bar."""
    s = _long_rows_system(transpose)
    which = 2 if transpose else 1
    lens = np.diff(s.col_ptr if transpose else s.row_ptr)
    ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
    seg = pkg.plss_query_segment(ctx, which, 0)
    L = lens[lens > 128]
    assert seg["fmt"] == 3 and seg["gsort"] == 1 and seg["nlong"] == len(L) == 70, seg
    assert seg["nchunks"] == int(np.sum((L + 383) // 384)), seg
    _spmv_bitwise_repeatable(pkg, ctx, s)
    b = torch.from_numpy(s.b).cuda()
    runs = [pkg.plss_solve(ctx, b, tol=s.tol, maxit=40) for _ in range(2)]
    pkg.plss_destroy(ctx)
    with _env(PLSS_FORK=0):
        ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
    runs.append(pkg.plss_solve(ctx, b, tol=s.tol, maxit=40))
    pkg.plss_destroy(ctx)
    for r in runs[1:]:
        assert r["iters"] == runs[0]["iters"]
        np.testing.assert_array_equal(r["hist"], runs[0]["hist"])
        np.testing.assert_array_equal(r["x"].cpu().numpy(), runs[0]["x"].cpu().numpy())
    with _env(PLSS_LCHUNK=0):                                  # the CTA-per-row k_longrows
        ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
    assert pkg.plss_query_segment(ctx, which, 0)["nchunks"] == 0
    _spmv_bitwise_repeatable(pkg, ctx, s)
    rows = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)
    pkg.plss_destroy(ctx)
    ref = oracle.plss_system(s, maxit=40)
    k = min(20, len(ref["hist"]) - 1)
    for res in (runs[0], rows):
        assert np.max(np.abs(res["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9


@pytest.mark.parametrize("name,slabs", [("C5xs", 4), ("C4xs", 1), ("C1", 1)])
def test_psi_summed_in_k3(pkg, name, slabs):
    """DESIGN.md R25: on one device with WI = I, K2's finalizing segment reads no p and K3 sums
    psi = y_k^T p_{k-1} from the y and p it reads anyway (psi3). Every other scalar record is
    bitwise the same as with psi summed in K2 (PLSS_PSI3=0); psi agrees to rounding and keeps the
    identity psi = -rho. Under PLSS W (and on a distributed ctx) K2 keeps summing psi."""
    s = plss_gen.make_config(name)
    A = _matrix(pkg, s)
    b = torch.from_numpy(s.b).cuda()
    runs = {}
    for flag in (1, 0):
        with _env(PLSS_PSI3=flag):
            ctx = pkg.plss_create(A, slabs=slabs, maxit_cap=40)
        S = pkg.plss_query(ctx)["slabs"]
        assert [pkg.plss_query_segment(ctx, 2, sl)["psi3"] for sl in range(S)] == [0] * (S - 1) + [flag]
        runs[flag] = pkg.plss_solve(ctx, b, tol=0.0, maxit=30, flags=1, want_diag=True)
        if flag:
            pkg.plss_set_wi(ctx, pkg.plss_column_norms(ctx))
            runs["w1"] = pkg.plss_solve(ctx, b, tol=0.0, maxit=30, flags=1, want_diag=True)
        else:
            pkg.plss_set_wi(ctx, pkg.plss_column_norms(ctx))
            runs["w0"] = pkg.plss_solve(ctx, b, tol=0.0, maxit=30, flags=1, want_diag=True)
        pkg.plss_destroy(ctx)
    d1, d0 = runs[1]["diag"], runs[0]["diag"]
    live = np.arange(1, 30)
    for col in (0, 1, 2, 4, 5, 6, 7):                      # hist, rho, phi, theta, tau, beta, gamma
        np.testing.assert_array_equal(d1[:31, col], d0[:31, col])
    np.testing.assert_allclose(d1[live, 3], d0[live, 3], rtol=1e-12, atol=0)
    assert np.all(np.abs(d1[live, 3] / d1[live, 1] + 1) <= 1e-9)         # psi = -rho
    np.testing.assert_array_equal(runs["w1"]["diag"], runs["w0"]["diag"])  # PLSS W: psi from K2 either way
    with _env(PLSS_DIST_CHUNKS=1):
        ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=1, maxit_cap=8)
    assert pkg.plss_query_segment(ctx, 2, 0)["psi3"] == 0
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("name,slabs", [("C5xs", 4), ("C4xs", 1), ("C1", 1)])
def test_x_every_other_step(pkg, name, slabs):
    """DESIGN.md R25: on one device K3 updates x every other step, x <- (x + p_{k-1}) + p_k, and
    plss_finish applies a pending update -- bitwise the sequential x_k = x_{k-1} + p_k (L813) after
    any number of steps, also across start / step / finish / step / finish and early stops."""
    s = plss_gen.make_config(name)
    A = _matrix(pkg, s)
    b = torch.from_numpy(s.b).cuda()
    out = {}
    for flag in (1, 0):
        with _env(PLSS_XDEFER=flag):
            ctx = pkg.plss_create(A, slabs=slabs, maxit_cap=40)
        assert pkg.plss_query_segment(ctx, 1, 0)["xdefer"] == flag
        for maxit in (29, 30):                                    # odd and even step counts
            r = pkg.plss_solve(ctx, b, tol=0.0, maxit=maxit, flags=1, want_diag=True)
            out[flag, maxit] = (r["x"].cpu().numpy(), r["diag"])
        r = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)           # stops on the tolerance (or maxit)
        out[flag, "tol"] = (r["x"].cpu().numpy(), r["iters"])
        pkg.plss_start(ctx, b, None, tol=0.0, maxit=40, flags=1)
        xs = []
        for k in (7, 6, 1):
            pkg.plss_step(ctx, k)
            xb = torch.empty(s.n, dtype=torch.float64, device="cuda")
            pkg.plss_finish(ctx, x=xb)
            xs.append(xb.cpu().numpy())
        out[flag, "split"] = xs
        pkg.plss_destroy(ctx)
    for key in ((29,), (30,)):
        np.testing.assert_array_equal(out[1, key[0]][0], out[0, key[0]][0])
        np.testing.assert_array_equal(out[1, key[0]][1], out[0, key[0]][1])
    np.testing.assert_array_equal(out[1, "tol"][0], out[0, "tol"][0])
    assert out[1, "tol"][1] == out[0, "tol"][1]
    for a, c in zip(out[1, "split"], out[0, "split"]):
        np.testing.assert_array_equal(a, c)
    # the row-block step (single-rank NCCL ctx, chunked all-reduce): x every other step and psi in K3
    # (k_dots_tail reads no p) as well; x and every record but psi bitwise their every-step forms
    dist_out = {}
    for flag in (1, 0):
        with _env(PLSS_DIST_CHUNKS=4, PLSS_XDEFER=flag, PLSS_PSI3=flag):
            ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=1, maxit_cap=40)
        assert pkg.plss_query_segment(ctx, 1, 0)["xdefer"] == flag
        r = pkg.plss_solve(ctx, b, tol=0.0, maxit=29, flags=1, want_diag=True)
        dist_out[flag] = (r["x"].cpu().numpy(), r["diag"])
        pkg.plss_destroy(ctx)
    np.testing.assert_array_equal(dist_out[1][0], dist_out[0][0])
    for col in (0, 1, 2, 4, 5, 6, 7):
        np.testing.assert_array_equal(dist_out[1][1][:, col], dist_out[0][1][:, col])
    np.testing.assert_allclose(dist_out[1][1][1:30, 3], dist_out[0][1][1:30, 3], rtol=1e-12, atol=0)


@pytest.mark.parametrize("name", ["C4s", "C4xs"])
def test_batched_one_step_slices_bitwise(pkg, name):
    """k_sell's batched phase 2 for the one-entry rows of a globally sorted K1 segment computes each
    row's sum, r update and per-slice dot partial as the one-slice-at-a-time path does: with the
    same CTA ranges (the batched slices costed like the others, PLSS_UC_S1=48) a solve is bitwise
    the PLSS_S1=0 solve (history, x, scalar records); with the default costing it still agrees with
    the oracle over the parity window."""
    s = plss_gen.make_config(name)
    b = torch.from_numpy(s.b).cuda()
    runs = {}
    for lab, env in (("off", dict(PLSS_S1=0)), ("same", dict(PLSS_UC_S1=48)), ("default", {})):
        with _env(**env):
            ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
        k1 = pkg.plss_query_segment(ctx, 1, 0)
        assert (k1["s1beg"] >= 0) == (lab != "off"), (lab, k1)
        res = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)
        runs[lab] = (res["hist"], res["x"].cpu().numpy())
        pkg.plss_destroy(ctx)
    np.testing.assert_array_equal(runs["same"][0], runs["off"][0])
    np.testing.assert_array_equal(runs["same"][1], runs["off"][1])
    ref = oracle.plss_system(s, maxit=40)
    with open(os.path.join(os.path.dirname(__file__), "golden", "parity_floor.json")) as f:
        k = json.load(f)[name]["kf_min"]                     # the window two oracle orderings agree on
    h = runs["default"][0]
    assert np.max(np.abs(h[:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9


@pytest.mark.parametrize("name", ["C4s", "C4xs"])
def test_inline_long_row_chunks_bitwise(pkg, name):
    """k_sell's phase 0 (opt-in, PLSS_LIN=1) runs the long rows' chunks with the same per-lane
    order, chunk order, row-dot groups and partial slot as the concurrent k_longchunks launch (the
    default): the solves are bitwise equal (history, x), and one launch per step fewer."""
    s = plss_gen.make_config(name)
    b = torch.from_numpy(s.b).cuda()
    runs = {}
    for lab, env in (("launch", {}), ("inline", dict(PLSS_LIN=1))):
        with _env(**env):
            ctx = pkg.plss_create(_matrix(pkg, s), maxit_cap=60)
        runs[lab + "_launches"] = pkg.plss_query(ctx)["launches_per_step"]
        _spmv_bitwise_repeatable(pkg, ctx, s)
        res = pkg.plss_solve(ctx, b, tol=s.tol, maxit=40)
        runs[lab] = (res["hist"], res["x"].cpu().numpy(), res["iters"])
        pkg.plss_destroy(ctx)
    assert runs["inline_launches"] == runs["launch_launches"] - 1
    np.testing.assert_array_equal(runs["inline"][0], runs["launch"][0])
    np.testing.assert_array_equal(runs["inline"][1], runs["launch"][1])
