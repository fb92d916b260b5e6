"""Peer-memory all-reduce of the distributed step (SURVEY 8(e) improvement 3, options.flags bit3,
paper_2207_07615_b200/csrc/peer_kernels.cuh).

With one GPU the cross-rank logic runs as its emulation: plss_peer_reduce_emulate launches the
step's own kernels cooperatively with one grid row per VIRTUAL rank over G sets of buffers (the
kernels' CTAs wait on one another, so they must be co-resident; B200_PROFILING.md forbids separate
launches that wait on each other). Checked: every virtual rank's reduced vector is bitwise the
rank-order sum ((part_0 + part_1) + ...) + part_{G-1}, elements outside the chunks are untouched,
ragged / empty / odd-aligned chunks, and the epoch carried by the flags across many steps.
The solve itself runs the peer step on a real single-rank distributed ctx (the peer table then maps
only its own region): bitwise the NCCL all-reduce step, with the chunks engaged.
"""
import numpy as np
import pytest

import oracle
import plss_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PF_EP = 2 * 8 * 8 + 8          # peer_kernels.cuh: flag block word holding the completed steps
PF_ERR = PF_EP + 1


@pytest.fixture(scope="module")
def pkg():
    from paper_2207_07615_b200 import build as pbuild
    pbuild.build()
    import paper_2207_07615_b200 as p
    p.load_library()
    assert torch.cuda.is_available()
    return p


def _rank_order_sum(parts):
    acc = parts[0].copy()
    for q in parts[1:]:
        acc = acc + q                      # binary64 adds in rank order, as the kernel does
    return acc


BOUNDS = {
    "one_chunk": lambda n: [0, n],
    "ragged": lambda n: [7, 1000, 1001, 1001, 5003, n - 3],      # odd offsets, a 1-element and an empty chunk
    "eight": lambda n: list(np.linspace(0, n, 9).astype(np.int64)),
}


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("kind", list(BOUNDS))
def test_peer_reduce_emulate(pkg, G, kind):
    n = 20001
    bounds = BOUNDS[kind](n)
    rng = np.random.default_rng(G * 10 + len(bounds))
    flags = [torch.zeros(256, dtype=torch.int32, device="cuda") for _ in range(G)]
    sentinel = 12345.0
    reds = [torch.full((n + 8,), sentinel, dtype=torch.float64, device="cuda") for _ in range(G)]
    lo, hi = bounds[0], bounds[-1]
    for step in range(3):                         # new data each step; the flags carry the epoch
        parts_h = [rng.standard_normal(n + 8) * 10.0 ** rng.integers(-3, 4) for _ in range(G)]
        parts = [torch.from_numpy(p).cuda() for p in parts_h]
        pkg.plss_peer_reduce_emulate(parts, reds, flags, bounds)
        want = _rank_order_sum(parts_h)
        for h in range(G):
            got = reds[h].cpu().numpy()
            np.testing.assert_array_equal(got[lo:hi], want[lo:hi])
            assert np.all(got[:lo] == sentinel) and np.all(got[hi:] == sentinel)
            f = flags[h].cpu().numpy()
            assert f[PF_EP] == step + 1 and f[PF_ERR] == 0


def test_peer_reduce_emulate_many_steps(pkg):
    """200 steps of 8 virtual ranks over 4 chunks: the epochs never desynchronize."""
    G, n = 8, 4099
    bounds = [0, 1024, 2048, 3072, n]
    flags = [torch.zeros(256, dtype=torch.int32, device="cuda") for _ in range(G)]
    reds = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(G)]
    parts = [torch.full((n,), float(h + 1), dtype=torch.float64, device="cuda") for h in range(G)]
    for step in range(200):
        parts[step % G].add_(1.0)
        pkg.plss_peer_reduce_emulate(parts, reds, flags, bounds)
    want = _rank_order_sum([p.cpu().numpy() for p in parts])
    for h in range(G):
        np.testing.assert_array_equal(reds[h].cpu().numpy(), want)
        assert flags[h].cpu().numpy()[PF_EP] == 200


def test_peer_reduce_emulate_errors(pkg):
    t = [torch.zeros(8, dtype=torch.float64, device="cuda")]
    f = [torch.zeros(256, dtype=torch.int32, device="cuda")]
    with pytest.raises(pkg.PlssError):
        pkg.plss_peer_reduce_emulate(t * 9, t * 9, f * 9, [0, 8])             # > 8 ranks
    with pytest.raises(pkg.PlssError):
        pkg.plss_peer_reduce_emulate(t, t, f, [0, 5, 3])                     # decreasing bounds
    with pytest.raises(pkg.PlssError):
        pkg.plss_peer_reduce_emulate(t, t, f, list(range(11)))               # > 8 chunks


def _solve(pkg, s, A, peer, slabs, xin=None, weighted=False, maxit=None):
    ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=slabs, maxit_cap=s.maxit,
                               peer=peer, validate=True)
    wi = None
    if weighted:
        wi = pkg.plss_column_norms(ctx)
        pkg.plss_set_wi(ctx, wi)
    q = pkg.plss_query(ctx)
    runs = []
    for _ in range(2):                            # a second solve on the same ctx: epochs continue
        res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), None if xin is None else torch.from_numpy(xin).cuda(),
                             tol=s.tol, maxit=maxit or s.maxit, flags=1 if s.freeze else 0)
        res["xh"] = res["x"].cpu().numpy()
        runs.append(res)
    pkg.plss_destroy(ctx)
    return q, runs, None if wi is None else wi.cpu().numpy()


@pytest.mark.parametrize("name,slabs,weighted,x0", [("C2s", 1, False, False), ("C5xs", 2, False, False),
                                                   ("C4xs", 2, False, False), ("C2s", 2, True, False),
                                                   ("C3_64", 1, False, True)])
def test_dist_peer_step(pkg, name, slabs, weighted, x0):
    """Single rank: the peer reduce is a copy of the partial into the reduced vector, as the NCCL
    single-rank all-reduce is the identity, so the two solves are bitwise equal; parity with the
    oracle as for every distributed solve."""
    s = plss_gen.make_config("C3", N=64) if name == "C3_64" else plss_gen.make_config(name)
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    xin = np.random.default_rng(3).standard_normal(s.n) if x0 else None
    qp, peer, wih = _solve(pkg, s, A, True, slabs, xin, weighted)
    qn, nccl, _ = _solve(pkg, s, A, False, slabs, xin, weighted)
    assert qp["launches_per_step"] > qn["launches_per_step"]           # reduce + wait kernels
    for a in peer + nccl[1:]:
        assert a["iters"] == nccl[0]["iters"] and a["outcome"] == nccl[0]["outcome"]
        np.testing.assert_array_equal(a["xh"], nccl[0]["xh"])
        np.testing.assert_array_equal(a["hist"], nccl[0]["hist"])
    ref = oracle.plss_system(s, x0=xin, wi=wih)
    from test_gpu_parity import _assert_parity, _floor
    _assert_parity(peer[0], ref, _floor(s, ref, x0=xin), s)


def test_dist_peer_profile_then_solve(pkg):
    """plss_profile runs the peer reduce / wait kernels one by one (advancing the epoch the same
    way); a solve afterwards is unchanged."""
    s = plss_gen.make_config("C5xs")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    _, base, _ = _solve(pkg, s, A, True, 2, maxit=40)
    ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=2, maxit_cap=s.maxit, peer=True)
    pkg.plss_start(ctx, torch.from_numpy(s.b).cuda(), tol=0.0, maxit=40, flags=1)
    ms = pkg.plss_profile(ctx, 3)
    assert all(np.isfinite(v) and v >= 0 for v in ms.values())
    res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, maxit=40, flags=1 if s.freeze else 0)
    pkg.plss_destroy(ctx)
    np.testing.assert_array_equal(res["x"].cpu().numpy(), base[0]["xh"])
    np.testing.assert_array_equal(res["hist"], base[0]["hist"])


def test_peer_flag_validation(pkg):
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    with pytest.raises(pkg.PlssError):
        pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, peer=True, rsag=True)
    import ctypes
    from paper_2207_07615_b200.plss import _opts, _alloc_workspace, _aligned
    lib = pkg.load_library()
    ms = A.c_struct()
    o = _opts(peer=True)
    nbytes = pkg.plss_workspace_bytes(A)
    ws = _alloc_workspace(nbytes, "cuda")
    h = ctypes.c_void_p()
    assert lib.plss_create(ctypes.byref(ms), ctypes.byref(o), _aligned(ws), nbytes, None, ctypes.byref(h)) != 0
