"""Distributed (row-block) path of libplss on the GPU.

With one GPU the dist ctx runs with nranks = 1: the same code path (K1 publishing the local rho,
K2 writing the local y, ncclAllReduce of n+1 doubles, the dots/tail kernel) over a real
single-rank NCCL communicator. With >= 2 GPUs, `test_two_ranks_torchrun` launches 2 ranks.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import plss_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.fixture(scope="module")
def pkg():
    from paper_2207_07615_b200 import build as pbuild
    pbuild.build()
    import paper_2207_07615_b200 as p
    p.load_library()
    return p


def _dist_solve(pkg, s, slabs=1, **kw):
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    uid = pkg.plss_get_unique_id()
    args = dict(tol=s.tol, tol_mode=s.tol_mode, maxit=s.maxit, flags=1 if s.freeze else 0)
    args.update(kw)
    ctx = pkg.plss_create_dist(A, 0, s.m, uid, 0, 1, slabs=slabs, maxit_cap=args["maxit"], validate=True)
    # K1 + K2 per slab, K3, the dots kernel; the last K2 may run as up to 4 column chunks
    assert 2 * slabs + 2 <= pkg.plss_query(ctx)["launches_per_step"] <= 2 * slabs + 5
    res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), **args)
    res["xh"] = res["x"].cpu().numpy()
    pkg.plss_destroy(ctx)
    return res


@pytest.mark.parametrize("name,slabs", [("C1", 1), ("C2s", 1), ("C2s", 3), ("C5xs", 2)])
def test_dist_single_rank_parity(pkg, name, slabs):
    s = plss_gen.make_config(name)
    ref = oracle.plss_system(s)
    res = _dist_solve(pkg, s, slabs=slabs)
    assert res["outcome"] == ref["outcome"]
    assert abs(res["iters"] - ref["iters"]) <= max(1, int(np.ceil(0.02 * ref["iters"])))
    k = min(25, len(ref["hist"]), len(res["hist"]))
    assert np.max(np.abs(res["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9
    assert np.linalg.norm(res["xh"] - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-7


def test_dist_zero_rhs(pkg):
    s = plss_gen.make_config("C2s")
    s.b = np.zeros(s.m)
    res = _dist_solve(pkg, s)
    assert res["iters"] == 0 and res["outcome"] == "converged"


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", ["allreduce", "rsag", "peer", "cols"])
def test_two_ranks_torchrun(tmp_path, mode):
    """Two ranks on two GPUs: every distributed step (the chunked NCCL all-reduce, the reduce-scatter
    step, the peer-memory step over CUDA IPC, the column-block partition); the worker also checks
    that both ranks hold bitwise the same x and per-iteration scalars."""
    script = os.path.join(ROOT, "tests", "dist_worker.py")
    out = tmp_path / "res.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), script, "--backend", "nccl",
           "--out", str(out), "--config", "C5xs"] + ([] if mode == "allreduce" else [f"--{mode}"])
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT)
    r = np.load(out)
    s = plss_gen.make_config("C5xs")
    ref = oracle.plss_system(s)
    k = 25
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9
    assert np.linalg.norm(r["x"] - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-7


def test_dist_single_rank_plssw(pkg):
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=2, maxit_cap=s.maxit)
    c = pkg.plss_column_norms(ctx)
    c_ref = oracle.column_norms(s.n, s.col_ptr, s.val_t)
    np.testing.assert_array_equal(c.cpu().numpy(), c_ref)
    pkg.plss_set_wi(ctx, c)
    res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, maxit=s.maxit)
    ref = oracle.plss_system(s, wi=c_ref)
    pkg.plss_destroy(ctx)
    assert res["outcome"] == ref["outcome"]
    assert abs(res["iters"] - ref["iters"]) <= max(1, int(np.ceil(0.02 * ref["iters"])))
    k = min(25, len(ref["hist"]), len(res["hist"]))
    assert np.max(np.abs(res["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9
    assert np.linalg.norm(res["x"].cpu().numpy() - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-7


def test_dist_ctx_rejects_single_device_methods(pkg):
    """Randomized projection, PLSS Kaczmarz and the growing-sketch engine run on single-device
    ctxs only (include/plss.h): a distributed ctx reports E_INVALID with a message, and its PLSS
    solve still works afterwards."""
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, maxit_cap=100)
    for call in (lambda: pkg.plss_rp_solve(ctx, s.b, r=4, maxit=3),
                 lambda: pkg.plss_kz_solve(ctx, s.b, np.arange(3), maxit=3),
                 lambda: pkg.plss_eg_solve(ctx, s.b, sketch="residual", maxit=3)):
        with pytest.raises(pkg.PlssError):
            call()
    out = pkg.plss_solve(ctx, s.b, tol=1e-6, maxit=100)
    assert out["outcome"] in ("converged", "maxit") and out["iters"] > 0
    pkg.plss_destroy(ctx)


@pytest.mark.parametrize("name", ["C5xs", "C2s"])
def test_dist_chunked_allreduce_bitwise(pkg, name):
    """The last K2 segment in column chunks, each all-reduced on a second stream while the next
    computes (PLSS_DIST_CHUNKS): every y element is the same sequential sum plus the same NCCL
    sum, so the solve is bitwise the unchunked one; the launch count shows the chunks engaged."""
    s = plss_gen.make_config(name)            # both have sigma-sorted K2 slices (chunkable)
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    out = {}
    for ch in ("1", "4"):
        old = os.environ.get("PLSS_DIST_CHUNKS")
        os.environ["PLSS_DIST_CHUNKS"] = ch
        try:
            ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=2, maxit_cap=s.maxit)
        finally:
            if old is None:
                os.environ.pop("PLSS_DIST_CHUNKS")
            else:
                os.environ["PLSS_DIST_CHUNKS"] = old
        q = pkg.plss_query(ctx)
        res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), tol=s.tol, maxit=min(s.maxit, 200),
                             flags=1 if s.freeze else 0)
        out[ch] = (q["launches_per_step"], res["x"].cpu().numpy(), res["hist"], res["iters"])
        pkg.plss_destroy(ctx)
    assert out["4"][0] > out["1"][0], (out["4"][0], out["1"][0])      # chunks engaged
    assert out["4"][3] == out["1"][3]
    np.testing.assert_array_equal(out["4"][1], out["1"][1])
    np.testing.assert_array_equal(out["4"][2], out["1"][2])


def test_dist_true_residual(pkg):
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, maxit_cap=s.maxit)
    res = pkg.plss_solve(ctx, s.b, tol=s.tol, maxit=s.maxit)
    t = pkg.plss_true_residual(ctx, s.b, res["x"])
    x = res["x"].cpu().numpy()
    ref = np.linalg.norm(s.b - oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, x)) / np.linalg.norm(s.b)
    pkg.plss_destroy(ctx)
    assert abs(t["rel"] - ref) <= 1e-12


@pytest.mark.parametrize("name,slabs,weighted,x0", [("C2s", 1, False, False), ("C5xs", 2, False, False),
                                                   ("C4xs", 2, False, False), ("C2s", 2, True, False),
                                                   ("C3_64", 1, False, True)])
def test_dist_reduce_scatter_step(pkg, name, slabs, weighted, x0):
    """options.flags bit2 (the reduce-scatter / all-gather step, SURVEY 8e improvement 2) on a
    single rank: parity with the oracle (the shard is the whole vector; the dots are shard partials
    summed by the all-reduce), and agreement with the all-reduce step over the live iterations."""
    s = plss_gen.make_config("C3", N=64) if name == "C3_64" else plss_gen.make_config(name)
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    xin = np.random.default_rng(3).standard_normal(s.n) if x0 else None
    out = {}
    for rsag in (True, False):
        ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=slabs, maxit_cap=s.maxit,
                                   rsag=rsag, validate=True)
        wi = None
        if weighted:
            wi = pkg.plss_column_norms(ctx)
            pkg.plss_set_wi(ctx, wi)
        res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), None if xin is None else torch.from_numpy(xin).cuda(),
                             tol=s.tol, maxit=s.maxit, flags=1 if s.freeze else 0)
        res["xh"] = res["x"].cpu().numpy()
        out[rsag] = (res, None if wi is None else wi.cpu().numpy())
        pkg.plss_destroy(ctx)
    res, wih = out[True]
    ref = oracle.plss_system(s, x0=xin, wi=wih)
    from test_gpu_parity import _assert_parity, _floor, HIST_TOL
    fl = _floor(s, ref, x0=xin)
    _assert_parity(res, ref, fl, s)
    h1, h0 = res["hist"], out[False][0]["hist"]
    k = min(len(h1), len(h0), 25, fl["kf"])                    # within the fp64 floor
    live = h0[:k] > 1e-10
    assert np.max(np.abs(h1[:k] - h0[:k])[live] / h0[:k][live]) <= HIST_TOL


def test_reduce_scatter_needs_dist(pkg):
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    import ctypes
    lib = pkg.load_library()
    from paper_2207_07615_b200.plss import _opts, _alloc_workspace, _aligned
    ms = A.c_struct()
    o = _opts(rsag=True)
    nbytes = pkg.plss_workspace_bytes(A)
    ws = _alloc_workspace(nbytes, "cuda")
    h = ctypes.c_void_p()
    assert lib.plss_create(ctypes.byref(ms), ctypes.byref(o), _aligned(ws), nbytes, None, ctypes.byref(h)) != 0


@pytest.mark.parametrize("name,slabs,weighted,x0", [("C2s", 1, False, False), ("C5xs", 2, False, False),
                                                   ("C4xs", 1, False, False), ("C2s", 2, True, False),
                                                   ("C3_64", 1, False, True)])
def test_dist_column_block_step(pkg, name, slabs, weighted, x0):
    """plss_create_dist_cols (the column-block partition) on a single rank: the block is
    the whole matrix; K1 into u, all-reduce of u | theta, replicated rho tail, K2 over the local
    columns, phi / psi all-reduce, shard K3. Parity with the oracle, agreement with the row-block
    step over the live iterations, and the true residual of its x."""
    s = plss_gen.make_config("C3", N=64) if name == "C3_64" else plss_gen.make_config(name)
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    xin = np.random.default_rng(3).standard_normal(s.n) if x0 else None
    out = {}
    for cols in (True, False):
        mk = pkg.plss_create_dist_cols if cols else pkg.plss_create_dist
        ctx = mk(A, 0, s.n if cols else s.m, pkg.plss_get_unique_id(), 0, 1, slabs=slabs, maxit_cap=s.maxit,
                 validate=True)
        if cols:
            S = pkg.plss_query(ctx)["slabs"]
            qs = [pkg.plss_query_segment(ctx, w, sl) for w in (1, 2) for sl in range(S)]
            extra = sum(1 for q in qs if q["fmt"] == 3 and q["nlong"] > 0 and not q["lin"])  # a long-row launch
            assert pkg.plss_query(ctx)["launches_per_step"] == 2 * S + 4 + extra
        wi = None
        if weighted:
            wi = pkg.plss_column_norms(ctx)
            pkg.plss_set_wi(ctx, wi)
        res = pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda(), None if xin is None else torch.from_numpy(xin).cuda(),
                             tol=s.tol, maxit=s.maxit, flags=1 if s.freeze else 0)
        res["xh"] = res["x"].cpu().numpy()
        if cols:
            t = pkg.plss_true_residual(ctx, s.b, res["x"])
            ref_t = np.linalg.norm(s.b - oracle.spmv(s.m, s.row_ptr, s.col_idx, s.val, res["xh"]))
            assert abs(t["abs"] - ref_t) <= 1e-12 * max(ref_t, np.linalg.norm(s.b))
        out[cols] = (res, None if wi is None else wi.cpu().numpy())
        pkg.plss_destroy(ctx)
    res, wih = out[True]
    if weighted:
        np.testing.assert_array_equal(wih, out[False][1])          # whole columns: same norms
    ref = oracle.plss_system(s, x0=xin, wi=wih)
    from test_gpu_parity import _assert_parity, _floor, HIST_TOL
    fl = _floor(s, ref, x0=xin)
    _assert_parity(res, ref, fl, s)
    h1, h0 = res["hist"], out[False][0]["hist"]
    k = min(len(h1), len(h0), 25, fl["kf"])                    # within the fp64 floor
    live = h0[:k] > 1e-10
    assert np.max(np.abs(h1[:k] - h0[:k])[live] / h0[:k][live]) <= HIST_TOL


def test_column_block_rejects_row_block_steps(pkg):
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    import ctypes
    from paper_2207_07615_b200.plss import _opts, _alloc_workspace, _aligned
    lib = pkg.load_library()
    ms = A.c_struct()
    nbytes = pkg.plss_workspace_bytes(A)
    ws = _alloc_workspace(nbytes, "cuda")
    uid = pkg.plss_get_unique_id()
    for o in (_opts(rsag=True), _opts(peer=True)):
        h = ctypes.c_void_p()
        assert lib.plss_create_dist_cols(ctypes.byref(ms), 0, s.n, uid, 0, 1, ctypes.byref(o), _aligned(ws), nbytes,
                                         None, ctypes.byref(h)) != 0
    with pytest.raises(pkg.PlssError):                      # block outside the global matrix
        pkg.plss_create_dist_cols(A, 1, s.n, uid, 0, 1)


def test_dist_nccl_failure_aborts_communicator(pkg, monkeypatch):
    """SURVEY 5 failure detection: while a distributed solve waits it polls
    ncclCommGetAsyncError; an error aborts the communicator (ncclCommAbort), the call fails with
    PLSS_E_NCCL instead of hanging, every later call on the ctx fails the same way, and the ctx
    can still be destroyed. The error is injected (PLSS_FAULT_NCCL=1 at ctx creation): a real one
    needs a second rank to die."""
    s = plss_gen.make_config("C2s")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    monkeypatch.setenv("PLSS_FAULT_NCCL", "1")
    ctx = pkg.plss_create_dist(A, 0, s.m, pkg.plss_get_unique_id(), 0, 1, slabs=2, maxit_cap=s.maxit)
    monkeypatch.delenv("PLSS_FAULT_NCCL")
    b = torch.from_numpy(s.b).cuda()
    with pytest.raises(pkg.PlssError, match="NCCL asynchronous error.*aborted"):
        pkg.plss_solve(ctx, b, tol=s.tol, maxit=s.maxit)
    with pytest.raises(pkg.PlssError, match="aborted"):
        pkg.plss_solve(ctx, b, tol=s.tol, maxit=s.maxit)
    with pytest.raises(pkg.PlssError, match="aborted"):
        pkg.plss_step(ctx, 1)
    pkg.plss_destroy(ctx)
    # a fresh ctx without the fault solves normally on the same device
    res = _dist_solve(pkg, s, slabs=2)
    assert res["outcome"] == "converged"


def test_binding_rejects_bad_device_vectors(pkg):
    s = plss_gen.make_config("C1")
    A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
    ctx = pkg.plss_create(A, maxit_cap=4)
    buf = torch.zeros(s.m + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(pkg.PlssError, match="CUDA tensor"):
        pkg.plss_spmv(ctx, np.zeros(s.n), buf[:s.m])
    with pytest.raises(pkg.PlssError, match="required"):
        pkg.plss_spmv(ctx, torch.zeros(s.n - 1, dtype=torch.float64, device="cuda"), buf[:s.m])
    with pytest.raises(pkg.PlssError, match="float64"):
        pkg.plss_solve(ctx, torch.from_numpy(s.b).cuda().float(), maxit=2)
    pkg.plss_destroy(ctx)
