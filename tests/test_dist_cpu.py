"""World-size-2 gloo test (CPU) of the row-block path's host logic and decomposition."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import plss_gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _run(world, cfg, tmp_path, chunks=1, rsag=False, cols=False, maxit=0):
    out = tmp_path / f"res_{world}_{chunks}_{int(rsag)}_{int(cols)}.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), "--backend", "gloo", "--out", str(out),
           "--config", cfg, "--chunks", str(chunks)] + (["--rsag"] if rsag else []) + (["--cols"] if cols else []) + ["--maxit", str(maxit)]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="1")
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT, env=env, capture_output=True)
    return np.load(out)


def test_row_blocks_world2_match_oracle(tmp_path):
    s = plss_gen.make_config("C2s")
    ref = oracle.plss_system(s)
    r = _run(2, "C2s", tmp_path)
    assert abs(int(r["iters"]) - ref["iters"]) <= max(1, int(np.ceil(0.02 * ref["iters"])))
    k = min(50, len(ref["hist"]))
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9
    assert np.linalg.norm(r["x"] - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-7


def test_row_blocks_world2_chunked_allreduce_bitwise(tmp_path):
    """The chunked all-reduce (the distributed ctx's PLSS_DIST_CHUNKS path) sums every element of
    the (n+1) buffer exactly as the single all-reduce does: bitwise the same solve, two ranks."""
    a = _run(2, "C2s", tmp_path, chunks=1)
    b = _run(2, "C2s", tmp_path, chunks=4)
    assert int(a["iters"]) == int(b["iters"])
    np.testing.assert_array_equal(a["hist"], b["hist"])
    np.testing.assert_array_equal(a["x"], b["x"])


def test_row_blocks_world2_reduce_scatter_step(tmp_path):
    """The reduce-scatter / all-gather decomposition (options.flags bit2) with two ranks: each owns
    a 32-aligned column shard of y, p, x; the scalars are shard partials in one all-reduce."""
    s = plss_gen.make_config("C2s")
    ref = oracle.plss_system(s)
    r = _run(2, "C2s", tmp_path, rsag=True)
    assert abs(int(r["iters"]) - ref["iters"]) <= max(1, int(np.ceil(0.02 * ref["iters"])))
    k = min(50, len(ref["hist"]))
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-9
    assert np.linalg.norm(r["x"] - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-7


@pytest.mark.parametrize("cfg,maxit", [("C2s", 0), ("C4xs", 60)])
def test_column_blocks_world2_match_oracle(tmp_path, cfg, maxit):
    """The column-block decomposition (plss_create_dist_cols) with two ranks: a full solve (C2s) and
    the first 60 steps of the underdetermined power-law system (C4xs: m < n, where the all-reduce of
    m + 1 values is the smaller message; its full solve takes ~5.5k ill-conditioned steps whose
    count moves with rounding)."""
    s = plss_gen.make_config(cfg)
    if maxit:
        s.maxit = maxit
    ref = oracle.plss_system(s)
    r = _run(2, cfg, tmp_path, cols=True, maxit=maxit)
    from test_gpu_parity import _assert_parity, _floor          # the floor-aware bars
    res = {"hist": r["hist"], "xh": r["x"], "iters": int(r["iters"]),
           "outcome": "maxit" if int(r["iters"]) >= s.maxit else "converged"}
    _assert_parity(res, ref, _floor(s, ref), s)


def test_column_block_slices():
    s = plss_gen.make_config("C2s")
    A = s.scipy_csr().toarray()
    for G in (1, 3):
        for g in range(G):
            blk = plss_gen.col_block(s, G, g)
            c0 = blk["col_offset"]
            d = np.zeros((s.m, blk["n"]))
            for i in range(s.m):
                for k in range(blk["row_ptr"][i], blk["row_ptr"][i + 1]):
                    d[i, blk["col_idx"][k]] = blk["val"][k]
            np.testing.assert_array_equal(d, A[:, c0:c0 + blk["n"]])
            assert np.all(np.diff(blk["row_ptr"]) >= 0)


def test_row_block_bounds_partition():
    for m in (0, 1, 7, 64_000_000):
        for G in (1, 2, 4, 8):
            b = [plss_gen.row_block_bounds(m, G, g) for g in range(G)]
            assert b[0][0] == 0 and b[-1][1] == m
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
