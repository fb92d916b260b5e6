"""World-size-2 gloo test (CPU) of the row-block path's host logic and decomposition."""
import os
import socket
import subprocess
import sys

import numpy as np

import oracle
import plss_gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _run(world, cfg, tmp_path, chunks=1, rsag=False):
    out = tmp_path / f"res_{world}_{chunks}_{int(rsag)}.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), "--backend", "gloo", "--out", str(out),
           "--config", cfg, "--chunks", str(chunks)] + (["--rsag"] if rsag else [])
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


def test_row_block_bounds_partition():
    for m in (0, 1, 7, 64_000_000):
        for G in (1, 2, 4, 8):
            b = [plss_gen.row_block_bounds(m, G, g) for g in range(G)]
            assert b[0][0] == 0 and b[-1][1] == m
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
