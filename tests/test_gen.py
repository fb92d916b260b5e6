"""Input generator checks (plss_gen): CSR/CSC invariants and the config recipes of SURVEY 8(d)."""
import numpy as np
import pytest

import plss_gen


def _check_csr(ptr, idx, nrows, ncols, nnz):
    assert ptr.dtype == np.int32 and idx.dtype == np.int32
    assert ptr[0] == 0 and ptr[-1] == nnz and ptr.shape[0] == nrows + 1
    assert np.all(np.diff(ptr) >= 0)
    assert np.all((idx >= 0) & (idx < ncols))
    # strictly ascending within each segment
    d = np.diff(idx.astype(np.int64))
    seg_start = np.zeros(nnz, bool)
    seg_start[ptr[:-1][ptr[:-1] < nnz]] = True
    assert np.all(d[~seg_start[1:]] > 0)


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5xs"])
def test_invariants_and_transpose(name):
    s = plss_gen.make_config(name)
    _check_csr(s.row_ptr, s.col_idx, s.m, s.n, s.nnz)
    _check_csr(s.col_ptr, s.row_idx, s.n, s.m, s.nnz)
    A = s.scipy_csr()
    T = A.T.tocsr()
    T.sort_indices()
    np.testing.assert_array_equal(T.indptr, s.col_ptr)
    np.testing.assert_array_equal(T.indices, s.row_idx)
    np.testing.assert_array_equal(T.data, s.val_t)
    assert np.all(np.isfinite(s.val)) and s.b.shape == (s.m,)


def test_c1_c2_shapes():
    s = plss_gen.make_config("C1")
    assert (s.m, s.n, s.nnz) == (200, 100, 20000) and s.tol == 1e-10
    s = plss_gen.make_config("C2s")
    assert np.all(np.diff(s.row_ptr) == 8)


def test_c3_structure():
    s = plss_gen.make_config("C3", N=16)
    A = s.scipy_csr().toarray()
    assert np.array_equal(A, A.T)
    d = np.diag(A)
    assert np.all((d >= 4.0) & (d < 4.1))
    assert s.nnz == 5 * 16 * 16 - 4 * 16
    np.testing.assert_allclose(A @ np.ones(s.n), s.b, rtol=0, atol=1e-15)


def test_c3_full_nnz_formula():
    N = 2048
    assert 5 * N * N - 4 * N == 20_963_328          # SURVEY 8(a) C3 nnz


def test_c4_rows_clipped_zipf():
    s = plss_gen.make_config("C4s")
    L = np.diff(s.row_ptr)
    assert L.min() >= 1 and L.max() <= 4096
    assert 3.0 < L.mean() < 6.5                      # Zipf(2.1) clipped: mean ~4.2
    assert (L == 1).mean() > 0.55
    assert np.count_nonzero(s.x_star) == 800


def test_c5_rows_band_plus_uniform():
    s = plss_gen.make_config("C5xs")
    L = np.diff(s.row_ptr)
    assert np.all(L == 12)
    half = 256
    w = 2 * half + 1
    i = np.arange(s.m)
    lo = np.clip(i * s.n // s.m - half, 0, s.n - w)
    cols = s.col_idx.reshape(s.m, 12)
    inband = (cols >= lo[:, None]) & (cols < lo[:, None] + w)
    assert np.all(inband.sum(axis=1) >= 6)
    assert s.freeze and s.tol == 0.0


def test_row_blocks_cover_rows():
    s = plss_gen.make_config("C5xs")
    G = 4
    total = 0
    for g in range(G):
        blk = plss_gen.row_block(s, G, g)
        r0, r1 = plss_gen.row_block_bounds(s.m, G, g)
        assert blk["row_offset"] == r0 and blk["m"] == r1 - r0
        _check_csr(blk["row_ptr"], blk["col_idx"], blk["m"], s.n, blk["col_idx"].shape[0])
        _check_csr(blk["col_ptr"], blk["row_idx"], s.n, blk["m"], blk["col_idx"].shape[0])
        total += blk["col_idx"].shape[0]
    assert total == s.nnz


def test_bytes_per_iter_model():
    # B_iter = 24 nnz + 28 m + 68 n (+8); the fused one-device flow (R25) 16 n less
    assert plss_gen.bytes_per_iter(64_000_000, 8_000_000, 768_000_000) == \
        24 * 768_000_000 + 28 * 64_000_000 + 68 * 8_000_000 + 8
    assert plss_gen.bytes_per_iter(5, 7, 11) - plss_gen.bytes_per_iter_fused(5, 7, 11) == 16 * 7
