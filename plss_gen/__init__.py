"""Seeded synthetic inputs for the PLSS hot path (shared by the oracle tests and the CUDA path).

This module holds NO arithmetic of the method (Algorithm 1). It only builds
the linear system A x = b that BASELINE.json's configs describe:

* CSR arrays (row_ptr int32[m+1], col_idx int32[nnz] strictly ascending per row, val f64[nnz]);
* the CSC copy (col_ptr int32[n+1], row_idx int32[nnz] strictly ascending per column,
  val_t f64[nnz]) by a stable counting transpose (pure index work);
* x* and b = A x* (b computed with scipy.sparse, a library product - input synthesis, not the
  method), tolerance / tolerance mode / iteration cap per config.

The paper's workloads are SuiteSparse / LIBSVM matrices that are not in the
container; C2-C5 stand in for them by shape, density and structure.

Generator recipes follow SURVEY.md 8(d) "Configs as concrete synthetic inputs":
numpy.random.default_rng(seed) (PCG64), draws in the order listed. The full-size C5
(768M nnz) is additionally available on a CUDA device through torch's Philox generator
(`make_c5_torch`); its stream differs from the numpy one, so each (config, backend) pair is its
own deterministic input.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "System", "make_config", "csr_to_csc", "CONFIGS", "row_block_bounds", "row_block",
    "c1_dense", "c2_random", "c3_laplace", "c4_powerlaw", "c5_banded", "make_c5_torch",
    "from_dense", "bytes_per_iter",
]


@dataclasses.dataclass
class System:
    """One consistent sparse system A x = b with both storage orders of A."""
    name: str
    m: int
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray
    col_ptr: np.ndarray
    row_idx: np.ndarray
    val_t: np.ndarray
    b: np.ndarray
    x_star: Optional[np.ndarray]
    tol: float
    tol_mode: int          # 0 relative ||r||/||b||, 1 absolute ||r||
    maxit: int
    freeze: bool = False   # fixed-iteration timing mode
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def scipy_csr(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col_idx, self.row_ptr), shape=(self.m, self.n))


def bytes_per_iter(m: int, n: int, nnz: int) -> int:
    """Algorithmic HBM bytes of one iteration: 24 nnz + 28 m + 68 n (+8).

    K1: 12 nnz + 4(m+1) + 8n + 16m;  K2: 12 nnz + 4(n+1) + 8m + 8n + 8n;  K3: 40n.
    """
    return 24 * nnz + 28 * m + 68 * n + 8


def bytes_per_iter_fused(m: int, n: int, nnz: int) -> int:
    """The bytes the one-device PLSS step's own data flow needs (R25): SURVEY 8(d)'s
    B_iter less K2's p read for psi (summed in K3 from the p it reads anyway, 8n) and half of K3's
    x read + write (x updated every other step, 8n on average): 24 nnz + 28 m + 52 n (+8)."""
    return 24 * nnz + 28 * m + 52 * n + 8


# ----------------------------------------------------------------------------------------------
# index plumbing
# ----------------------------------------------------------------------------------------------

def csr_to_csc(m: int, n: int, row_ptr: np.ndarray, col_idx: np.ndarray, val: np.ndarray):
    """Stable transpose: entries of each column keep ascending row order (counting sort)."""
    nnz = col_idx.shape[0]
    counts = np.bincount(col_idx, minlength=n).astype(np.int64)
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    order = np.argsort(col_idx, kind="stable")
    rows = np.repeat(np.arange(m, dtype=np.int32), np.diff(row_ptr).astype(np.int64))
    row_idx = rows[order].astype(np.int32, copy=False)
    val_t = val[order]
    assert col_ptr[-1] == nnz
    return col_ptr.astype(np.int32), row_idx, np.ascontiguousarray(val_t)


def _finish(name, m, n, row_ptr, col_idx, val, x_star, tol, tol_mode, maxit, b=None,
            freeze=False, meta=None) -> System:
    import scipy.sparse as sp
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    if b is None:
        A = sp.csr_matrix((val, col_idx, row_ptr), shape=(m, n))
        b = np.ascontiguousarray(A @ x_star, dtype=np.float64)
    col_ptr, row_idx, val_t = csr_to_csc(m, n, row_ptr, col_idx, val)
    return System(name, m, n, row_ptr, col_idx, val, col_ptr, row_idx, val_t, b, x_star,
                  tol, tol_mode, maxit, freeze, dict(meta or {}))


def from_dense(A: np.ndarray, b: np.ndarray, name="dense", tol=1e-10, tol_mode=0, maxit=None,
               keep_zeros=False, x_star=None) -> System:
    """Dense matrix -> CSR/CSC system (zero entries dropped unless keep_zeros)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    mask = np.ones_like(A, dtype=bool) if keep_zeros else (A != 0)
    counts = mask.sum(axis=1)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    rr, cc = np.nonzero(mask)
    return _finish(name, m, n, row_ptr, cc, A[rr, cc], x_star, tol, tol_mode,
                   maxit if maxit is not None else max(1, min(m, n) * 4),
                   b=np.ascontiguousarray(b, dtype=np.float64))


def _distinct_rows(rng, draw, nrows, width):
    """Draw (nrows, width) int columns with `draw(k)`; redraw rows holding duplicates."""
    cols = np.sort(draw(np.arange(nrows)), axis=1)
    while True:
        dup = np.nonzero((cols[:, 1:] == cols[:, :-1]).any(axis=1))[0]
        if dup.size == 0:
            return cols
        cols[dup] = np.sort(draw(dup), axis=1)


# ----------------------------------------------------------------------------------------------
# configs (BASELINE.json "configs")
# ----------------------------------------------------------------------------------------------

def c1_dense(seed=0, m=200, n=100) -> System:
    """C1: dense N(0,1) 200x100 stored as CSR; x* N(0,1); b = A x*; rel tol 1e-10, maxit 100."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n))
    x_star = rng.standard_normal(n)
    row_ptr = np.arange(0, m * n + 1, n, dtype=np.int64)
    col_idx = np.tile(np.arange(n, dtype=np.int32), m)
    return _finish(f"C1[{m}x{n}]", m, n, row_ptr, col_idx, A.reshape(-1), x_star,
                   1e-10, 0, 100, b=np.ascontiguousarray(A @ x_star))


def c2_random(seed=0, m=200_000, n=100_000, per_row=8) -> System:
    """C2: 8 distinct uniform columns per row, N(0,1) values; rel tol 1e-8, maxit 20000."""
    rng = np.random.default_rng(seed)
    cols = _distinct_rows(rng, lambda rows: rng.integers(0, n, (rows.size, per_row)), m, per_row)
    val = rng.standard_normal(m * per_row)
    x_star = rng.standard_normal(n)
    row_ptr = np.arange(0, m * per_row + 1, per_row, dtype=np.int64)
    return _finish(f"C2[{m}x{n}]", m, n, row_ptr, cols.reshape(-1), val, x_star, 1e-8, 0, 20_000)


def c3_laplace(seed=0, N=2048) -> System:
    """C3: 5-point Dirichlet Laplacian-like on an N x N grid, natural order idx = i*N + j.

    diagonal 4 + 0.1*U(0,1), -1 to each existing N/S/E/W neighbour; b = A 1; rel 1e-8.
    """
    rng = np.random.default_rng(seed)
    nn = N * N
    diag = 4.0 + 0.1 * rng.random(nn)
    idx = np.arange(nn, dtype=np.int64)
    i, j = idx // N, idx % N
    # neighbours in ascending column order: north (idx-N), west (idx-1), self, east, south
    cand = np.stack([idx - N, idx - 1, idx, idx + 1, idx + N], axis=1)
    ok = np.stack([i > 0, j > 0, np.ones(nn, bool), j < N - 1, i < N - 1], axis=1)
    vals = np.where(cand == idx[:, None], diag[:, None], -1.0)
    counts = ok.sum(axis=1)
    row_ptr = np.zeros(nn + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return _finish(f"C3[{N}^2]", nn, nn, row_ptr, cand[ok], vals[ok], np.ones(nn),
                   1e-8, 0, 20_000, meta={"grid": N})


def c4_powerlaw(seed=0, m=2_000_000, n=8_000_000, alpha=2.1, clip=4096, support=80_000) -> System:
    """C4: row lengths min(zipf(alpha), clip), distinct uniform columns, U(-1,1) values,
    sparse x* (support indices without replacement, N(0,1)); underdetermined; rel 1e-6."""
    rng = np.random.default_rng(seed)
    L = np.minimum(rng.zipf(alpha, m), min(clip, n)).astype(np.int64)
    nnz = int(L.sum())
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(L, out=row_ptr[1:])
    rows = np.repeat(np.arange(m, dtype=np.int64), L)
    cols = rng.integers(0, n, nnz)
    while True:  # rejection: redraw entries colliding with an earlier entry of the same row
        key = rows * n + cols
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = order[1:][ks[1:] == ks[:-1]]
        if dup.size == 0:
            break
        cols[dup] = rng.integers(0, n, dup.size)
    key = rows * n + cols
    cols = (np.sort(key) - rows * n)  # rows are already grouped; sort columns within rows
    val = rng.uniform(-1.0, 1.0, nnz)
    x_star = np.zeros(n)
    sup = rng.choice(n, min(support, n), replace=False)
    x_star[sup] = rng.standard_normal(sup.size)
    return _finish(f"C4[{m}x{n},a={alpha}]", m, n, row_ptr, cols, val, x_star, 1e-6, 0, 20_000,
                   meta={"alpha": alpha})


def c5_banded(seed=0, m=64_000_000, n=8_000_000, band=6, unif=6, half=1024, maxit=500) -> System:
    """C5: 12 entries per row: 6 distinct in the shifted window [lo_i, lo_i + 2*half] with
    lo_i = clip(i*n//m - half, 0, n - 2*half - 1), plus 6 distinct uniform columns not colliding;
    N(0,1) values, x* N(0,1), b = A x*; tol 0 with fixed iterations in freeze mode."""
    rng = np.random.default_rng(seed)
    w = min(2 * half + 1, n)
    c = (np.arange(m, dtype=np.int64) * n) // m
    lo = np.clip(c - half, 0, n - w)

    def draw(rows):
        bcols = lo[rows, None] + rng.integers(0, w, (rows.size, band))
        ucols = rng.integers(0, n, (rows.size, unif))
        return np.concatenate([bcols, ucols], axis=1)

    per = band + unif
    cols = _distinct_rows(rng, draw, m, per)
    val = rng.standard_normal(m * per)
    x_star = rng.standard_normal(n)
    row_ptr = np.arange(0, m * per + 1, per, dtype=np.int64)
    return _finish(f"C5[{m}x{n}]", m, n, row_ptr, cols.reshape(-1), val, x_star, 0.0, 0, maxit,
                   freeze=True)


def make_c5_torch(device="cuda", seed=0, m=64_000_000, n=8_000_000, band=6, unif=6, half=1024,
                  rows=None, chunk=1_000_000):
    """Full-size C5 generated on a device with torch's Philox stream (same recipe as
    `c5_banded`, different stream). Rows are drawn in chunks of `chunk` rows, chunk c from its
    own generator seeded (seed, c), so any row block [r0, r1) aligned to chunks (every
    m/G block for G in 1, 2, 4, 8) is generated identically on its own by the rank that owns
    it. Returns a dict of torch tensors on `device` for the row block `rows` (default all):
    row_ptr, col_idx, val (local CSR), col_ptr, row_idx, val_t (local CSC over all n columns),
    b (local), x_star (full n), plus m, n, row_offset, m_global."""
    import torch
    r0, r1 = (0, m) if rows is None else rows
    assert r0 % chunk == 0 and (r1 % chunk == 0 or r1 == m), "row block must align to chunks"
    per = band + unif
    w = min(2 * half + 1, n)
    gx = torch.Generator(device=device)
    gx.manual_seed(seed * 1_000_003 + 999_999)
    x_star = torch.randn(n, generator=gx, device=device, dtype=torch.float64)
    ml = r1 - r0
    col_idx = torch.empty(ml * per, dtype=torch.int32, device=device)
    val = torch.empty(ml * per, dtype=torch.float64, device=device)
    b = torch.empty(ml, dtype=torch.float64, device=device)
    for c0 in range(r0, r1, chunk):
        c1 = min(r1, c0 + chunk)
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + c0 // chunk)
        rws = torch.arange(c0, c1, device=device, dtype=torch.int64)
        lo = torch.clamp(rws * n // m - half, 0, n - w)

        def draw(k, lo_k):
            bc = lo_k[:, None] + torch.randint(0, w, (k, band), generator=g, device=device)
            uc = torch.randint(0, n, (k, unif), generator=g, device=device)
            return torch.sort(torch.cat([bc, uc], dim=1), dim=1).values

        cols = draw(c1 - c0, lo)
        while True:
            dup = torch.nonzero((cols[:, 1:] == cols[:, :-1]).any(dim=1)).flatten()
            if dup.numel() == 0:
                break
            cols[dup] = draw(dup.numel(), lo[dup])
        seg = slice((c0 - r0) * per, (c1 - r0) * per)
        col_idx[seg] = cols.reshape(-1).to(torch.int32)
        v = torch.randn((c1 - c0) * per, generator=g, device=device, dtype=torch.float64)
        val[seg] = v
        # b = A x* for these rows (input synthesis, library product)
        b[c0 - r0:c1 - r0] = (v * x_star[cols.reshape(-1)]).view(c1 - c0, per).sum(dim=1)
        del cols, rws, lo, v
    row_ptr = torch.arange(0, ml * per + 1, per, device=device, dtype=torch.int32)
    # stable transpose on device (index work only)
    order = torch.sort(col_idx, stable=True).indices
    row_idx = torch.div(order, per, rounding_mode="floor").to(torch.int32)
    val_t = val[order]
    del order
    counts = torch.bincount(col_idx, minlength=n)
    col_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=col_ptr[1:])
    return {"m": ml, "n": n, "row_offset": r0, "m_global": m, "row_ptr": row_ptr,
            "col_idx": col_idx, "val": val, "col_ptr": col_ptr.to(torch.int32), "row_idx": row_idx,
            "val_t": val_t, "b": b, "x_star": x_star}


# name -> (factory, kwargs). "s" suffixes are scaled versions for parity tests on CPU time.
CONFIGS = {
    "C1": (c1_dense, {}),
    "C2": (c2_random, {}),
    "C3": (c3_laplace, {}),
    "C4": (c4_powerlaw, {}),
    "C4alt": (c4_powerlaw, {"alpha": 1.845}),
    "C5": (c5_banded, {}),
    # scaled (oracle finishes in seconds; still many tiles and ragged tails)
    "C2s": (c2_random, {"m": 20_000, "n": 10_000}),
    "C3s": (c3_laplace, {"N": 256}),
    "C4s": (c4_powerlaw, {"m": 20_000, "n": 80_000, "support": 800}),
    "C4xs": (c4_powerlaw, {"m": 2_000, "n": 8_000, "support": 80}),
    "C5s": (c5_banded, {"m": 640_000, "n": 80_000, "maxit": 60}),
    "C5xs": (c5_banded, {"m": 64_000, "n": 8_000, "half": 256, "maxit": 60}),
}


def make_config(name: str, seed: int = 0, **overrides) -> System:
    fn, kw = CONFIGS[name]
    kw = dict(kw)
    kw.update(overrides)
    return fn(seed=seed, **kw)


# ----------------------------------------------------------------------------------------------
# row-block sharding: GPU g owns rows [g*m/G, (g+1)*m/G)
# ----------------------------------------------------------------------------------------------

def row_block_bounds(m: int, G: int, g: int):
    return (g * m) // G, ((g + 1) * m) // G


def row_block(sysm: System, G: int, g: int) -> dict:
    """Local CSR + CSC (over all n columns) of row block g, rows rebased to 0."""
    r0, r1 = row_block_bounds(sysm.m, G, g)
    a, e = int(sysm.row_ptr[r0]), int(sysm.row_ptr[r1])
    rp = (sysm.row_ptr[r0:r1 + 1] - a).astype(np.int32)
    ci = sysm.col_idx[a:e]
    v = sysm.val[a:e]
    cp, ri, vt = csr_to_csc(r1 - r0, sysm.n, rp, ci, v)
    return {"row_offset": r0, "m": r1 - r0, "n": sysm.n, "row_ptr": rp, "col_idx": ci, "val": v,
            "col_ptr": cp, "row_idx": ri, "val_t": vt, "b": sysm.b[r0:r1]}


def col_block(sysm: System, G: int, g: int) -> dict:
    """Column block g (columns [c0, c1) = row_block_bounds(n, G, g)) as an m x (c1 - c0) matrix:
    its CSC slice (rows global) and the CSR over local column indices; b is the full right-hand side
    (replicated in the column-block partition)."""
    c0, c1 = row_block_bounds(sysm.n, G, g)
    a, e = int(sysm.col_ptr[c0]), int(sysm.col_ptr[c1])
    cp = (sysm.col_ptr[c0:c1 + 1] - a).astype(np.int32)
    ri = sysm.row_idx[a:e]
    vt = sysm.val_t[a:e]
    rp, ci, v = csr_to_csc(c1 - c0, sysm.m, cp, ri, vt)       # the transpose of a CSC is its CSR
    return {"col_offset": c0, "m": sysm.m, "n": c1 - c0, "row_ptr": rp, "col_idx": ci, "val": v,
            "col_ptr": cp, "row_idx": ri, "val_t": vt, "b": sysm.b}
