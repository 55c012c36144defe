"""Model-problem generators (seeded, synthetic) — inputs only, no method arithmetic.

Readings:
  R14  Dirichlet-eliminated finite differences without h^2: the isotropic 7-point
       operator has diagonal 6 and off-diagonals -1 (Eq. 4.1;
       SPEC.md:124); the anisotropic one has diagonal 2(k1+k2+k3) and
       off-diagonal -k_d (PAPER.md:537-549 supplementary anisotropic problem).
  R15  Lexicographic numbering, x fastest, then y, then z.  A contiguous row
       block [row_begin, row_end) of whole z-planes is a z-slab.
  R16  BASELINE.json configs[4]: 27-point operator with piecewise-constant
       coefficient kappa = 10^U(-3,3) on 8x8x8 coefficient blocks; couplings are
       harmonic means h_ij = 2 k_i k_j / (k_i + k_j); a_ii = sum over all 26
       stencil neighbours of h_ij, an outside (Dirichlet-eliminated) neighbour
       taking kappa_j = kappa_i.
  R17  RNG: u = (PCG64(seed).random_raw(n) >> 11) * 2^-53.

Matrices are returned as CSR with int64 row pointers, int64 GLOBAL column
indices sorted ascending within each row, and float64 values.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CSR:
    n_global: int          # global number of rows/cols
    row_begin: int         # first global row held here
    row_end: int           # one past the last global row held here
    rowptr: np.ndarray     # int64, (row_end-row_begin)+1, 0-based
    colind: np.ndarray     # int64 global column indices, ascending per row
    values: np.ndarray     # float64

    @property
    def n_local(self) -> int:
        return self.row_end - self.row_begin

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.colind, self.rowptr),
                             shape=(self.n_local, self.n_global))


# --------------------------------------------------------------------------- RNG
def _raw(seed: int, begin: int, count: int) -> np.ndarray:
    bg = np.random.PCG64(seed)
    if begin:
        bg.advance(begin)
    return bg.random_raw(count)


def uniform01(seed: int, n: int, begin: int = 0) -> np.ndarray:
    """U[0,1) stream entries [begin, begin+n) (R17)."""
    r = _raw(seed, begin, n)
    return (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(seed: int, n: int, begin: int = 0) -> np.ndarray:
    """U[-1,1) = 2u - 1 (R17)."""
    return 2.0 * uniform01(seed, n, begin) - 1.0


# --------------------------------------------------------------------- 7-point
def poisson7(nx: int, ny: int, nz: int, k=(1.0, 1.0, 1.0),
             row_begin: int = 0, row_end: int | None = None,
             chunk_rows: int = 1 << 22) -> CSR:
    """7-point (an)isotropic Dirichlet Laplacian, rows [row_begin,row_end)."""
    n = nx * ny * nz
    if row_end is None:
        row_end = n
    if not (0 <= row_begin <= row_end <= n):
        raise ValueError("bad row range")
    k1, k2, k3 = (float(v) for v in k)
    diag = 2.0 * (k1 + k2 + k3)
    plane = nx * ny
    # offsets in ascending column order
    offs = np.array([-plane, -nx, -1, 0, 1, nx, plane], dtype=np.int64)
    vals = np.array([-k3, -k2, -k1, diag, -k1, -k2, -k3], dtype=np.float64)
    nloc = row_end - row_begin
    counts = np.empty(nloc, dtype=np.int64)
    cols_parts, vals_parts = [], []
    for c0 in range(row_begin, row_end, chunk_rows):
        c1 = min(row_end, c0 + chunk_rows)
        idx = np.arange(c0, c1, dtype=np.int64)
        x = idx % nx
        y = (idx // nx) % ny
        z = idx // plane
        mask = np.empty((c1 - c0, 7), dtype=bool)
        mask[:, 0] = z > 0
        mask[:, 1] = y > 0
        mask[:, 2] = x > 0
        mask[:, 3] = True
        mask[:, 4] = x < nx - 1
        mask[:, 5] = y < ny - 1
        mask[:, 6] = z < nz - 1
        cols = idx[:, None] + offs[None, :]
        counts[c0 - row_begin:c1 - row_begin] = mask.sum(axis=1)
        cols_parts.append(cols[mask])
        vals_parts.append(np.broadcast_to(vals, (c1 - c0, 7))[mask])
    rowptr = np.zeros(nloc + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    colind = np.concatenate(cols_parts) if cols_parts else np.zeros(0, np.int64)
    values = np.concatenate(vals_parts) if vals_parts else np.zeros(0)
    return CSR(n, row_begin, row_end, rowptr, colind, values)


# -------------------------------------------------------------------- 27-point
def jump_kappa(nb: int = 8, seed: int = 50) -> np.ndarray:
    """kappa[bz][by][bx] = 10^(6u-3), u from the PCG64 stream (R16, R17)."""
    u = uniform01(seed, nb * nb * nb)
    return (10.0 ** (6.0 * u - 3.0)).reshape(nb, nb, nb)


def _harm(ki: np.ndarray, kj: np.ndarray) -> np.ndarray:
    # symmetric evaluation order: (2*lo*hi)/(lo+hi) with lo <= hi
    lo = np.minimum(ki, kj)
    hi = np.maximum(ki, kj)
    return ((2.0 * lo) * hi) / (lo + hi)


def jump27(N: int, nb: int = 8, seed: int = 50,
           row_begin: int = 0, row_end: int | None = None,
           chunk_rows: int = 1 << 20) -> CSR:
    """27-point jump-coefficient diffusion operator on an N^3 grid (R16)."""
    if N % nb:
        raise ValueError("N must be a multiple of the coefficient-block count")
    n = N ** 3
    if row_end is None:
        row_end = n
    kap = jump_kappa(nb, seed)
    bs = N // nb
    plane = N * N
    offs = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    nloc = row_end - row_begin
    counts = np.empty(nloc, dtype=np.int64)
    cols_parts, vals_parts = [], []
    for c0 in range(row_begin, row_end, chunk_rows):
        c1 = min(row_end, c0 + chunk_rows)
        idx = np.arange(c0, c1, dtype=np.int64)
        x = idx % N
        y = (idx // N) % N
        z = idx // plane
        ki = kap[z // bs, y // bs, x // bs]
        m = c1 - c0
        mask = np.empty((m, 27), dtype=bool)
        cols = np.empty((m, 27), dtype=np.int64)
        vals = np.empty((m, 27), dtype=np.float64)
        diag = np.zeros(m)
        for t, (dz, dy, dx) in enumerate(offs):
            if (dz, dy, dx) == (0, 0, 0):
                mask[:, t] = True
                cols[:, t] = idx
                continue
            xx, yy, zz = x + dx, y + dy, z + dz
            inside = ((xx >= 0) & (xx < N) & (yy >= 0) & (yy < N) & (zz >= 0) & (zz < N))
            kj = ki.copy()
            kj[inside] = kap[zz[inside] // bs, yy[inside] // bs, xx[inside] // bs]
            h = _harm(ki, kj)
            diag += h
            mask[:, t] = inside
            cols[:, t] = idx + dz * plane + dy * N + dx
            vals[:, t] = -h
        vals[:, 13] = diag
        counts[c0 - row_begin:c1 - row_begin] = mask.sum(axis=1)
        cols_parts.append(cols[mask])
        vals_parts.append(vals[mask])
    rowptr = np.zeros(nloc + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return CSR(n, row_begin, row_end, rowptr,
               np.concatenate(cols_parts), np.concatenate(vals_parts))


# ------------------------------------------------------------ irregular graph
def random_spd(n: int, deg: int = 6, window: int = 64, hubs: int = 0, hub_deg: int = 300,
               shift: float = 1e-2, seed: int = 70) -> CSR:
    """Irregular symmetric M-matrix (edge-case inputs, not a paper workload).

    Each row i draws `deg` partners i + d, d uniform in [1, window] (dropped if
    >= n); `hubs` evenly spaced rows each draw `hub_deg` partners anywhere.
    Edge weights w in [0.1, 1.1); duplicate edges add.  a_ij = -w_ij,
    a_ii = sum_j w_ij + shift * (1 + u_i), so A is symmetric, strictly
    diagonally dominant and SPD, with a ragged row-length distribution (the
    irregular-pattern edge cases of the format selection and the matching).
    """
    import scipy.sparse as sp
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    d = 1 + (uniform01(seed, n * deg) * window).astype(np.int64)
    cols = rows + d
    w = 0.1 + uniform01(seed + 1, n * deg)
    keep = cols < n
    rows, cols, w = rows[keep], cols[keep], w[keep]
    if hubs and n > 1:
        hr = np.repeat(np.linspace(0, n - 1, hubs).astype(np.int64), hub_deg)
        hc = (uniform01(seed + 2, hr.size) * n).astype(np.int64)
        hw = 0.1 + uniform01(seed + 3, hr.size)
        ok = hr != hc
        rows = np.concatenate([rows, hr[ok]])
        cols = np.concatenate([cols, hc[ok]])
        w = np.concatenate([w, hw[ok]])
    W = sp.coo_matrix((w, (rows, cols)), shape=(n, n)).tocsr()
    W = (W + W.T).tocsr()
    W.sum_duplicates()
    diag = np.asarray(W.sum(axis=1)).ravel() + shift * (1.0 + uniform01(seed + 4, n))
    A = (sp.diags(diag) - W).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return CSR(n, 0, n, A.indptr.astype(np.int64), A.indices.astype(np.int64),
               A.data.astype(np.float64))


def diagonal_spd(n: int, seed: int = 71) -> CSR:
    """Diagonal SPD matrix a_ii = 1 + u_i (no couplings: the matching's empty-graph case)."""
    return CSR(n, 0, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
               1.0 + uniform01(seed, n))


def islands(seed: int = 73) -> CSR:
    """Disconnected graph: poisson7(12,12,12) (+) poisson7(9,7,5) (+) 37 isolated rows, symmetrically
    permuted by a seeded permutation so the components interleave in the row order (the matching's
    unmatched-vertex and disconnected-component cases, away from the lexicographic order)."""
    blocks = [poisson7(12, 12, 12), poisson7(9, 7, 5), diagonal_spd(37, seed=seed + 1)]
    rows, cols, vals, off = [], [], [], 0
    for B in blocks:
        r = np.repeat(np.arange(B.n_global, dtype=np.int64), np.diff(B.rowptr))
        rows.append(r + off)
        cols.append(B.colind + off)
        vals.append(B.values)
        off += B.n_global
    n = off
    perm = np.argsort(uniform01(seed, n), kind="stable")  # new index of old row i: inv[i]
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n, dtype=np.int64)
    r = inv[np.concatenate(rows)]
    c = inv[np.concatenate(cols)]
    v = np.concatenate(vals)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return CSR(n, 0, n, np.cumsum(rp), c, v)


# ------------------------------------------------------------------- configs
CONFIGS = {
    # name: (grid builder, rhs, pre, post, maxsize_per_gpu)
    1: dict(kind="poisson7", grid=(16, 16, 16), k=(1.0, 1.0, 1.0), rhs="ones", seed=None, sweeps=(1, 1)),
    2: dict(kind="poisson7", grid=(128, 128, 128), k=(1.0, 1.0, 1.0), rhs="u01", seed=2, sweeps=(1, 1)),
    3: dict(kind="poisson7", grid=(256, 256, 256), k=(1.0, 1.0, 0.01), rhs="upm1", seed=3, sweeps=(2, 2)),
    4: dict(kind="poisson7", grid=(256, 256, 256), k=(1.0, 1.0, 1.0), rhs="ones", seed=None, sweeps=(1, 1)),
    5: dict(kind="jump27", grid=(512, 512, 512), k=None, rhs="u01", seed=5, sweeps=(1, 1)),
}


def rhs_vector(kind: str, seed, n_local: int, begin: int) -> np.ndarray:
    if kind == "ones":
        return np.ones(n_local)
    if kind == "u01":
        return uniform01(seed, n_local, begin)
    if kind == "upm1":
        return uniform_pm1(seed, n_local, begin)
    raise ValueError(kind)


def config_problem(cfg: int, nranks: int = 1, rank: int = 0, grid=None):
    """Return (A_local CSR, b_local, meta) for BASELINE config `cfg`.

    Config 4 is weak scaling: the global grid is 256 x 256 x (256*nranks).
    `grid` overrides the grid (small analogues with the same generator).
    Rows are split into contiguous z-slabs (R15): rank g owns planes
    [g*nz/np, (g+1)*nz/np).
    """
    c = CONFIGS[cfg]
    if grid is None:
        grid = c["grid"]
        if cfg == 4:
            grid = (grid[0], grid[1], grid[2] * nranks)
    nx, ny, nz = grid
    if nz % nranks:
        raise ValueError("nz must be divisible by the number of ranks")
    plane = nx * ny
    z0 = rank * (nz // nranks)
    z1 = (rank + 1) * (nz // nranks)
    r0, r1 = z0 * plane, z1 * plane
    if c["kind"] == "poisson7":
        A = poisson7(nx, ny, nz, c["k"], r0, r1)
    else:
        if not (nx == ny == nz):
            raise ValueError("jump27 needs a cube")
        A = jump27(nx, 8, 50, r0, r1)
    b = rhs_vector(c["rhs"], c["seed"], r1 - r0, r0)
    meta = dict(config=cfg, grid=(nx, ny, nz), sweeps=c["sweeps"],
                max_coarse_size=200 * nranks, rhs=c["rhs"], seed=c["seed"])
    return A, b, meta
