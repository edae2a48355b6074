"""Seeded synthetic input generators shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic.  It only produces the inputs
the paper's experiments are shaped like (§4.1, P435-442):

* the 2D 5-point Laplacian, stencil {-1,-1,4,-1,-1} with offsets {-N,-1,0,1,N}
  and the stencil truncated at the grid edges (P435-438; SPEC S126-S160);
* the 3D 7-point analogue (not in the paper; reading R24);
* the random right-hand side, uniform in [-1, 1] (P440 "We use a random RHS";
  SPEC S135, S165; DESIGN.md input recipe);
* a seeded Voronoi ("graph-partitioned", irregular) owner array standing in for
  METIS output (P217, P288-290), and the one-id-per-line
  partition file format (SPEC S236-S244).

The regular block partition is *not* here: it is part of the method (P277-286)
and is implemented independently by `oracle/` and by the CUDA library.

Grid numbering: 2D point (x, y) -> y*nx + x; 3D (x, y, z) -> (z*ny + y)*nx + x
(SPEC S166; reading R23).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "CSR",
    "laplace_2d",
    "laplace_3d",
    "laplace_2d_rows",
    "laplace_3d_rows",
    "rhs",
    "rhs_rows",
    "varcoef_2d",
    "voronoi_partition",
    "read_partition_file",
    "write_partition_file",
    "PartitionFileError",
]


class CSR:
    """Plain CSR container (0-based, sorted columns).

    indptr : int64[nrows+1] relative to the first stored row
    indices: int32[nnz]     global column ids
    data   : float64[nnz]
    n      : global dimension
    row0   : global id of the first stored row (0 for a full matrix)
    """

    __slots__ = ("indptr", "indices", "data", "n", "row0")

    def __init__(self, indptr, indices, data, n, row0=0):
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self.n = int(n)
        self.row0 = int(row0)

    @property
    def nrows(self) -> int:
        return len(self.indptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp

        return sp.csr_matrix((self.data, self.indices, self.indptr), shape=(self.nrows, self.n))


def _stencil_rows(r0: int, r1: int, dims, diag: float) -> CSR:
    """Rows [r0, r1) of the (2D or 3D) stencil matrix, columns ascending."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    if not (0 <= r0 <= r1 <= n):
        raise ValueError(f"row window [{r0},{r1}) outside [0,{n})")
    rows = np.arange(r0, r1, dtype=np.int64)
    # coordinates, x fastest
    coords = []
    rem = rows.copy()
    for d in dims:
        coords.append(rem % d)
        rem //= d
    strides = [1]
    for d in dims[:-1]:
        strides.append(strides[-1] * d)
    # slots in ascending column order: -stride_k (k descending), 0, +stride_k (k ascending)
    offs, masks, vals = [], [], []
    for k in reversed(range(len(dims))):
        offs.append(-strides[k])
        masks.append(coords[k] > 0)
        vals.append(-1.0)
    offs.append(0)
    masks.append(np.ones(len(rows), dtype=bool))
    vals.append(diag)
    for k in range(len(dims)):
        offs.append(strides[k])
        masks.append(coords[k] < dims[k] - 1)
        vals.append(-1.0)
    M = np.stack(masks, axis=1)  # (nrows, nslots)
    cols = rows[:, None] + np.asarray(offs, dtype=np.int64)[None, :]
    V = np.broadcast_to(np.asarray(vals, dtype=np.float64)[None, :], M.shape)
    counts = M.sum(axis=1)
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = cols[M].astype(np.int32)
    data = V[M].astype(np.float64)
    return CSR(indptr, indices, data, n, r0)


def laplace_2d(nx: int, ny: int | None = None) -> CSR:
    """2D 5-point Laplacian on an nx-by-ny grid (P435-438). N x N when ny is None."""
    ny = nx if ny is None else ny
    if nx < 1 or ny < 1:
        raise ValueError("grid dimensions must be >= 1")
    return _stencil_rows(0, nx * ny, (nx, ny), 4.0)


def laplace_2d_rows(nx: int, ny: int, r0: int, r1: int) -> CSR:
    """Rows [r0, r1) of laplace_2d(nx, ny) (a row window for large problems)."""
    return _stencil_rows(r0, r1, (nx, ny), 4.0)


def laplace_3d(nx: int, ny: int | None = None, nz: int | None = None) -> CSR:
    """3D 7-point Laplacian (6 on the diagonal, -1 at +-1, +-nx, +-nx*ny); reading R24."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    return _stencil_rows(0, nx * ny * nz, (nx, ny, nz), 6.0)


def laplace_3d_rows(nx: int, ny: int, nz: int, r0: int, r1: int) -> CSR:
    return _stencil_rows(r0, r1, (nx, ny, nz), 6.0)


def varcoef_2d(nx: int, ny: int, levels=(1.0, 2.0, 3.0, 4.0), seed: int = 3) -> CSR:
    """Variable-coefficient 5-point diffusion on an nx-by-ny grid: an irregular
    sparse SPD M-matrix of the paper's problem class (A x = b, A sparse SPD,
    P114-118) for exercising the matrix formats, not one of its workloads.

    Every grid edge (x,y)-(x+1,y) / (x,y)-(x,y+1) and every Dirichlet boundary
    edge gets a weight drawn uniformly from `levels` (default_rng(seed)); row i
    holds -w_e for each interior edge e at i and, on the diagonal, the sum of
    the weights of all four edges at i (the 2D Laplacian is every w_e = 1).
    Few distinct values, many distinct rows."""
    rng = np.random.default_rng(seed)
    lv = np.asarray(levels, dtype=np.float64)
    wx = lv[rng.integers(0, len(lv), size=(ny, nx + 1))]  # wx[y, x]: edge left of (x, y); x = nx: right boundary
    wy = lv[rng.integers(0, len(lv), size=(ny + 1, nx))]  # wy[y, x]: edge below (x, y); y = ny: top boundary
    n = nx * ny
    yy, xx = np.divmod(np.arange(n, dtype=np.int64), nx)
    diag = wx[yy, xx] + wx[yy, xx + 1] + wy[yy, xx] + wy[yy + 1, xx]
    # column slots ascending: -nx, -1, 0, +1, +nx
    offs = np.array([-nx, -1, 0, 1, nx], dtype=np.int64)
    M = np.stack([yy > 0, xx > 0, np.ones(n, bool), xx < nx - 1, yy < ny - 1], axis=1)
    V = np.stack([-wy[yy, xx], -wx[yy, xx], diag, -wx[yy, xx + 1], -wy[yy + 1, xx]], axis=1)
    cols = np.arange(n, dtype=np.int64)[:, None] + offs[None, :]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(M.sum(axis=1), out=indptr[1:])
    return CSR(indptr, cols[M].astype(np.int32), V[M], n, 0)


def rhs(n: int, seed: int = 0) -> np.ndarray:
    """Random RHS, uniform in [-1, 1], FP64 (P440; SPEC S135)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, int(n))


def rhs_rows(n: int, r0: int, r1: int, seed: int = 0) -> np.ndarray:
    """rhs(n, seed)[r0:r1] without drawing the prefix (PCG64 advance: one 64-bit
    draw per double), for row windows of very large problems."""
    if not (0 <= r0 <= r1 <= n):
        raise ValueError("bad window")
    g = np.random.default_rng(seed)
    g.bit_generator.advance(int(r0))
    return g.uniform(-1.0, 1.0, int(r1 - r0))


def _morton2(ix: np.ndarray, iy: np.ndarray) -> np.ndarray:
    def spread(v):
        v = v.astype(np.uint64) & np.uint64(0xFFFF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v

    return spread(ix) | (spread(iy) << np.uint64(1))


def _nearest_site(px, py, sx, sy, w=None):
    best = np.full(len(px), np.inf)
    arg = np.zeros(len(px), dtype=np.int32)
    for s in range(len(sx)):
        d = (px - sx[s]) ** 2 + (py - sy[s]) ** 2
        if w is not None:
            d = d - w[s]  # power distance (weighted Voronoi)
        better = d < best  # strict: ties keep the lower id
        best = np.where(better, d, best)
        arg = np.where(better, np.int32(s), arg)
    return arg


def voronoi_partition(nx: int, ny: int, P: int, seed: int = 1, chunk: int = 1 << 22, lloyd: int = 0,
                      balance: int = 0) -> np.ndarray:
    """Seeded irregular partition of an nx-by-ny grid into P Voronoi cells.

    Stand-in for the paper's METIS partition (P217, P288-290), SURVEY §8d C5:
    sites ~ default_rng(seed) uniform in [0,nx) x [0,ny); sites renumbered along
    a Morton curve (so contiguous id blocks are spatially compact and map to one
    GPU); each grid point (x, y) goes to the nearest site in Euclidean distance,
    ties to the lower id.  Raises ValueError on an empty or disconnected cell.

    lloyd > 0: that many Lloyd relaxation steps first (each site moves to the
    centroid of its cell, evaluated on the grid subsampled to <= ~10^6 points),
    i.e. a near-centroidal Voronoi tessellation: cells of nearly equal size with
    irregular boundaries -- closer to a graph partitioner's balanced parts.
    balance > 0: then that many steps of a power-diagram (weighted Voronoi)
    balancing, w_s += (target - cells_s) * step^2 / pi on the subsampled grid,
    so that the cells have nearly equal sizes (within ~1-2 % after 60 steps),
    like a graph partitioner's balance constraint; cells stay convex polygons.
    """
    rng = np.random.default_rng(seed)
    sx = rng.uniform(0.0, nx, P)
    sy = rng.uniform(0.0, ny, P)
    w = None
    if lloyd > 0 or balance > 0:
        st = max(1, int(np.ceil(np.sqrt(nx * ny / 1.0e6))))
        gx, gy = np.meshgrid(np.arange(0, nx, st, dtype=np.float64), np.arange(0, ny, st, dtype=np.float64))
        gx, gy = gx.ravel(), gy.ravel()
        for _ in range(lloyd):
            a = _nearest_site(gx, gy, sx, sy)
            cnt = np.bincount(a, minlength=P)
            keep = cnt > 0
            sx = np.where(keep, np.bincount(a, weights=gx, minlength=P) / np.maximum(cnt, 1), sx)
            sy = np.where(keep, np.bincount(a, weights=gy, minlength=P) / np.maximum(cnt, 1), sy)
        if balance > 0:
            w = np.zeros(P)
            target = len(gx) / P
            for _ in range(balance):
                cnt = np.bincount(_nearest_site(gx, gy, sx, sy, w), minlength=P)
                w = w + (target - cnt) * st * st / np.pi
    q = 65535.0
    code = _morton2(np.floor(sx / nx * q).astype(np.int64), np.floor(sy / ny * q).astype(np.int64))
    order = np.argsort(code, kind="stable")
    sx, sy = sx[order], sy[order]
    if w is not None:
        w = w[order]
    n = nx * ny
    owner = np.empty(n, dtype=np.int32)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        idx = np.arange(c0, c1, dtype=np.int64)
        px = (idx % nx).astype(np.float64)
        py = (idx // nx).astype(np.float64)
        owner[c0:c1] = _nearest_site(px, py, sx, sy, w)
    _validate_cells(owner.reshape(ny, nx), P)
    return owner


def _validate_cells(grid: np.ndarray, P: int) -> None:
    from scipy import ndimage

    counts = np.bincount(grid.ravel(), minlength=P)
    if (counts == 0).any():
        raise ValueError(f"empty Voronoi cell(s): {np.nonzero(counts == 0)[0].tolist()}")
    # connectivity (4-neighbour) of every cell
    objs = ndimage.find_objects(grid + 1)
    for p, sl in enumerate(objs):
        if sl is None:
            continue
        sub = grid[sl] == p
        _, ncomp = ndimage.label(sub)
        if ncomp != 1:
            raise ValueError(f"Voronoi cell {p} is not 4-connected ({ncomp} components)")


class PartitionFileError(ValueError):
    pass


def read_partition_file(path: str, P: int, n: int) -> np.ndarray:
    """SPEC S236-S244: n lines, line i = owner id of global index i, in [0, P)."""
    owner = []
    with open(path) as f:
        for lineno, line in enumerate(f, 1):
            s = line.strip()
            if s == "":
                continue
            try:
                v = int(s)
            except ValueError:
                raise PartitionFileError(f"{path}:{lineno}: not an integer: {s!r}")
            if not (0 <= v < P):
                raise PartitionFileError(f"{path}:{lineno}: subdomain id {v} outside [0,{P})")
            owner.append(v)
    if len(owner) != n:
        raise PartitionFileError(f"{path}: {len(owner)} entries, expected n={n}")
    return np.asarray(owner, dtype=np.int32)


def write_partition_file(path: str, owner: np.ndarray) -> None:
    np.savetxt(path, np.asarray(owner, dtype=np.int64), fmt="%d")
