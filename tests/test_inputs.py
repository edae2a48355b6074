"""Pins for the seeded input generators (ras_inputs), against the paper's stencil
definition (P435-438), SPEC's worked example (S129) and closed-form spectra."""
import math

import numpy as np
import pytest

import ras_inputs as ri


def dense(A):
    return A.to_scipy().toarray()


def test_laplace_2d_n2_matches_spec_example():
    # SPEC S129: laplace_2d(N=2)
    want = np.array([[4, -1, -1, 0], [-1, 4, 0, -1], [-1, 0, 4, -1], [0, -1, -1, 4]], float)
    assert np.array_equal(dense(ri.laplace_2d(2)), want)


def test_laplace_2d_center_row_n3():
    # SPEC S131: N=3, row 4 -> -1 at {1,3,5,7}, 4 at 4
    A = ri.laplace_2d(3)
    lo, hi = A.indptr[4], A.indptr[5]
    assert A.indices[lo:hi].tolist() == [1, 3, 4, 5, 7]
    assert A.data[lo:hi].tolist() == [-1, -1, 4, -1, -1]


@pytest.mark.parametrize("N", [2, 3, 7, 16, 33])
def test_laplace_2d_nnz_and_symmetry(N):
    A = ri.laplace_2d(N)
    assert A.nnz == 5 * N * N - 4 * N  # S160
    D = dense(A)
    assert np.array_equal(D, D.T)
    # columns strictly increasing per row
    for i in range(A.nrows):
        c = A.indices[A.indptr[i]:A.indptr[i + 1]]
        assert (np.diff(c) > 0).all()


def test_laplace_2d_eigenpairs_closed_form():
    # lambda_jk = 4 - 2cos(j pi/(N+1)) - 2cos(k pi/(N+1)), v = sin (x) sin
    nx, ny = 7, 5
    D = dense(ri.laplace_2d(nx, ny))
    xs = np.arange(1, nx + 1)
    ys = np.arange(1, ny + 1)
    for j in (1, 3, nx):
        for k in (1, 2, ny):
            v = np.outer(np.sin(k * math.pi * ys / (ny + 1)), np.sin(j * math.pi * xs / (nx + 1))).ravel()
            lam = 4 - 2 * math.cos(j * math.pi / (nx + 1)) - 2 * math.cos(k * math.pi / (ny + 1))
            assert np.abs(D @ v - lam * v).max() < 1e-13


def test_laplace_3d_eigenpairs_closed_form():
    nx, ny, nz = 4, 3, 5
    A = ri.laplace_3d(nx, ny, nz)
    assert A.nnz == 7 * nx * ny * nz - 2 * (ny * nz + nx * nz + nx * ny)
    D = dense(A)
    x = np.arange(1, nx + 1)
    y = np.arange(1, ny + 1)
    z = np.arange(1, nz + 1)
    for (i, j, k) in [(1, 1, 1), (2, 3, 4), (4, 2, 5)]:
        v = np.einsum("z,y,x->zyx", np.sin(k * math.pi * z / (nz + 1)), np.sin(j * math.pi * y / (ny + 1)),
                      np.sin(i * math.pi * x / (nx + 1))).ravel()
        lam = 6 - 2 * (math.cos(i * math.pi / (nx + 1)) + math.cos(j * math.pi / (ny + 1)) + math.cos(k * math.pi / (nz + 1)))
        assert np.abs(D @ v - lam * v).max() < 1e-13


def test_row_windows_match_full_matrix():
    full = ri.laplace_2d(9, 6).to_scipy()
    w = ri.laplace_2d_rows(9, 6, 10, 31)
    assert w.row0 == 10 and w.nrows == 21
    assert (w.to_scipy() != full[10:31]).nnz == 0
    full3 = ri.laplace_3d(4, 3, 5).to_scipy()
    w3 = ri.laplace_3d_rows(4, 3, 5, 7, 50)
    assert (w3.to_scipy() != full3[7:50]).nnz == 0


def test_rhs_deterministic_and_in_range():
    a = ri.rhs(1000, 42)
    assert np.array_equal(a, ri.rhs(1000, 42))
    assert not np.array_equal(ri.rhs(4, 1), ri.rhs(4, 2))
    assert a.min() >= -1 and a.max() <= 1 and a.dtype == np.float64


def test_voronoi_partition_valid_and_deterministic():
    own = ri.voronoi_partition(64, 48, 12, seed=1)
    assert own.shape == (64 * 48,)
    assert np.array_equal(own, ri.voronoi_partition(64, 48, 12, seed=1))
    assert set(np.unique(own).tolist()) == set(range(12))


def test_partition_file_roundtrip_and_errors(tmp_path):
    p = tmp_path / "part.txt"
    p.write_text("0\n0\n1\n1\n")
    assert ri.read_partition_file(str(p), 2, 4).tolist() == [0, 0, 1, 1]  # S238
    p.write_text("0\n2\n1\n1\n")
    with pytest.raises(ri.PartitionFileError, match=":2:"):
        ri.read_partition_file(str(p), 2, 4)
    p.write_text("0\n1\n1\n")
    with pytest.raises(ri.PartitionFileError):
        ri.read_partition_file(str(p), 2, 4)
    own = ri.voronoi_partition(20, 20, 5)
    ri.write_partition_file(str(p), own)
    assert np.array_equal(ri.read_partition_file(str(p), 5, 400), own)


def test_rhs_rows_window_equals_slice():
    full = ri.rhs(5000, 3)
    assert np.array_equal(ri.rhs_rows(5000, 1234, 4321, 3), full[1234:4321])
    assert np.array_equal(ri.rhs_rows(5000, 0, 5000, 3), full)


def test_varcoef_2d_is_spd_m_matrix_and_reduces_to_laplacian():
    A = ri.varcoef_2d(9, 7, seed=4)
    S = A.to_scipy().toarray()
    assert np.array_equal(S, S.T)
    off = S - np.diag(np.diag(S))
    assert (off <= 0).all()  # M-matrix sign pattern
    # strictly diagonally dominant on boundary rows, weakly inside: SPD
    assert (np.diag(S) >= -off.sum(axis=1)).all() and np.linalg.eigvalsh(S).min() > 0
    assert len(np.unique(A.data)) <= 4 + 13  # few distinct values (4 weights, sums of 4 of them)
    one = ri.varcoef_2d(6, 5, levels=(1.0,))
    np.testing.assert_array_equal(one.to_scipy().toarray(), ri.laplace_2d(6, 5).to_scipy().toarray())


def test_balanced_voronoi_cells_nearly_equal_and_connected():
    # lloyd + power-diagram balancing: a graph partitioner's balance constraint
    # stand-in for C5 (cells within a few % of n / P), still valid 4-connected cells
    o = ri.voronoi_partition(300, 260, 12, seed=3, lloyd=6, balance=60)
    c = np.bincount(o, minlength=12)
    assert c.min() > 0.93 * c.mean() and c.max() < 1.07 * c.mean(), c
    plain = np.bincount(ri.voronoi_partition(300, 260, 12, seed=3), minlength=12)
    assert plain.max() / plain.mean() > c.max() / c.mean()  # balancing did something
