"""Oracle pins: partitioning, overlap, subdomain extraction (P133-142, P247-303).

Pinned against SPEC's hand-derived examples, closed-form overlap sizes, and an
independent brute-force reachability computation (dense boolean matrix powers)."""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri


def test_regular1d_spec_examples():
    assert O.partition_regular1d(4, 2).tolist() == [0] * 8 + [1] * 8  # S215
    own = O.partition_regular1d(4, 4)  # S216: one grid row each
    assert own.reshape(4, 4).tolist() == [[0] * 4, [1] * 4, [2] * 4, [3] * 4]


def test_regular2d_spec_examples():
    own = O.partition_regular2d(4, 4).reshape(4, 4)  # S224 quadrants
    assert own.tolist() == [[0, 0, 1, 1], [0, 0, 1, 1], [2, 2, 3, 3], [2, 2, 3, 3]]
    own2 = O.partition_regular2d(4, 2).reshape(4, 4)  # S225: 1x2 -> two 4x2 halves
    assert own2.tolist() == [[0] * 4, [0] * 4, [1] * 4, [1] * 4]
    assert O.factor_pair(2) == (1, 2) and O.factor_pair(6) == (2, 3) and O.factor_pair(16) == (4, 4)


def test_regular_earlier_blocks_take_remainder():
    own = O.partition_regular(10, 1, 1, 3, 1, 1)
    assert own.tolist() == [0, 0, 0, 0, 1, 1, 1, 2, 2, 2]
    with pytest.raises(ValueError):
        O.partition_regular(3, 3, 1, 4, 1, 1)


def test_regular_3d_ids():
    own = O.partition_regular(4, 4, 4, 2, 2, 2).reshape(4, 4, 4)  # [z][y][x]
    assert own[0, 0, 0] == 0 and own[0, 0, 3] == 1 and own[0, 3, 0] == 2 and own[3, 0, 0] == 4
    assert own[3, 3, 3] == 7


def test_expand_overlap_spec_example():
    A = ri.laplace_2d(4)
    own = O.partition_regular1d(4, 2)
    om0, ow0, gh0 = O.overlap_sets(A, own, 0, 1)
    om1, ow1, gh1 = O.overlap_sets(A, own, 1, 1)
    assert om0[~ow0].tolist() == [8, 9, 10, 11]  # S252
    assert om1[~ow1].tolist() == [4, 5, 6, 7]
    assert len(om0) == 12 and gh0.tolist() == [12, 13, 14, 15]  # S261
    om, ow, gh = O.overlap_sets(A, own, 0, 0)
    assert (ow).all() and len(om) == 8


def test_setup_spec_example_local_dim_24():
    # S483: laplace(8), regular2d P=4, gamma=1 -> local dim 16 + 8
    A = ri.laplace_2d(8)
    subs = O.setup(A, np.zeros(64), O.partition_regular2d(8, 4), 1)
    assert [len(s.omega) for s in subs] == [24] * 4


def _reach_bruteforce(A, owner, p, gamma):
    D = (A.to_scipy().toarray() != 0).astype(np.int64)
    v = (owner == p).astype(np.int64)
    for _ in range(gamma):
        v = ((D @ v) > 0).astype(np.int64) | v
    omega = np.nonzero(v)[0]
    g = ((D @ v) > 0) & (v == 0)
    return omega, np.nonzero(g)[0]


@pytest.mark.parametrize("gamma", [0, 1, 2, 3, 5])
def test_overlap_matches_bruteforce_reachability(gamma):
    A = ri.laplace_2d(11, 9)
    owner = ri.voronoi_partition(11, 9, 6, seed=3)
    for p in range(6):
        om, ow, gh = O.overlap_sets(A, owner, p, gamma)
        om2, gh2 = _reach_bruteforce(A, owner, p, gamma)
        assert np.array_equal(om, om2) and np.array_equal(gh, gh2)
        assert np.array_equal(ow, owner[om] == p)


def test_overlap_saturates():
    A = ri.laplace_2d(6)
    own = O.partition_regular2d(6, 4)
    om, ow, gh = O.overlap_sets(A, own, 0, 100)
    assert len(om) == 36 and len(gh) == 0


def _omega_2d_interior(a, b, g):
    return a * b + 2 * g * (a + b) + 2 * g * (g - 1)


@pytest.mark.parametrize("a,b,g", [(6, 5, 1), (6, 5, 2), (7, 7, 3), (5, 8, 4)])
def test_overlap_size_formula_2d_interior_tile(a, b, g):
    # centre tile of a 3x3 tiling, far from the grid boundary
    nx, ny = 3 * a, 3 * b
    A = ri.laplace_2d(nx, ny)
    own = O.partition_regular(nx, ny, 1, 3, 3, 1)
    om, ow, gh = O.overlap_sets(A, own, 4, g)
    assert len(om) == _omega_2d_interior(a, b, g)
    assert len(gh) == 2 * (a + b) + 4 * g


@pytest.mark.parametrize("a,g", [(4, 1), (5, 2), (6, 3)])
def test_overlap_size_formula_3d_corner_tile(a, g):
    A = ri.laplace_3d(2 * a)
    own = O.partition_regular(2 * a, 2 * a, 2 * a, 2, 2, 2)
    om, ow, gh = O.overlap_sets(A, own, 0, g)
    want = a ** 3 + 3 * a * a * g + 3 * a * g * (g - 1) // 2 + g * (g - 1) * (g - 2) // 6
    assert len(om) == want


def test_c1_sizes():
    # |Omega|=1153, |Gamma|=66, nnz(A_p)=5629, nnz(B_p)=68, halo 195
    A = ri.laplace_2d(64)
    own = O.partition_regular(64, 64, 1, 2, 2, 1)
    subs = O.setup(A, ri.rhs(4096), own, 2)
    for s in subs:
        assert (len(s.omega), len(s.ghosts), s.A.nnz, s.B.nnz) == (1153, 66, 5629, 68)
    assert O.comm_pattern(subs, own).sum(1).tolist() == [195] * 4


def test_row_tiling_reproduces_A():
    # S257/S276: local (+) interface reproduce A's rows over Omega_p bit-exactly
    A = ri.laplace_2d(13, 10)
    As = A.to_scipy()
    owner = ri.voronoi_partition(13, 10, 5, seed=2)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(130)
    for s in O.setup(A, np.zeros(130), owner, 2):
        y = s.A @ x[s.omega] + s.B @ x[s.ghosts]
        assert np.allclose(y, As[s.omega] @ x, rtol=0, atol=1e-14)
        assert s.A.nnz + s.B.nnz == As[s.omega].nnz


def test_comm_pattern_properties():
    A = ri.laplace_2d(8)
    own = O.partition_regular1d(8, 4)
    subs = O.setup(A, np.zeros(64), own, 1)
    C = O.comm_pattern(subs, own, include_overlap=False)
    for p in range(4):
        for q in range(4):
            if abs(p - q) > 1:
                assert C[p, q] == 0  # S269 tridiagonal (Fig. 2b)
    assert ((C > 0) == (C.T > 0)).all()
    subs1 = O.setup(A, np.zeros(64), np.zeros(64, np.int32), 0)
    assert O.comm_pattern(subs1, np.zeros(64, np.int32)).sum() == 0


def test_neighbour_bounds_gamma0():
    # P277-286: regular1d <= 2 neighbours, regular2d <= 4 (gamma=0 adjacency, R3)
    A = ri.laplace_2d(16)
    for own, bound in [(O.partition_regular1d(16, 8), 2), (O.partition_regular2d(16, 9), 4)]:
        subs = O.setup(A, np.zeros(256), own, 0)
        C = O.comm_pattern(subs, own)
        assert ((C > 0).sum(1) <= bound).all()
    # with hop overlap diagonal tiles also contribute (R3): centre of 3x3 at gamma=1 -> 8 owners
    own = O.partition_regular2d(15, 9)
    subs = O.setup(ri.laplace_2d(15), np.zeros(225), own, 1)
    assert (O.comm_pattern(subs, own)[4] > 0).sum() == 8
