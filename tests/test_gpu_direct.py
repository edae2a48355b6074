"""NEXT f1: the direct local solve (RAS_LS_CHOLESKY: complete banded Cholesky
factor from the host, two banded triangular solves per local solve on the GPU)
against the oracle's exact local solve (dense / LAPACK banded Cholesky,
P311-318).  Bar: sync iterates within 1e-10 (FP64), sweep counts equal."""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def oracle_exact(A, b, owner, gamma, K, tol=1e-300):
    subs = O.setup(A, b, owner, gamma)
    for s in subs:
        O.make_local_solver(s, "exact")
    return O.ras_sync(A, b, subs, tol, K, record_iterates=True)


def test_c1_iterates_sweeps_and_solution():
    # C1: 64x64, 2x2, overlap 2, exact local solves: 106 sweeps to 1e-8 (oracle)
    N = 64
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = R.partition_regular(N, N, 1, 2, 2, 1)
    ref = oracle_exact(A, b, owner, 2, 1000, tol=1e-8)
    assert ref.sweeps == 106
    s = R.Solver(A, b, owner, 2, R.options("cholesky"))
    for k in (1, 2, 7):
        st, x = s.solve(1e-300, k, "sync")
        assert rel(x, ref.iterates[k]) <= 1e-10, (k, rel(x, ref.iterates[k]))
    st, x = s.solve(1e-8, 1000, "sync")
    assert st == 0 and s.stats()["sweeps"] == 106
    assert rel(x, ref.x) <= 1e-10
    assert s.stats()["inner_iters_total"] == 0
    s.close()


@pytest.mark.parametrize("case", ["voronoi_ragged", "strips", "3d"])
def test_iterates_match_oracle(case):
    if case == "voronoi_ragged":
        nx, ny = 83, 71
        A = ri.laplace_2d(nx, ny)
        owner = ri.voronoi_partition(nx, ny, 7, seed=4)
        gamma, n = 3, nx * ny
    elif case == "strips":
        nx, ny = 40, 96
        A = ri.laplace_2d(nx, ny)
        owner = R.partition_regular(nx, ny, 1, 1, 5, 1)
        gamma, n = 1, nx * ny
    else:
        N = 14
        A = ri.laplace_3d(N)
        owner = O.partition_regular(N, N, N, 2, 2, 2)
        gamma, n = 2, N ** 3
    b = ri.rhs(n, 1)
    ref = oracle_exact(A, b, owner, gamma, 5)
    s = R.Solver(A, b, owner, gamma, R.options("cholesky"))
    for k in (1, 5):
        st, x = s.solve(1e-300, k, "sync")
        assert rel(x, ref.iterates[k]) <= 1e-10, (case, k, rel(x, ref.iterates[k]))
    s.close()


def test_one_subdomain_no_overlap_is_the_exact_solve():
    # north_star invariant: RAS with one subdomain and zero overlap = the exact solve
    N = 40
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 3)
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    s = R.Solver(A, b, np.zeros(N * N, np.int32), 0, R.options("cholesky"))
    st, x = s.solve(1e-12, 10, "sync")
    assert st == 0 and s.stats()["sweeps"] == 1
    assert rel(x, xs) <= 1e-12
    s.close()


def test_async_converges():
    N = 64
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = ri.voronoi_partition(N, N, 6, seed=2)
    s = R.Solver(A, b, owner, 3, R.options("cholesky", detector="central"))
    st, x = s.solve(1e-8, 20000, "async")
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0]
    s.close()


def test_errors():
    big = ri.laplace_2d(120)
    with pytest.raises(R.RasError, match="rows"):
        R.Solver(big, ri.rhs(120 * 120), np.zeros(120 * 120, np.int32), 0, R.options("cholesky"))
    N = 16
    B = ri.laplace_2d(N)
    B.data[B.indptr[5]:B.indptr[6]] *= -1.0  # row 5 no longer SPD-compatible
    with pytest.raises(R.RasError, match="RAS_ENOTSPD.*subdomain 0"):
        R.Solver(B, ri.rhs(N * N), np.zeros(N * N, np.int32), 1, R.options("cholesky"))
