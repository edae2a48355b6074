"""Oracle pins for Optimized RAS (NEXT f3; PAPER P760-763 names ORAS as future
work without a formula -- DESIGN.md R30: A~_p = A_p - robin * diag(|B_p| 1),
the local solve only).  Pinned to optimized-Schwarz theory: with the exact
Dirichlet-to-Neumann value as the Robin term, two overlapping subdomains of the
1D Laplacian converge in two sweeps."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
import ras_inputs as ri


def lap1d(n):
    A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    A.sort_indices()
    return A


def iterate(A, b, owner, gamma, robin, K, kind="exact"):
    subs = O.setup(A, b, owner, gamma, robin=robin)
    for s in subs:
        O.make_local_solver(s, kind, 20)
    return O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)


def test_robin_zero_is_ras():
    N = 24
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    own = O.partition_regular(N, N, 1, 2, 2, 1)
    r0 = iterate(A, b, own, 2, 0.0, 3)
    subs = O.setup(A, b, own, 2)
    for s in subs:
        O.make_local_solver(s, "exact")
    r1 = O.ras_sync(A, b, subs, 1e-300, 3, record_iterates=True)
    assert all(np.array_equal(r0.iterates[k], r1.iterates[k]) for k in range(4))


@pytest.mark.parametrize("gamma", [1, 2, 3])
def test_exact_dtn_robin_converges_in_two_sweeps(gamma):
    # 1D, two subdomains of 20 owned rows: Omega_0 = rows 0..19+gamma, and the
    # m = 20 - gamma rows outside it (Dirichlet end) have the Schur complement
    # (A_out^-1)_00 = m / (m + 1): a Robin term robin = m/(m+1) makes A~_p the
    # exact Schur complement (symmetric for both subdomains) -> exact after 2 sweeps
    n = 40
    A = lap1d(n)
    b = np.random.default_rng(0).uniform(-1, 1, n)
    owner = np.array([0] * 20 + [1] * 20)
    xs = np.linalg.solve(A.toarray(), b)
    m = 20 - gamma
    ex = iterate(A, b, owner, gamma, m / (m + 1), 2)
    ras = iterate(A, b, owner, gamma, 0.0, 2)
    err = lambda x: np.linalg.norm(x - xs) / np.linalg.norm(xs)  # noqa: E731
    assert err(ex.iterates[2]) <= 1e-12
    assert err(ras.iterates[2]) >= 1e-2


def test_local_matrix_closed_form():
    # 2x2 tiles of a 32^2 Laplacian, overlap 2: every row of Omega_0 drops one
    # coupling per grid neighbour (4-neighbourhood, inside the grid) that is not
    # in Omega_0: A~_ii = 4 - robin * dropped, counted here from the grid geometry
    N, g, w = 32, 2, 0.4
    A = ri.laplace_2d(N)
    own = O.partition_regular(N, N, 1, 2, 2, 1)
    s0 = O.setup(A, np.zeros(N * N), own, g, robin=w)[0]
    d = s0.Asolve.diagonal()
    inside = np.zeros((N, N), bool)
    inside[s0.omega // N, s0.omega % N] = True
    dropped = np.zeros(len(s0.omega), int)
    for k, gid in enumerate(s0.omega):
        y, x = divmod(int(gid), N)
        for yy, xx in ((y - 1, x), (y + 1, x), (y, x - 1), (y, x + 1)):
            if 0 <= yy < N and 0 <= xx < N and not inside[yy, xx]:
                dropped[k] += 1
    assert dropped.max() == 2 and (dropped == 1).sum() > 0
    np.testing.assert_array_equal(d, 4.0 - w * dropped)
    assert (s0.Asolve - s0.A).count_nonzero() == int((dropped > 0).sum())  # off-diagonals untouched


def test_robin_accelerates_2d():
    N = 32
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    own = O.partition_regular(N, N, 1, 2, 2, 1)
    sweeps = {}
    for w in (0.0, 0.6):
        subs = O.setup(A, b, own, 2, robin=w)
        for s in subs:
            O.make_local_solver(s, "exact")
        res = O.ras_sync(A, b, subs, 1e-8, 2000)
        assert O.verify_global(A, res.x, b, 1e-8)[0]  # converges to the solution of A x = b
        sweeps[w] = res.sweeps
    assert sweeps[0.6] < 0.8 * sweeps[0.0], sweeps
