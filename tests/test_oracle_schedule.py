"""Oracle pins: asynchronous update schedules (ras_schedule; P163-176).

Pinned against (i) the synchronous sweep (a schedule whose steps contain every
subdomain is ras_sync's double-buffered sweep), (ii) the exact solve (one
subdomain, no overlap: one update solves A x = b), (iii) the textbook
alternating Schwarz contraction of two overlapping 1D subdomains with exact
local solves, a closed form (error at the interface shrinks by
(a-g)(n-a-g) / ((a+g+1)(n+1-a+g)) per round for the 1D Laplacian, Schwarz 1870 /
Lions 1988), and (iv) brute force: the sequential schedule equals an explicit
Gauss-Seidel-ordered loop over dense local solves on a tiny grid."""
import numpy as np

import oracle as O
import ras_inputs as ri


def _subs(A, b, owner, gamma, kind="exact", m=0):
    subs = O.setup(A, b, owner, gamma)
    for s in subs:
        O.make_local_solver(s, kind, m)
    return subs


def test_all_in_one_step_is_the_sync_sweep():
    N = 24
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 1)
    owner = O.partition_regular(N, N, 1, 2, 3, 1)
    subs = _subs(A, b, owner, 2, "jacobi", 7)
    K = 4
    ref = O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)
    x = O.ras_schedule(A, b, subs, [list(range(len(subs)))] * K)
    np.testing.assert_array_equal(x, ref.iterates[K])


def test_single_subdomain_update_is_the_exact_solve():
    N = 12
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 2)
    subs = _subs(A, b, np.zeros(N * N, np.int32), 0)
    x = O.ras_schedule(A, b, subs, [[0]])
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) < 1e-12


def test_alternating_schwarz_1d_closed_form():
    # 1D Laplacian tridiag(-1, 2, -1) on n points, b = 0, x0 = ones: the error is
    # harmonic (linear) inside each subdomain, so one exact solve maps the value at
    # the far interface node linearly.  Subdomain 0 owns rows [0, a), subdomain 1
    # [a, n); with overlap g, Omega_0 = [0, a+g), Omega_1 = [a-g, n).  One
    # sequential round (0 then 1) multiplies the error at node a-1 by
    #   rho = (a - g) (n - a - g) / ((a + g + 1) (n + 1 - a + g))   (1-based
    # distances to the Dirichlet ends), so two rounds give rho^2.
    n, a, g = 40, 20, 3
    main = 2.0 * np.ones(n)
    off = -np.ones(n - 1)
    import scipy.sparse as sp

    A = sp.diags([off, main, off], [-1, 0, 1]).tocsr()
    Ac = ri.CSR(A.indptr, A.indices, A.data, n)
    b = np.zeros(n)
    owner = np.array([0] * a + [1] * (n - a), np.int32)
    subs = _subs(Ac, b, owner, g)
    x0 = np.ones(n)
    x1 = O.ras_schedule(Ac, b, subs, [[0], [1]], x0=x0)
    x2 = O.ras_schedule(Ac, b, subs, [[0], [1]], x0=x1)
    rho = (a - g) * (n - a - g) / ((a + g + 1) * (n + 1 - a + g))
    # after subdomain 1 solves, the error on [a-g, n) is linear from x[a-g-1] to 0
    assert abs(x2[a - 1] / x1[a - 1] - rho) < 1e-12


def test_sequential_schedule_is_gauss_seidel_ordered_loop_brute_force():
    N = 10
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 3)
    owner = O.partition_regular(N, N, 1, 2, 2, 1)
    subs = _subs(A, b, owner, 1)
    Ad = A.to_scipy().toarray()
    x = np.zeros(N * N)
    for _ in range(3):
        for s in subs:  # dense restricted solve, in place: the multiplicative order
            om = s.omega
            r = b[om] - Ad[om] @ x
            d = np.linalg.solve(Ad[np.ix_(om, om)], r)
            x[om[s.owned]] += d[s.owned]
    y = O.ras_schedule(A, b, subs, [[p] for p in range(len(subs))] * 3)
    assert np.linalg.norm(x - y) / np.linalg.norm(x) < 1e-12
