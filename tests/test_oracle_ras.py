"""Oracle pins: the RAS operator and the synchronous iteration (P144-161, Alg. 1).

* P=1, gamma=0 -> one sweep is the exact solve (north_star invariant; S500);
* saturated overlap -> one sweep; fixed point x0 = x* (S492, S525);
* closed-form two-strip contraction factor (separable Laplacian, exact solves);
* regression sweep counts measured by an independent scratch probe (SURVEY
  Appendix: SciPy splu local solves) and the qualitative paper/SPEC claims
  (monotone in overlap, regular1d growth with P, P277-282, P574-586);
* verification criterion (P344-348) and error vs the exact solution (R25)."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle as O
import ras_inputs as ri


def run(N, owner, gamma, kind="exact", tol=1e-8, max_iters=5000, b=None, x0=None, m=20, rec=False, inner_tol=0.0):
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0) if b is None else b
    subs = O.setup(A, b, owner, gamma)
    for s in subs:
        O.make_local_solver(s, kind, m, inner_tol)
    return A, b, O.ras_sync(A, b, subs, tol, max_iters, x0=x0, record_iterates=rec)


def test_single_subdomain_no_overlap_is_exact_solve():
    A, b, res = run(16, np.zeros(256, np.int32), 0, tol=1e-12)
    assert res.sweeps == 1 and res.converged
    xs = spla.spsolve(A.to_scipy().tocsc(), b)
    assert np.linalg.norm(res.x - xs) <= 1e-12 * np.linalg.norm(xs)


def test_saturated_overlap_is_one_sweep():
    A, b, res = run(12, O.partition_regular2d(12, 4), 30, tol=1e-12)
    assert res.sweeps == 1


def test_fixed_point():
    N = 16
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    xs = spla.spsolve(A.to_scipy().tocsc(), b)
    own = O.partition_regular2d(N, 4)
    for kind in ("exact", "jacobi", "ic0"):
        subs = O.setup(A, b, own, 2)
        for s in subs:
            O.make_local_solver(s, kind, 10)
        res = O.ras_sync(A, b, subs, 1e-300, 1, x0=xs)
        assert np.linalg.norm(res.x - xs) <= 1e-12 * np.linalg.norm(xs)


@pytest.mark.parametrize("N,a,g,kmode", [(32, 16, 2, 1), (32, 16, 2, 3), (24, 10, 3, 2), (20, 12, 1, 5)])
def test_two_strip_closed_form_contraction(N, a, g, kmode):
    """Error e = f(row) sin(k pi (c+1)/(N+1)); with exact solves strip 0 (rows 1..a)
    maps the error at row a+g+1 to rows <= a by sinh(theta r)/sinh(theta(a+g+1)),
    strip 1 likewise from row a-g; two sweeps multiply the error at row a+g+1 by
    rho^2 = [sinh th(a-g)/sinh th(a+g+1)] [sinh th(N-a-g)/sinh th(N+1-a+g)],
    cosh th = 2 - cos(k pi/(N+1))."""
    owner = O.partition_regular(N, N, 1, 1, 2, 1)
    if (owner.reshape(N, N)[:, 0] == 0).sum() != a:
        owner = (np.arange(N * N) // N >= a).astype(np.int32)
    c = np.arange(N)
    prof = np.random.default_rng(5).uniform(-1, 1, N)
    x0 = (prof[:, None] * np.sin(kmode * np.pi * (c[None, :] + 1) / (N + 1))).ravel()
    _, _, res = run(N, owner, g, b=np.zeros(N * N), x0=x0, tol=1e-300, max_iters=3, rec=True)
    X = [v.reshape(N, N) for v in res.iterates]
    th = math.acosh(2 - math.cos(kmode * math.pi / (N + 1)))
    rho2 = (math.sinh(th * (a - g)) / math.sinh(th * (a + g + 1))) * (math.sinh(th * (N - a - g)) / math.sinh(th * (N + 1 - a + g)))
    row = a + g  # 0-based index of 1-based row a+g+1
    big = np.abs(X[1][row]) > 1e-3 * np.abs(X[1][row]).max()  # skip nodes of the sine
    ratio = X[3][row][big] / X[1][row][big]
    assert np.allclose(ratio, rho2, rtol=1e-11, atol=0)
    if (N, a, g, kmode) == (32, 16, 2, 1):
        assert abs(rho2 - 0.3530334425563440) < 1e-15  # SURVEY §8c pin value


def test_c1_sweep_counts_regression():
    own = O.partition_regular(64, 64, 1, 2, 2, 1)
    counts = {}
    for g in (0, 1, 2, 4, 8):
        _, _, res = run(64, own, g)
        counts[g] = res.sweeps
        assert res.converged
    # independent scratch probe (SciPy splu local solves): SURVEY Appendix
    assert counts == {0: 516, 1: 176, 2: 106, 4: 59, 8: 31}


def test_regular1d_information_propagation():
    # P279-282: N subdomains need N-1 hops; iters(P=8) >= 2 iters(P=2) (S632 #6)
    it = {}
    for P in (2, 4, 8):
        _, _, res = run(64, O.partition_regular1d(64, P), 2, tol=1e-7)
        it[P] = res.sweeps
    assert it[2] < it[4] < it[8] and it[8] >= 2 * it[2]
    assert it == {2: 58, 4: 89, 8: 157}  # scratch probe, SURVEY Appendix


def test_overlap_monotone_and_solution_error():
    N = 64
    own = O.partition_regular2d(N, 6)
    prev = None
    for g in (1, 2, 4, 8):
        A, b, res = run(N, own, g, tol=1e-8)
        if prev is not None:
            assert res.sweeps < prev
        prev = res.sweeps
        ok, rel = O.verify_global(A, res.x, b, 1e-8)
        assert ok and rel < 1e-8
        xs = spla.spsolve(A.to_scipy().tocsc(), b)
        assert np.linalg.norm(res.x - xs) / np.linalg.norm(xs) <= 1e-6  # R25, N <= 256


def test_inexact_pcg_ras_converges_and_exactish_matches_exact():
    N = 32
    own = O.partition_regular2d(N, 4)
    _, _, ex = run(N, own, 2, rec=True, max_iters=8, tol=1e-300)
    _, _, pc = run(N, own, 2, kind="jacobi", m=10 * 400, inner_tol=1e-14, rec=True, max_iters=8, tol=1e-300)
    for a, b in zip(ex.iterates, pc.iterates):
        assert np.linalg.norm(a - b) <= 1e-10 * max(np.linalg.norm(a), 1e-300)
    for kind in ("jacobi", "ic0", "ilu0"):
        A, b, res = run(N, own, 2, kind=kind, m=10)
        assert res.converged and O.verify_global(A, res.x, b, 1e-8)[0]


def test_verify_global_zero_guess():
    A = ri.laplace_2d(8)
    b = ri.rhs(64, 0)
    ok, rel = O.verify_global(A, np.zeros(64), b, 1e-7)
    assert not ok and rel == 1.0


def test_max_iters_returns_last_iterate():
    own = O.partition_regular2d(16, 4)
    _, _, r3 = run(16, own, 1, max_iters=3, tol=1e-300, rec=True)
    assert not r3.converged and r3.sweeps == 3
    assert np.array_equal(r3.x, r3.iterates[3])


def test_local_convergence_criterion():
    assert O.local_converged(1e-16, 1.0, 1e-7)  # S398 example
    assert not O.local_converged(1e-14, 1.0, 1e-7)
    assert O.local_converged(0.0, 0.0, 1e-7) and not O.local_converged(1e-30, 0.0, 1e-7)
