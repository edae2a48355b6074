"""Oracle pins: local solvers (P309-323).

* Cholesky against SPEC's worked example and dense LU (numpy.linalg.solve);
* PCG against the Krylov-optimality characterisation of CG (the m-th PCG
  iterate minimises the A-norm error over x0 + K_m(M^-1 A, M^-1 r0)), computed
  by a Galerkin projection — a sign/index slip in the recurrences breaks it;
* IC(0) against the closed-form 5-point recurrence and, on a tridiagonal
  matrix, against exact Cholesky (IC(0) has no dropped fill there);
* ILU(0) on a tridiagonal matrix against scipy's LU;
* level counts against nx+ny-1 (2D) / nx+ny+nz-2 (3D)."""
import math

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import oracle as O
import ras_inputs as ri


def test_cholesky_spec_example():
    F = O.cholesky_factor(sp.csr_matrix(np.array([[4.0, -1], [-1, 4]])))
    L = F[1]
    assert np.allclose(L, [[2, 0], [-0.5, math.sqrt(3.75)]], atol=1e-15)  # S62
    x = O.cholesky_solve(F, np.array([3.0, 3.0]))
    assert np.allclose(x, [1, 1], atol=1e-15)
    with pytest.raises(ValueError):
        O.cholesky_factor(sp.csr_matrix(np.array([[1.0, 2], [2, 1]])))


@pytest.mark.parametrize("n", [8, 24])
def test_exact_local_solve_vs_dense_lu(n):
    A = ri.laplace_2d(n).to_scipy()
    b = ri.rhs(n * n, 3)
    x = O.cholesky_solve(O.cholesky_factor(A), b)
    assert np.allclose(x, np.linalg.solve(A.toarray(), b), rtol=1e-12, atol=1e-13)


def test_banded_cholesky_path():
    A = ri.laplace_2d(70, 60).to_scipy()  # 4200 rows > 4096 -> banded
    F = O.cholesky_factor(A)
    assert F[0] == "banded"
    b = ri.rhs(4200, 1)
    x = O.cholesky_solve(F, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12


def _krylov_optimal(A, minv, r0, m):
    """argmin_{d in K_m} ||d - A^-1 r0||_A via Galerkin projection on an
    orthonormalised Krylov basis of M^-1 A."""
    n = len(r0)
    V = np.zeros((n, m))
    v = minv(r0)
    for j in range(m):
        for i in range(j):
            v = v - (V[:, i] @ v) * V[:, i]
        v = v / np.linalg.norm(v)
        V[:, j] = v
        v = minv(A @ v)
    G = V.T @ (A @ V)
    return V @ np.linalg.solve(G, V.T @ r0)


@pytest.mark.parametrize("m", [1, 2, 3, 5])
def test_pcg_krylov_optimality_jacobi(m):
    rng = np.random.default_rng(7)
    A = ri.laplace_2d(9, 7).to_scipy() + sp.diags(rng.uniform(0, 3, 63))
    A = A.tocsr()
    dinv = 1.0 / A.diagonal()
    r0 = rng.uniform(-1, 1, 63)
    d, it = O.pcg(A, lambda r: dinv * r, r0, m)
    assert it == m
    ref = _krylov_optimal(A, lambda r: dinv * r, r0, m)
    assert np.linalg.norm(d - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_krylov_optimality_ic0():
    A = ri.laplace_2d(8, 6).to_scipy()
    L = O.ic0(A)
    Lt = L.T.tocsr()
    import scipy.sparse.linalg as spla

    def minv(r):
        return spla.spsolve_triangular(Lt, spla.spsolve_triangular(L, r, lower=True), lower=False)

    r0 = ri.rhs(48, 4)
    for m in (1, 3, 4):
        d, _ = O.pcg(A, minv, r0, m)
        ref = _krylov_optimal(A, minv, r0, m)
        assert np.linalg.norm(d - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_converges_to_direct_and_spec_cg_example():
    A = ri.laplace_2d(8).to_scipy()  # S81: CG on laplace(8) matches Cholesky to 1e-8
    b = ri.rhs(64, 0)
    d, it = O.pcg(A, lambda r: 0.25 * r, b, 10 * 64, inner_tol=1e-14)
    x = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(d - x) <= 1e-10 * np.linalg.norm(x)
    assert it < 64


def test_pcg_breakdown_guards():
    A = ri.laplace_2d(4).to_scipy()
    d, it = O.pcg(A, lambda r: 0.25 * r, np.zeros(16), 5)
    assert it == 0 and not d.any()  # rho == 0 -> keep d (R7)


def test_ic0_closed_form_5pt_recurrence():
    nx, ny = 7, 5
    A = ri.laplace_2d(nx, ny).to_scipy()
    L = O.ic0(A).toarray()
    n = nx * ny
    d = np.zeros(n)
    Ad = A.toarray()
    for i in range(n):
        s = Ad[i, i]
        for j in (i - 1, i - nx):
            if j >= 0 and Ad[i, j] != 0:
                s -= (Ad[i, j] / d[j]) ** 2
        d[i] = math.sqrt(s)
    Lref = np.diag(d)
    for i in range(n):
        for j in (i - 1, i - nx):
            if j >= 0 and Ad[i, j] != 0:
                Lref[i, j] = Ad[i, j] / d[j]
    assert np.abs(L - Lref).max() < 1e-15


def test_ic0_tridiagonal_is_cholesky():
    rng = np.random.default_rng(1)
    n = 40
    main = rng.uniform(3, 5, n)
    off = rng.uniform(-1, 1, n - 1)
    T = sp.diags([off, main, off], [-1, 0, 1]).tocsr()
    L = O.ic0(T).toarray()
    assert np.abs(L - np.linalg.cholesky(T.toarray())).max() < 1e-14


def test_ilu0_tridiagonal_is_lu_and_matches_ic0_scaling():
    rng = np.random.default_rng(2)
    n = 30
    main = rng.uniform(3, 5, n)
    off = rng.uniform(-1, 1, n - 1)
    T = sp.diags([off, main, off], [-1, 0, 1]).tocsr()
    L, U = O.ilu0(T)
    P_, Ls, Us = sla.lu(T.toarray())
    assert np.allclose(P_, np.eye(n))
    assert np.abs(L.toarray() - Ls).max() < 1e-14 and np.abs(U.toarray() - Us).max() < 1e-13
    # R10: for SPD A, ILU(0) = IC(0) up to diagonal scaling: U = D L^T, D = diag(L)
    A = ri.laplace_2d(6, 5).to_scipy()
    Lic = O.ic0(A).toarray()
    L2, U2 = O.ilu0(A)
    D = np.diag(np.diag(Lic))
    assert np.abs(U2.toarray() - D @ Lic.T).max() < 1e-13
    assert np.abs(L2.toarray() - Lic @ np.linalg.inv(D)).max() < 1e-13


def test_level_counts():
    L2 = O.ic0(ri.laplace_2d(40, 24).to_scipy())
    assert O.level_sets(L2).max() + 1 == 40 + 24 - 1
    assert O.level_sets(L2.T.tocsr(), lower=False).max() + 1 == 63
    L3 = O.ic0(ri.laplace_3d(6, 5, 4).to_scipy())
    assert O.level_sets(L3).max() + 1 == 6 + 5 + 4 - 2
