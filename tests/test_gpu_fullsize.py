"""Full-size parity at the bench configuration (BASELINE.json configs[1], C2).

C2: 2D 5-point Laplacian 4096^2 (16.8 M unknowns), 16 subdomains of 1024^2,
overlap 8, Jacobi-PCG m = 20, sync RAS -- the same problem, options and local-solve
path (AUTO -> RESIDENT) that bench.py times.  The oracle cannot run whole sweeps
at this size in seconds, so the first sweep is checked on SAMPLED subdomains: from
x^0 = 0 every subdomain of the synchronous sweep sees x^0, so x^1[S_p] = delta_p[S_p]
with delta_p = PCG_m(A_p, R_p b) (P147-153 restricted prolongation, P309-315 local
solve), which the oracle computes one subdomain at a time.  Later sweeps are checked
through a property that holds at any size: the reported true relative residual of
the returned iterate equals ||b - A x|| / ||b|| recomputed on the host.

Bar: 1e-10 relative (north_star FP64 tolerance, as in test_gpu_sync.py).
"""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")

NX = NY = 4096
PX = PY = 4
GAMMA = 8
M = 20
SAMPLE = [0, 1, 5, 15]  # corner, edge, interior, opposite corner


@pytest.fixture(scope="module")
def c2():
    A = ri.laplace_2d(NX, NY)
    b = ri.rhs(NX * NY, 0)
    owner = R.partition_regular(NX, NY, 1, PX, PY, 1)
    s = R.Solver(A, b, owner, GAMMA, R.options("jacobi", M), comm={"rank": 0, "world": 1, "device": 0})
    yield A, b, owner, s
    s.close()


def test_c2_first_sweep_matches_oracle_on_sampled_subdomains(c2):
    A, b, owner, s = c2
    st, x1 = s.solve(1e-300, 1, "sync")
    assert s.stats()["sweeps"] == 1
    assert s.stats()["pcg_path"] == 3  # RESIDENT, the path bench.py times (ras_pcg_path)
    As = O.as_scipy(A)
    zero = np.zeros(NX * NY)
    oowner = O.partition_regular(NX, NY, 1, PX, PY, 1)
    assert np.array_equal(np.asarray(owner), oowner)
    for p in SAMPLE:
        om, ow, gh = O.overlap_sets(As, oowner, p, GAMMA)
        rows = As[om]
        sub = O.Subdomain(p, om, ow, gh, rows[:, om].tocsr(), rows[:, gh].tocsr(), b[om].copy())
        O.make_local_solver(sub, "jacobi", M)
        d = sub.solver(O.local_residual(sub, zero))
        ref = d[sub.owned]
        got = x1[sub.owned_global]
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert err <= 1e-10, (p, err)
        assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref)), p


def test_c2_reported_residual_matches_host_recomputation(c2):
    A, b, owner, s = c2
    st, x = s.solve(1e-300, 3, "sync")
    stats = s.stats()
    assert stats["sweeps"] == 3
    As = O.as_scipy(A)
    host = np.linalg.norm(b - As @ x) / np.linalg.norm(b)
    assert abs(stats["final_rel_residual"] - host) <= 1e-10 * host
    assert host < 1.0


def test_c2_second_sweep_matches_oracle_on_interior_subdomain(c2):
    # sweep 2 element by element on the interior subdomain p = 5: x^2[S_p] =
    # x^1[S_p] + delta_p[S_p], delta_p = PCG_m(A_p, r~_p(x^1)), where x^1 on
    # Omega_p u Gamma_p comes from the first-sweep local solves of p and of its
    # eight neighbours (every owner of a value p reads; P147-153, P294-297)
    A, b, owner, s = c2
    st, x2 = s.solve(1e-300, 2, "sync")
    assert s.stats()["sweeps"] == 2
    As = O.as_scipy(A)
    oowner = O.partition_regular(NX, NY, 1, PX, PY, 1)
    zero = np.zeros(NX * NY)

    def sub_of(q):
        om, ow, gh = O.overlap_sets(As, oowner, q, GAMMA)
        rows = As[om]
        sb = O.Subdomain(q, om, ow, gh, rows[:, om].tocsr(), rows[:, gh].tocsr(), b[om].copy())
        O.make_local_solver(sb, "jacobi", M)
        return sb

    p = 5
    # owners of Omega_5 u Gamma_5: p and its 8 neighbours in the 4x4 block grid
    sp_ = sub_of(p)
    need = np.concatenate([sp_.omega, sp_.ghosts])
    owners = np.unique(oowner[need])
    assert len(owners) == 9
    x1 = np.zeros(NX * NY)
    for q in owners:
        sq = sp_ if q == p else sub_of(q)
        d = sq.solver(O.local_residual(sq, zero))
        x1[sq.owned_global] = d[sq.owned]
    d2 = sp_.solver(O.local_residual(sp_, x1))
    ref = x1[sp_.owned_global] + d2[sp_.owned]
    got = x2[sp_.owned_global]
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-10, err
