"""NEXT f3 on the GPU: Optimized RAS (ras_options.robin, R30) against the
oracle's ORAS on every local-solve kernel path.  Bar: sync iterates within
1e-10 (FP64); converged sweep counts equal the oracle's."""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("kind,path", [("jacobi", "tiled"), ("jacobi", "block"), ("jacobi", "resident"),
                                       ("ic0", "auto"), ("cholesky", "auto"), ("exact", "auto")])
def test_oras_iterates_match_oracle(kind, path):
    nx, ny = 83, 71
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    owner = ri.voronoi_partition(nx, ny, 6, seed=4)
    gamma, m, w = 2, 10, 0.5
    subs = O.setup(A, b, owner, gamma, robin=w)
    for s in subs:
        O.make_local_solver(s, "exact" if kind == "cholesky" else kind, m)  # the oracle's direct solve
    ref = O.ras_sync(A, b, subs, 1e-300, 4, record_iterates=True)
    s = R.Solver(A, b, owner, gamma, R.options(kind, m, robin=w, path=path))
    for k in (1, 4):
        st, x = s.solve(1e-300, k, "sync")
        assert rel(x, ref.iterates[k]) <= 1e-10, (kind, path, k, rel(x, ref.iterates[k]))
    s.close()


def test_oras_converges_faster_and_matches_sweeps():
    N = 64
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = R.partition_regular(N, N, 1, 2, 2, 1)
    sweeps = {}
    for w in (0.0, 0.6):
        subs = O.setup(A, b, owner, 2, robin=w)
        for sb in subs:
            O.make_local_solver(sb, "exact")
        ref = O.ras_sync(A, b, subs, 1e-8, 1000)
        s = R.Solver(A, b, owner, 2, R.options("cholesky", robin=w))
        st, x = s.solve(1e-8, 1000, "sync")
        assert st == 0 and s.stats()["sweeps"] == ref.sweeps
        assert rel(x, ref.x) <= 1e-10
        sweeps[w] = ref.sweeps
        s.close()
    assert sweeps[0.6] < sweeps[0.0]


def test_oras_async_and_errors():
    N = 48
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = ri.voronoi_partition(N, N, 5, seed=1)
    s = R.Solver(A, b, owner, 2, R.options("jacobi", 20, robin=0.5))
    st, x = s.solve(1e-8, 20000, "async")
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0]
    s.close()
    with pytest.raises(R.RasError, match="overlap"):
        R.Solver(A, b, owner, 0, R.options("jacobi", 5, robin=0.5))
    with pytest.raises(R.RasError, match="robin"):
        R.Solver(A, b, owner, 1, R.options("jacobi", 5, robin=1.0))
