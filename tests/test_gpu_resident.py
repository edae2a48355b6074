"""RESIDENT local-solve path (k_resident_pcg) on matrices that are not stencils.

The row-pattern dictionary SpMV applies when every chunk of a subdomain has at
most 128 distinct rows (interior / edge / corner rows of a stencil).  A
variable-coefficient diffusion (ras_inputs.varcoef_2d: few distinct values,
hundreds of distinct rows per chunk) keeps the matrix SELL-Z-compressible but
forces the other branch: the SELL-Z stream from L2.  Iterates must match the
oracle within 1e-10 (north_star FP64 tolerance) on both branches."""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("matrix,pattern", [("varcoef", 0), ("laplace", 1)])
@pytest.mark.parametrize("part", ["regular", "voronoi"])
def test_resident_branches_match_oracle(matrix, pattern, part):
    nx, ny = 240, 220
    A = ri.varcoef_2d(nx, ny, seed=7) if matrix == "varcoef" else ri.laplace_2d(nx, ny)
    b = ri.rhs(A.n, 0)
    owner = O.partition_regular(nx, ny, 1, 2, 2, 1) if part == "regular" else ri.voronoi_partition(nx, ny, 5, seed=3)
    gamma, m = 3, 10
    subs = O.setup(A, b, owner, gamma)
    for s in subs:
        O.make_local_solver(s, "jacobi", m)
    ref = O.ras_sync(A, b, subs, 1e-300, 3, record_iterates=True)
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, path="resident"))
    for k in (1, 3):
        st, x = s.solve(1e-300, k, "sync")
        t = s.stats()
        assert t["pcg_path"] == 3 and t["resident_pattern"] == pattern, t
        assert rel(x, ref.iterates[k]) <= 1e-10, (matrix, part, k, rel(x, ref.iterates[k]))
    s.close()


def test_resident_irregular_converges_sync_and_async():
    nx, ny = 260, 250
    A = ri.varcoef_2d(nx, ny, seed=11)
    b = ri.rhs(A.n, 0)
    owner = O.partition_regular(nx, ny, 1, 2, 2, 1)
    s = R.Solver(A, b, owner, 4, R.options("jacobi", 12))
    for mode in ("sync", "async"):
        st, x = s.solve(1e-8, 50000, mode)
        t = s.stats()
        assert st == 0 and t["pcg_path"] == 3 and t["resident_pattern"] == 0, (mode, t)
        assert O.verify_global(A, x, b, 1e-8)[0]
    s.close()
