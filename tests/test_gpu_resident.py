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


@pytest.mark.parametrize("kernel", ["v1", "v2"])
@pytest.mark.parametrize("shape", ["c2like", "many_pairs", "big_chunks", "odd_count"])
def test_resident_kernels_match_oracle(kernel, shape, monkeypatch):
    # k_resident_pcg (v1: r, d in shared memory) and k_resident2 (v2: r, d in tensor
    # memory; two subdomains interleaved per CTA when they fit, else one lane with
    # chunks up to 512 x 24 rows) on row-pattern matrices, 1e-10 vs the oracle
    if kernel == "v1":
        if shape == "big_chunks":
            pytest.skip("v1 holds at most 768 x 10 rows per CTA")
        monkeypatch.setenv("RAS_RESIDENT_KERNEL", "1")
    else:
        monkeypatch.delenv("RAS_RESIDENT_KERNEL", raising=False)
    if shape == "c2like":    # 4 x 4 subdomains of 256^2 (+ overlap): two lanes per CTA
        N, px, gamma, m, owner = 1024, 4, 8, 20, None
    elif shape == "many_pairs":  # 4 x 4 subdomains of 512^2: 4 groups of 37 CTAs, two pairs each (lanes reused)
        N, px, gamma, m, owner = 2048, 4, 8, 8, None
    elif shape == "big_chunks":  # one subdomain of 1300^2 rows on the whole GPU: one lane, > 7.7 K rows per CTA
        N, px, gamma, m, owner = 1300, 1, 0, 6, None
    else:                    # 5 strips: the last pair has one live lane
        N, px, gamma, m = 600, 0, 3, 8
        owner = O.partition_regular(N, N, 1, 1, 5, 1)
    A = ri.laplace_2d(N)
    b = ri.rhs(A.n, 0)
    if owner is None:
        owner = O.partition_regular(N, N, 1, px, px, 1)
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, path="resident"))
    K = 2
    st, x = s.solve(1e-300, K, "sync")
    t = s.stats()
    assert t["pcg_path"] == 3 and t["resident_pattern"] == 1, t
    if kernel == "v1":
        assert t["resident_lanes"] == 0
    else:
        assert t["resident_lanes"] == (1 if shape == "big_chunks" else 2), t
    s.close()
    # oracle: sampled subdomains at the larger sizes would be slow; the whole
    # problem at these sizes runs in seconds with scipy
    subs = O.setup(A, b, owner, gamma)
    for sb in subs:
        O.make_local_solver(sb, "jacobi", m)
    ref = O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)
    assert rel(x, ref.iterates[K]) <= 1e-10, rel(x, ref.iterates[K])


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


@pytest.mark.parametrize("lanes_case", ["one_lane_big_cells", "two_lanes"])
def test_resident2_sell_z_stream_on_voronoi_cells(lanes_case):
    # Voronoi cells: hundreds of distinct rows per chunk -> k_resident2 without the
    # row-pattern table, the SELL-Z local matrix streamed from L2 (the C5 path)
    if lanes_case == "one_lane_big_cells":
        # one 1.69 M-row subdomain of the variable-coefficient matrix: one lane,
        # chunks of ~11.4 K rows, never a row-pattern table
        N, P, gamma, m = 1300, 1, 0, 6
        A = ri.varcoef_2d(N, N, seed=5)
        owner = np.zeros(N * N, np.int32)
    else:
        N, P, gamma, m = 700, 6, 3, 8
        A = ri.laplace_2d(N)
        owner = ri.voronoi_partition(N, N, P, seed=2, lloyd=4, balance=40)
    b = ri.rhs(A.n, 0)
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, path="resident"))
    K = 2
    st, x = s.solve(1e-300, K, "sync")
    t = s.stats()
    assert t["pcg_path"] == 3 and t["resident_pattern"] == 0 and t["resident_lanes"] >= 1, t
    s.close()
    subs = O.setup(A, b, owner, gamma)
    for sb in subs:
        O.make_local_solver(sb, "jacobi", m)
    ref = O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)
    assert rel(x, ref.iterates[K]) <= 1e-10, rel(x, ref.iterates[K])
