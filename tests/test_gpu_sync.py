"""GPU parity of the synchronous RAS path against the oracle, through the C ABI.

Bar (BASELINE.json north_star): sync iterates within 1e-10 relative (FP64),
converged solutions reach true relative residual <= tol, index maps bit-exact.
"""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def oracle_iterates(A, b, owner, gamma, kind, m, k, inner_tol=0.0):
    subs = O.setup(A, b, owner, gamma)
    for s in subs:
        O.make_local_solver(s, kind, m, inner_tol)
    return O.ras_sync(A, b, subs, 1e-300, k, record_iterates=True)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("fmt", ["plain", "z", "fuse_p", "stage", "z_stage", "tiled", "plain_tiled", "resident",
                                 "plain_resident"])
@pytest.mark.parametrize("case", ["c1", "voronoi_ragged", "strips"])
def test_sync_iterates_match_oracle(case, fmt):
    if case == "c1":
        nx = ny = 64
        A = ri.laplace_2d(nx)
        owner = R.partition_regular(nx, ny, 1, 2, 2, 1)
        gamma, m = 2, 20
    elif case == "voronoi_ragged":
        nx, ny = 203, 157  # several 256-row tiles per subdomain and ragged tails
        A = ri.laplace_2d(nx, ny)
        owner = ri.voronoi_partition(nx, ny, 7, seed=4)
        gamma, m = 3, 15
    else:
        nx, ny = 96, 64
        A = ri.laplace_2d(nx, ny)
        owner = R.partition_regular(nx, ny, 1, 1, 5, 1)
        gamma, m = 1, 7
    b = ri.rhs(nx * ny, 0)
    K = 6
    ref = oracle_iterates(A, b, owner, gamma, "jacobi", m, K)
    path = "resident" if fmt.endswith("resident") else "tiled" if fmt.endswith("tiled") or "stage" in fmt else "auto"
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, fuse_p=fmt == "fuse_p", plain=fmt.startswith("plain") or fmt == "stage",
                                              stage=fmt.endswith("stage"), path=path))
    for k in (1, 2, K):
        st, x = s.solve(1e-300, k, "sync")
        assert st == R._ffi.RAS_ENOCONV
        assert s.stats()["sweeps"] == k
        if path != "auto":
            assert s.stats()["pcg_path"] == getattr(R._ffi, "RAS_PCG_" + path.upper())
        assert rel(x, ref.iterates[k]) <= 1e-10, (case, k, rel(x, ref.iterates[k]))
    s.close()


def test_sync_converges_to_tolerance_and_matches_oracle_solution():
    N = 64
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = R.partition_regular(N, N, 1, 2, 2, 1)
    s = R.Solver(A, b, owner, 2, R.options("jacobi", 20))
    st, x = s.solve(1e-8, 5000, "sync")
    assert st == R._ffi.RAS_OK
    ok, relres = O.verify_global(A, x, b, 1e-8)
    assert ok
    st_ = s.stats()
    assert abs(st_["final_rel_residual"] - relres) <= 1e-12 + 1e-6 * relres
    subs = O.setup(A, b, owner, 2)
    for sb in subs:
        O.make_local_solver(sb, "jacobi", 20)
    ref = O.ras_sync(A, b, subs, 1e-8, 5000)
    assert st_["sweeps"] == ref.sweeps
    assert rel(x, ref.x) <= 1e-10
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    assert rel(x, xs) <= 1e-6  # R25 (N <= 256)
    s.close()


@pytest.mark.parametrize("path", ["auto", "tiled", "resident"])
def test_exact_mode_c1_sweeps_and_solution(path):
    # C1: 64x64, 2x2, overlap 2, "exact" local solve (PCG to 1e-14, R6): 106 sweeps (oracle)
    N = 64
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = R.partition_regular(N, N, 1, 2, 2, 1)
    subs = O.setup(A, b, owner, 2)
    for sb in subs:
        O.make_local_solver(sb, "exact")
    ref = O.ras_sync(A, b, subs, 1e-8, 1000, record_iterates=True)
    assert ref.sweeps == 106
    s = R.Solver(A, b, owner, 2, R.options("exact", path=path))
    for k in (1, 5):
        st, x = s.solve(1e-300, k, "sync")
        assert rel(x, ref.iterates[k]) <= 1e-10
    st, x = s.solve(1e-8, 1000, "sync")
    assert st == R._ffi.RAS_OK
    assert s.stats()["sweeps"] == 106
    assert rel(x, ref.x) <= 1e-10
    s.close()


@pytest.mark.parametrize("plain", [False, True])
def test_resident_path_is_auto_for_medium_subdomains(plain):
    # 2x2 subdomains of ~134^2 rows (> the one-CTA limit of 9216): AUTO picks the
    # grid-resident kernel (one group of all SMs per subdomain, ragged last chunk)
    nx, ny = 262, 250
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 2)
    owner = R.partition_regular(nx, ny, 1, 2, 2, 1)
    ref = oracle_iterates(A, b, owner, 4, "jacobi", 12, 3)
    s = R.Solver(A, b, owner, 4, R.options("jacobi", 12, plain=plain))
    for k in (1, 3):
        st, x = s.solve(1e-300, k, "sync")
        assert s.stats()["pcg_path"] == R._ffi.RAS_PCG_RESIDENT
        assert s.stats()["inner_iters_total"] == 12 * 4 * k
        assert rel(x, ref.iterates[k]) <= 1e-10, (k, rel(x, ref.iterates[k]))
    s.close()


def test_forced_paths_that_do_not_apply_are_errors():
    N = 40
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N)
    owner = R.partition_regular(N, N, 1, 2, 2, 1)
    with pytest.raises(R.RasError, match="pcg_path"):
        R.Solver(A, b, owner, 1, R.options("ic0", 5, path="resident"))
    big = ri.laplace_2d(200)
    with pytest.raises(R.RasError, match="BLOCK"):
        R.Solver(big, ri.rhs(200 * 200), np.zeros(200 * 200, np.int32), 0, R.options("jacobi", 5, path="block"))


def test_edge_cases():
    N = 24
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 1)
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    # one subdomain, no overlap, exact local solve: one sweep solves (north_star invariant)
    s = R.Solver(A, b, np.zeros(N * N, np.int32), 0, R.options("exact"))
    st, x = s.solve(1e-10, 10, "sync")
    assert st == 0 and s.stats()["sweeps"] == 1 and rel(x, xs) <= 1e-12
    s.close()
    owner = R.partition_regular(N, N, 1, 3, 2, 1)
    s = R.Solver(A, b, owner, 1, R.options("jacobi", 5))
    # max_iters = 0 returns x0 and its residual
    st, x = s.solve(1e-8, 0, "sync")
    assert st == R._ffi.RAS_ENOCONV and not x.any() and abs(s.stats()["final_rel_residual"] - 1.0) < 1e-14
    # x0 = exact solution: converged at sweep 0
    st, x = s.solve(1e-8, 10, "sync", x0=xs)
    assert st == 0 and s.stats()["sweeps"] == 0 and np.array_equal(x, xs)
    s.close()
    # b = 0 -> x = 0 converged immediately (R11)
    s = R.Solver(A, np.zeros(N * N), owner, 1, R.options("jacobi", 5))
    st, x = s.solve(1e-8, 10, "sync")
    assert st == 0 and not x.any()
    s.close()


def test_errors_are_reported():
    N = 8
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N)
    owner = np.zeros(N * N, np.int32)
    owner[5] = 3  # subdomains 1, 2 empty
    with pytest.raises(R.RasError, match="empty"):
        R.Solver(A, b, owner, 1)
    with pytest.raises(R.RasError, match="overlap"):
        R.Solver(A, b, np.zeros(N * N, np.int32), -1)
    B = ri.laplace_2d(N)
    B.data[B.indptr[3]:B.indptr[4]] *= -1.0  # negative diagonal in row 3
    with pytest.raises(R.RasError, match="RAS_ENOTSPD.*subdomain 0"):
        R.Solver(B, b, np.zeros(N * N, np.int32), 1)


def test_non_compressible_matrix_takes_plain_path():
    # > 256 distinct values: the SELL-Z dictionary does not apply, plain FP64 SELL is used
    N = 40
    A = ri.laplace_2d(N)
    rng = np.random.default_rng(3)
    A.data = A.data * (1.0 + 0.01 * rng.random(A.nnz))
    As = A.to_scipy()
    As = ((As + As.T) * 0.5).tocsr()
    As.sort_indices()
    A2 = ri.CSR(As.indptr, As.indices, As.data, N * N)
    owner = R.partition_regular(N, N, 1, 2, 2, 1)
    s = R.Solver(A2, ri.rhs(N * N), owner, 2, R.options("jacobi", 8))
    assert s.plan().info()["z_format"] == 0
    ref = oracle_iterates(A2, ri.rhs(N * N), owner, 2, "jacobi", 8, 3)
    st, x = s.solve(1e-300, 3, "sync")
    assert rel(x, ref.iterates[3]) <= 1e-10
    s.close()


def test_block_path_with_d_in_l2():
    # subdomains of 9216..14336 padded rows: the one-CTA kernel keeps p, r in
    # shared memory and the correction d in L2
    nx, ny = 150, 150
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 4)
    owner = R.partition_regular(nx, ny, 1, 1, 2, 1)  # 150 x 75 + overlap 3 = 11700 rows
    ref = oracle_iterates(A, b, owner, 3, "jacobi", 15, 3)
    s = R.Solver(A, b, owner, 3, R.options("jacobi", 15, path="block"))
    for k in (1, 3):
        st, x = s.solve(1e-300, k, "sync")
        assert s.stats()["pcg_path"] == R._ffi.RAS_PCG_BLOCK
        assert rel(x, ref.iterates[k]) <= 1e-10, (k, rel(x, ref.iterates[k]))
    st, x = s.solve(1e-8, 50000, "async")
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0]
    s.close()


@pytest.mark.parametrize("pairs", ["0", "1"])
def test_async_sequential_schedule_on_resident_subdomains(pairs, monkeypatch):
    # R34: RESIDENT-sized subdomains in async mode on one GPU run on one stream,
    # one after another (RAS_ASYNC_PAIRS=0) or two at a time (default) -- legal
    # asynchronous schedules: converge, verify, and need fewer updates than sync sweeps
    monkeypatch.setenv("RAS_ASYNC_PAIRS", pairs)
    nx, ny = 262, 250
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 2)
    owner = R.partition_regular(nx, ny, 1, 2, 2, 1)
    s = R.Solver(A, b, owner, 4, R.options("jacobi", 12))
    st, x = s.solve(1e-8, 100000, "sync")
    sync_sweeps = s.stats()["sweeps"]
    st, x = s.solve(1e-8, 100000, "async")
    stt = s.stats()
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0], stt
    assert stt["updates_max"] < sync_sweeps, (stt["updates_max"], sync_sweeps)
    s.close()


def test_async_paired_resident_updates_match_oracle_schedule(monkeypatch):
    # R34 (default): RESIDENT-sized subdomains updated two at a time, both reading
    # the latest data -- the asynchronous schedule [[0, 1], [2, 3]] per round,
    # written out by oracle.ras_schedule (P163-176)
    monkeypatch.delenv("RAS_ASYNC_PAIRS", raising=False)
    nx, ny, m, K = 262, 250, 12, 3
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 2)
    owner = R.partition_regular(nx, ny, 1, 2, 2, 1)
    subs = O.setup(A, b, owner, 4)
    for sd in subs:
        O.make_local_solver(sd, "jacobi", m)
    ref = O.ras_schedule(A, b, subs, [[0, 1], [2, 3]] * K)
    s = R.Solver(A, b, owner, 4, R.options("jacobi", m, max_resumes=0))
    st, x = s.solve(1e-300, K, "async")
    assert s.stats()["pcg_path"] == 3, s.stats()["pcg_path"]
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-10, np.linalg.norm(x - ref) / np.linalg.norm(ref)
    s.close()
