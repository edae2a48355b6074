"""GPU asynchronous RAS through the C ABI.

* detectors (P331-357): in the scripted lock-step mode the per-subdomain stop
  sweeps must equal the oracle's level-flag simulation exactly, for the
  centralized tree and the decentralized spanning-tree saturation;
* true async runs (independent per-subdomain streams, no barriers): the
  verified true relative residual reaches tol and the solution lies within
  1e-6 of the exact one (N <= 256, R25).  Async iterates themselves are
  non-reproducible by design (P170-172): parity unpinned, end state pinned.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def problem(nx, ny, P, seed=0, voronoi=True):
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, seed)
    owner = ri.voronoi_partition(nx, ny, P, seed=3) if voronoi else O.partition_regular(nx, ny, 1, 2, P // 2, 1)
    return A, b, owner


@pytest.mark.parametrize("detector", ["central", "decentral"])
@pytest.mark.parametrize("pattern", ["all_from", "random", "retract"])
def test_scripted_detector_matches_oracle(detector, pattern):
    A, b, owner = problem(48, 40, 7)
    P = 7
    K = 40
    rng = np.random.default_rng(1)
    if pattern == "all_from":
        flags = np.zeros((K, P), bool)
        flags[5:] = True
    elif pattern == "random":
        flags = rng.random((K, P)) < 0.85
        flags[25:] = True
    else:
        flags = np.ones((K, P), bool)
        flags[:12, 3] = False
        flags[14:16, 3] = False
        flags[:3, 5] = False
    s = R.Solver(A, b, owner, 2, R.options("jacobi", 3, detector=detector, scripted_flags=1))
    s.set_scripted_flags(flags.astype(np.uint8))
    st, _ = s.solve(1e-8, K + 5, "async")
    stops = s.detector_stops()
    subs = O.setup(A, b, owner, 2)
    if detector == "central":
        parent = O.default_central_tree([0] * P)
        want = O.detector_sim_centralized(parent, flags)
    else:
        parent = O.bfs_tree(O.subdomain_graph(subs, owner))
        want = O.detector_sim_decentralized(parent, flags)
    assert stops.tolist() == want, (stops.tolist(), want)
    s.close()


@pytest.mark.parametrize("detector", ["central", "decentral"])
@pytest.mark.parametrize("owned_only", [0, 1])
def test_async_converges_verified(detector, owned_only):
    nx, ny, P = 64, 64, 6
    A, b, owner = problem(nx, ny, P)
    s = R.Solver(A, b, owner, 4, R.options("jacobi", 10, detector=detector, local_crit_owned_only=owned_only))
    st, x = s.solve(1e-8, 20000, "async")
    assert st == R._ffi.RAS_OK, R._ffi.STATUS_NAMES[st]
    ok, rel = O.verify_global(A, x, b, 1e-8)
    assert ok
    stats = s.stats()
    assert stats["converged"] == 1 and stats["verified"] == 1
    assert abs(stats["final_rel_residual"] - rel) <= 1e-6 * rel + 1e-15
    upd = s.update_counts()
    assert (upd >= 1).all() and stats["updates_max"] == upd.max() and stats["updates_min"] == upd.min()
    xs = spla.spsolve(A.to_scipy().tocsc(), b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 1e-6
    s.close()


def test_async_exact_local_solves_and_max_iters():
    A, b, owner = problem(40, 40, 4, voronoi=False)
    s = R.Solver(A, b, owner, 2, R.options("exact"))
    st, x = s.solve(1e-8, 5000, "async")
    assert st == R._ffi.RAS_OK
    assert O.verify_global(A, x, b, 1e-8)[0]
    st, x = s.solve(1e-8, 3, "async")  # per-subdomain update cap (R21)
    assert st == R._ffi.RAS_ENOCONV
    assert s.stats()["updates_max"] <= 3
    s.close()


def test_async_single_subdomain_is_exact():
    A, b, _ = problem(24, 24, 1)
    s = R.Solver(A, b, np.zeros(576, np.int32), 0, R.options("exact"))
    st, x = s.solve(1e-10, 10, "async")
    assert st == R._ffi.RAS_OK
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)
    s.close()


@pytest.mark.parametrize("persistent", [0, 1])
@pytest.mark.parametrize("detector", ["central", "decentral"])
def test_async_single_gpu_modes_converge(persistent, detector):
    # BLOCK-sized subdomains on one GPU: the persistent cooperative kernel
    # (default) and the stream-per-subdomain driver both reach tol and verify
    N = 96
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 3)
    owner = ri.voronoi_partition(N, N, 9, seed=6)
    s = R.Solver(A, b, owner, 3, R.options("jacobi", 20, detector=detector, async_persistent=persistent))
    st, x = s.solve(1e-8, 50000, "async")
    stt = s.stats()
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0], stt
    assert stt["updates_min"] > 0 and stt["kernel_launches"] >= 1
    if persistent == 1:
        assert stt["kernel_launches"] <= 10 * (stt["resumes"] + 1) + 20  # one persistent launch per attempt
    s.close()


def test_async_persistent_more_subdomains_than_ctas():
    # 13 x 13 = 169 subdomains > the 148 co-resident CTAs: every CTA loops over
    # two subdomains of its own; the solve still detects, verifies and matches
    N = 13 * 12
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 8)
    owner = R.partition_regular(N, N, 1, 13, 13, 1)
    s = R.Solver(A, b, owner, 2, R.options("jacobi", 10, detector="decentral", async_persistent=1))
    st, x = s.solve(1e-8, 200000, "async")
    stt = s.stats()
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0], stt
    assert stt["updates_min"] > 0 and stt["kernel_launches"] < 50
    s.close()


@pytest.mark.parametrize("seqlock", ["1", "0"])
def test_async_persistent_default(seqlock, monkeypatch):
    # R33: on one GPU the persistent kernel reads every neighbour's update whole
    # (sequence counters), so fixed-m local solves take it by default like exact
    # (tolerance) solves; with the snapshots turned off fixed-m solves go back to
    # the stream driver (the torn-snapshot schedule diverges on thin strips)
    monkeypatch.setenv("RAS_PERSISTENT_SEQLOCK", seqlock)
    N = 128
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 2)
    owner = R.partition_regular(N, N, 1, 1, 8, 1)
    for kind in ("jacobi", "exact"):
        few_launches = kind == "exact" or seqlock == "1"
        s = R.Solver(A, b, owner, 4, R.options(kind, 20))
        st, x = s.solve(1e-8, 50000, "async")
        stt = s.stats()
        assert st == 0 and O.verify_global(A, x, b, 1e-8)[0], (kind, stt)
        assert (stt["kernel_launches"] < 50) == few_launches, (kind, stt["kernel_launches"])
        s.close()


def test_r33_thin_strips_converge_with_whole_update_snapshots():
    # the configuration that diverged (1e70) with one CTA per strip and fixed-m
    # PCG(20) while neighbours' corrections were read half-written (R33): with
    # whole-update snapshots the fully concurrent schedule converges
    N = 256
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = R.partition_regular(N, N, 1, 1, 16, 1)
    s = R.Solver(A, b, owner, 4, R.options("jacobi", 20, async_persistent=1, persistent_grid=16, max_resumes=0))
    st, x = s.solve(1e-8, 4000, "async")
    stt = s.stats()
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0], stt
    assert stt["updates_max"] < 2000, stt
    s.close()
