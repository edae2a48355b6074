"""C-ABI behaviour on the GPU beyond single-solve parity: restart / warm start
(RAS is a stationary iteration: x^{k1+k2} = F^{k2}(x^{k1})), new right-hand
sides, device-resident solves, statistics, and kernel timing."""
import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def setup(N=48, P=6, gamma=2, m=8, seed=0):
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, seed)
    owner = ri.voronoi_partition(N, N, P, seed=5)
    return A, b, owner, gamma, m


def test_warm_start_continues_the_iteration():
    A, b, owner, gamma, m = setup()
    subs = O.setup(A, b, owner, gamma)
    for s in subs:
        O.make_local_solver(s, "jacobi", m)
    ref = O.ras_sync(A, b, subs, 1e-300, 7, record_iterates=True)
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m))
    _, x3 = s.solve(1e-300, 3, "sync")
    _, x7 = s.solve(1e-300, 4, "sync", x0=x3)
    assert rel(x7, ref.iterates[7]) <= 1e-10
    s.close()


def test_set_rhs_and_stats():
    A, b, owner, gamma, m = setup()
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m))
    b2 = ri.rhs(A.n, 7)
    s.set_rhs(b2)
    st, x = s.solve(1e-8, 20000, "sync")
    assert st == 0
    ok, r = O.verify_global(A, x, b2, 1e-8)
    assert ok
    stt = s.stats()
    P = 6
    assert stt["inner_iters_total"] == stt["sweeps"] * m * P  # fixed m, no breakdown
    assert stt["model_bytes"] > 0 and stt["kernel_launches"] > 0
    assert stt["num_subdomains"] == P and stt["local_subdomains"] == P and stt["world"] == 1
    assert stt["updates_min"] == stt["updates_max"] == stt["sweeps"]  # sync spread is 0 (Fig. 7c)
    s.close()


def test_solve_device_owned_order_and_kernel_timing():
    import torch

    A, b, owner, gamma, m = setup()
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, path="tiled"))
    gids = s.owned_gids()
    assert sorted(gids.tolist()) == list(range(A.n))
    x = torch.zeros(len(gids), dtype=torch.float64, device="cuda")
    s.kernel_timing(True)
    st = s.solve_device(1e-300, 5, "sync", None, x.data_ptr())
    kt = s.kernel_times()
    s.kernel_timing(False)
    st2, xh = s.solve(1e-300, 5, "sync")
    assert np.array_equal(x.cpu().numpy(), xh[gids])  # deterministic: bitwise reproducible
    assert kt["k_spmv_dot"][0] == 5 * m and kt["k_spmv_dot"][1] > 0  # the check-only sweep 5 launches no PCG
    assert kt["k_small_pcg"][0] == 0 and kt["k_resident_pcg"][0] == 0
    # start from a device x0 = the 5-sweep result: 5 more sweeps = 10 sweeps from zero
    y = torch.zeros_like(x)
    s.solve_device(1e-300, 5, "sync", x.data_ptr(), y.data_ptr())
    _, x10 = s.solve(1e-300, 10, "sync")
    assert rel(y.cpu().numpy(), x10[gids]) <= 1e-12
    s.close()


@pytest.mark.parametrize("path", ["block", "resident"])
def test_whole_solve_kernels_are_timed(path):
    A, b, owner, gamma, m = setup()
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, path=path))
    s.kernel_timing(True)
    s.solve(1e-300, 4, "sync")
    kt = s.kernel_times()
    name = "k_small_pcg" if path == "block" else ("k_resident2" if "k_resident2" in kt else "k_resident_pcg")
    assert kt[name][0] == 4 and kt[name][1] > 0 and kt["k_spmv_dot"][0] == 0 and kt["k_prolong"][0] == 0
    assert s.stats()["pcg_path"] == getattr(R._ffi, "RAS_PCG_" + path.upper())
    s.close()


@pytest.mark.parametrize("kind", ["jacobi", "ilu0"])
def test_async_3d(kind):
    A = ri.laplace_3d(14)
    b = ri.rhs(A.n, 0)
    owner = O.partition_regular(14, 14, 14, 2, 2, 2)
    s = R.Solver(A, b, owner, 2, R.options(kind, 8, detector="central"))
    st, x = s.solve(1e-8, 20000, "async")
    assert st == 0 and O.verify_global(A, x, b, 1e-8)[0]
    s.close()


@pytest.mark.parametrize("path", ["block", "tiled"])
def test_set_rhs_async_uses_new_eq2_norms(path):
    # ras_set_rhs must refresh the per-subdomain ||b~_p||^2 that the async Eq. 2
    # flags compare against (P337-340): with a 1000x larger RHS the old norms would
    # let the flags fire far too late / the new ones must still verify first time
    A, b, owner, gamma, m = setup()
    # (Eq. 2 over overlapping rows can fire before the global criterion holds, R12:
    # a resume or two is legitimate; stale norms 1e6 x too large would make every
    # detection round stop at once and exhaust the resumes -> RAS_EVERIFY)
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m, path=path, max_resumes=3))
    b2 = 1e3 * ri.rhs(A.n, 7)
    s.set_rhs(b2)
    st, x = s.solve(1e-8, 50000, "async")
    stt = s.stats()
    assert st == 0, stt
    assert O.verify_global(A, x, b2, 1e-8)[0]
    # and back to a small RHS: stale (large) norms would stop at once and fail verification
    s.set_rhs(1e-3 * b)
    st, x = s.solve(1e-8, 50000, "async")
    assert st == 0, s.stats()
    assert O.verify_global(A, x, 1e-3 * b, 1e-8)[0]
    s.close()


@pytest.mark.parametrize("mode", ["sync", "async"])
@pytest.mark.parametrize("path", ["block", "tiled", "resident"])
def test_phase_times_populated(mode, path):
    # ras_stats_t per-phase times (Figs. 3a-7a): nonzero where the phase runs, and
    # (sync) their sum is the device part of the time to solution
    N, P = (48, 6) if path != "resident" else (200, 4)
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = ri.voronoi_partition(N, N, P, seed=5) if path != "resident" else O.partition_regular(N, N, 1, 2, 2, 1)
    s = R.Solver(A, b, owner, 2, R.options("jacobi", 8, path=path))
    st, x = s.solve(1e-8, 50000, mode)
    t = s.stats()
    assert st == 0
    assert t["t_residual"] > 0 and t["t_local_solve"] > 0 and t["t_convcheck"] > 0
    assert t["t_exchange"] >= 0 and t["t_prolong"] >= 0
    if path == "tiled":
        assert t["t_prolong"] > 0  # separate k_prolong (fused into the solve kernel on BLOCK / RESIDENT)
    tot = t["t_residual"] + t["t_local_solve"] + t["t_prolong"] + t["t_exchange"] + t["t_convcheck"]
    assert tot <= 1.05 * t["time_to_solution_s"] + 1e-3
    if mode == "sync":
        assert tot >= 0.5 * t["time_to_solution_s"], t
    s.close()


def test_solve_device_accepts_host_owned_buffers():
    # ras_solve_device with HOST pointers (the distributed e2e form): same iterate as
    # the gathered ras_solve, restricted to the owned values
    A, b, owner, gamma, m = setup()
    s = R.Solver(A, b, owner, gamma, R.options("jacobi", m))
    gids = s.owned_gids()
    x0 = np.zeros(len(gids))
    xo = np.empty(len(gids))
    s.solve_device(1e-300, 4, "sync", x0.ctypes.data, xo.ctypes.data)
    _, xg = s.solve(1e-300, 4, "sync")
    np.testing.assert_array_equal(xo, xg[gids])
    # warm start from host owned values continues the iteration
    y = np.empty(len(gids))
    s.solve_device(1e-300, 3, "sync", xo.ctypes.data, y.ctypes.data)
    _, x7 = s.solve(1e-300, 7, "sync")
    assert rel(y, x7[gids]) <= 1e-12
    s.close()
