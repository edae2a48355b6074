"""Row a0 on the device: the gamma-hop overlap sets, owned / halo slot maps and
receive counts built by CUDA kernels (ras_options.device_setup = 1, the default)
must equal the host plan's (device_setup = 0), which tests/test_plan.py pins
bit-exactly against the oracle -- integer work, so bit-exact (P133-142, R1)."""
import os
import threading

import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def _plan_dump(s):
    pl = s.plan()
    info = pl.info()
    out = {"info": {k: info[k] for k in ("n_own", "n_halo", "rows_local", "local_subdomains", "nnz_residual",
                                         "nnz_local")}}
    for li in range(info["local_subdomains"]):
        p, om, ow, gh = pl.subdomain(li)
        rs, ps, gs = pl.maps(li)
        out[li] = (p, om, ow, gh, rs, ps, gs)
    out["storage"] = pl.storage_gids()
    out["comm"] = pl.comm_pattern()
    return out


def _same(a, b):
    assert a["info"] == b["info"]
    for k in a:
        if k == "info":
            continue
        x, y = a[k], b[k]
        if isinstance(x, tuple):
            assert len(x) == len(y)
            for u, v in zip(x, y):
                if isinstance(u, np.ndarray):
                    np.testing.assert_array_equal(u, v)
                else:
                    assert u == v
        else:
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("case", ["2d_regular", "voronoi", "3d", "gamma0"])
def test_device_setup_equals_host_plan(case):
    if case == "2d_regular":
        A = ri.laplace_2d(96, 80)
        owner = O.partition_regular(96, 80, 1, 3, 2, 1)
        gamma = 3
    elif case == "voronoi":
        A = ri.laplace_2d(120)
        owner = ri.voronoi_partition(120, 120, 9, seed=4)
        gamma = 5
    elif case == "3d":
        A = ri.laplace_3d(20, 18, 16)
        owner = O.partition_regular(20, 18, 16, 2, 2, 2)
        gamma = 2
    else:
        A = ri.laplace_2d(64)
        owner = O.partition_regular(64, 64, 1, 2, 2, 1)
        gamma = 0
    b = ri.rhs(A.n, 0)
    sd = R.Solver(A, b, owner, gamma, R.options("jacobi", 4, device_setup=1))
    sh = R.Solver(A, b, owner, gamma, R.options("jacobi", 4, device_setup=0))
    _same(_plan_dump(sd), _plan_dump(sh))
    # and the sets are the oracle's (the host plan is pinned to it; checked directly here too)
    As = O.as_scipy(A)
    pl = sd.plan()
    for li in range(pl.info()["local_subdomains"]):
        p, om, ow, gh = pl.subdomain(li)
        oom, oow, ogh = O.overlap_sets(As, np.asarray(owner), p, gamma)
        np.testing.assert_array_equal(om, oom)
        np.testing.assert_array_equal(gh, ogh)
    x1, x2 = sd.solve(1e-300, 3, "sync")[1], sh.solve(1e-300, 3, "sync")[1]
    np.testing.assert_array_equal(x1, x2)
    sd.close()
    sh.close()


def test_device_setup_multi_rank_windows_loopback():
    # three virtual ranks with row windows: halo order (owning rank, gid), slots and
    # send lists identical to the host plan on every rank
    nx, ny, P, gamma, world = 90, 84, 7, 3, 3
    owner = ri.voronoi_partition(nx, ny, P, seed=8)
    b_full = ri.rhs(nx * ny, 0)
    dumps = {}
    errs = {}
    for dev in (1, 0):
        key = os.urandom(128)

        def worker(rank):
            try:
                s2r = np.array([(p * world) // P for p in range(P)])
                rows = np.nonzero(s2r[owner] == rank)[0]
                r0 = max(0, rows.min() - (gamma + 1) * nx)
                r1 = min(nx * ny, rows.max() + 1 + (gamma + 1) * nx)
                A = ri.laplace_2d_rows(nx, ny, r0, r1)
                s = R.Solver(A, b_full[r0:r1], owner, gamma, R.options("jacobi", 4, device_setup=dev),
                             comm={"rank": rank, "world": world, "device": 0, "nccl_id": key, "transport": "loopback"})
                d = _plan_dump(s)
                d["send"] = [s.plan().send_list(q) for q in range(world)]
                dumps[(dev, rank)] = d
                s.close()
            except Exception:
                import traceback

                errs[(dev, rank)] = traceback.format_exc()

        ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(300)
    assert not errs, errs
    for r in range(world):
        a, b = dumps[(1, r)], dumps[(0, r)]
        sa, sb = a.pop("send"), b.pop("send")
        _same(a, b)
        for (g1, s1, o1), (g2, s2, o2) in zip(sa, sb):
            np.testing.assert_array_equal(g1, g2)
            np.testing.assert_array_equal(s1, s2)
            assert o1 == o2


def test_device_setup_reports_window_errors():
    # an Omega_p row outside the rank's CSR window is an argument error on both paths
    nx = ny = 40
    owner = O.partition_regular(nx, ny, 1, 1, 2, 1)
    A = ri.laplace_2d_rows(nx, ny, 0, 21 * nx)  # rank window too small for overlap 3
    b = ri.rhs(nx * ny, 0)[: 21 * nx]
    for dev in (1, 0):
        with pytest.raises(R.RasError) as e:
            R.Solver(A, b, owner, 3, R.options("jacobi", 4, device_setup=dev))
        assert "window" in str(e.value)
