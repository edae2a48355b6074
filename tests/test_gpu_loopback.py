"""Multi-rank RAS on ONE GPU through the loopback transport (ras_comm.transport =
RAS_TRANSPORT_LOOPBACK; SURVEY §4 layer 4): `world` virtual ranks, one host thread
each, in this process.  The same library code as the one-process-per-GPU NCCL
run executes -- pack lists, halo offsets and the grouped exchange (a5, P376-387),
the owned-residual allreduce (a6, P344-346), the async NVLink-style puts into the
peers' halo storage with release-published version counters (P389-397), and the
cross-rank detector boards (P331-357) -- only the transport underneath the
collectives differs (host rendezvous + device copies instead of NCCL; the peers'
windows are plain device pointers instead of CUDA IPC mappings).

Sync iterates are compared with the oracle element by element (1e-10, north_star);
async end states by the verified true residual and the error vs a dense solve."""
import os
import threading

import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2003_05361_b200")


def _run(world, cfg, timeout=600):
    """Run one rank per thread; returns {rank: outputs}."""
    key = os.urandom(128)
    res, errs = {}, {}

    def worker(rank):
        try:
            nx, ny, P, gamma = cfg["nx"], cfg["ny"], cfg["P"], cfg["gamma"]
            A = ri.laplace_2d(nx, ny)
            b = ri.rhs(nx * ny, 0)
            owner = cfg["owner"]
            if cfg.get("window"):
                # this rank's rows +- (gamma+1) grid rows: exercises the row-window ABI
                s2r = np.array([(p * world) // P for p in range(P)])
                rows = np.nonzero(s2r[owner] == rank)[0]
                r0 = max(0, rows.min() - (gamma + 1) * nx)
                r1 = min(nx * ny, rows.max() + 1 + (gamma + 1) * nx)
                A = ri.laplace_2d_rows(nx, ny, r0, r1)
                b = b[r0:r1]
            opts = R.options(cfg["solver"], cfg["m"], detector=cfg.get("detector", "decentral"),
                             path=cfg.get("path", "auto"), async_timeout_s=120.0, **cfg.get("opts", {}))
            s = R.Solver(A, b, owner, gamma, opts,
                         comm={"rank": rank, "world": world, "device": 0, "nccl_id": key, "transport": "loopback"})
            out = {"nl": s.plan().info()["local_subdomains"]}
            for k in cfg.get("ks", []):
                st, x = s.solve(1e-300, k, "sync")
                out[("sync", k)] = (st, x, s.stats()["sweeps"])
            if cfg.get("converge"):
                st, x = s.solve(1e-8, cfg.get("max_iters", 20000), cfg["converge"])
                out[("conv", cfg["converge"])] = (st, x, s.stats())
            s.close()
            res[rank] = out
        except Exception:  # report, do not hang the other threads' rendezvous forever
            import traceback

            errs[rank] = traceback.format_exc()

    ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not errs, errs
    assert len(res) == world, "a rank did not finish"
    return res


def _oracle(cfg, K):
    A = ri.laplace_2d(cfg["nx"], cfg["ny"])
    b = ri.rhs(cfg["nx"] * cfg["ny"], 0)
    subs = O.setup(A, b, cfg["owner"], cfg["gamma"])
    for s in subs:
        O.make_local_solver(s, cfg["solver"], cfg["m"])
    return A, b, O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)


@pytest.mark.parametrize("world,path", [(2, "auto"), (3, "auto"), (4, "auto"), (2, "resident"), (2, "tiled"),
                                        (3, "block")])
def test_loopback_sync_parity(world, path):
    # irregular (Voronoi) subdomains split over the virtual ranks: diagonal and
    # multi-owner halos, row windows, every local-solve path
    nx, ny = 96, 80
    P = 8
    cfg = dict(nx=nx, ny=ny, P=P, gamma=3, solver="jacobi", m=12, ks=[1, 2, 4],
               owner=ri.voronoi_partition(nx, ny, P, seed=5), window=True, path=path)
    if path == "resident":
        nx, ny = 260, 240  # RESIDENT-sized subdomains (BLOCK would take the small ones)
        cfg.update(nx=nx, ny=ny, owner=O.partition_regular(nx, ny, 1, 2, 4, 1))
    res = _run(world, cfg)
    A, b, ref = _oracle(cfg, 4)
    for r in range(world):
        assert res[r]["nl"] >= 1
        for k in (1, 2, 4):
            st, x, sw = res[r][("sync", k)]
            assert sw == k
            err = np.linalg.norm(x - ref.iterates[k]) / np.linalg.norm(ref.iterates[k])
            assert err <= 1e-10, (r, k, err)


def test_loopback_sync_converges_same_sweeps():
    nx = ny = 64
    cfg = dict(nx=nx, ny=ny, P=4, gamma=2, solver="jacobi", m=20, converge="sync",
               owner=O.partition_regular(nx, ny, 1, 2, 2, 1))
    res = _run(2, cfg)
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    subs = O.setup(A, b, cfg["owner"], 2)
    for s in subs:
        O.make_local_solver(s, "jacobi", 20)
    ref = O.ras_sync(A, b, subs, 1e-8, 20000)
    for r in range(2):
        st, x, stats = res[r][("conv", "sync")]
        assert st == 0 and stats["sweeps"] == ref.sweeps and stats["world"] == 2
        assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-10


@pytest.mark.parametrize("detector", ["central", "decentral"])
@pytest.mark.parametrize("persistent", [0, 1])
def test_loopback_async_puts_and_boards(detector, persistent):
    # async: every rank's updates store into the other rank's halo storage and bump
    # its version counters; termination is decided on the shared detector boards
    nx, ny = 80, 80
    cfg = dict(nx=nx, ny=ny, P=6, gamma=4, solver="jacobi", m=10, converge="async", detector=detector,
               owner=ri.voronoi_partition(nx, ny, 6, seed=2), opts={"async_persistent": persistent})
    res = _run(2, cfg)
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    for r in range(2):
        st, x, stats = res[r][("conv", "async")]
        assert st == 0, stats
        assert stats["verified"] and stats["final_rel_residual"] < 1e-8
        assert O.verify_global(A, x, b, 1e-8)[0]
        assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 1e-6
        assert stats["fresh_halo_reads"] > 0  # the peer's puts arrived and bumped the versions
        assert stats["updates_min"] >= 1
    np.testing.assert_array_equal(res[0][("conv", "async")][1], res[1][("conv", "async")][1])


def test_loopback_async_resident_sequential():
    # R34 across virtual ranks: RESIDENT-sized subdomains, per-rank paired on-chip
    # updates with puts into the peer's halo storage
    nx, ny = 262, 250
    cfg = dict(nx=nx, ny=ny, P=4, gamma=4, solver="jacobi", m=12, converge="async",
               owner=O.partition_regular(nx, ny, 1, 2, 2, 1))
    res = _run(2, cfg)
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    for r in range(2):
        st, x, stats = res[r][("conv", "async")]
        assert st == 0, stats
        assert O.verify_global(A, x, b, 1e-8)[0]
        assert stats["pcg_path"] == 3  # the on-chip (R34) schedule ran
        assert stats["fresh_halo_reads"] > 0


def test_loopback_async_forced_stop_resumes():
    # R20 (P346-348): the first detection round is forced to terminate early
    # (force_first_stop hook) -> the verification fails on every rank -> flags are
    # cleared and the asynchronous iteration resumes, then converges and verifies
    nx = ny = 64
    cfg = dict(nx=nx, ny=ny, P=4, gamma=2, solver="jacobi", m=10, converge="async",
               owner=O.partition_regular(nx, ny, 1, 2, 2, 1), opts={"force_first_stop": 1})
    res = _run(2, cfg)
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    for r in range(2):
        st, x, stats = res[r][("conv", "async")]
        assert st == 0, stats
        assert stats["resumes"] == 1 and stats["verified"] == 1
        assert O.verify_global(A, x, b, 1e-8)[0]


def test_loopback_put_stress_versions_and_words():
    # R17 machinery on one device: epoch-tagged words + release-published versions
    # (the NVLink variant of the same test runs in test_gpu_multi.py)
    nx = ny = 128
    owner = O.partition_regular(nx, ny, 1, 1, 2, 1)
    key = os.urandom(128)
    out, errs = {}, {}

    def worker(rank):
        try:
            s = R.Solver(ri.laplace_2d(nx, ny), ri.rhs(nx * ny, 0), owner, 2, R.options("jacobi", 4),
                         comm={"rank": rank, "world": 2, "device": 0, "nccl_id": key, "transport": "loopback"})
            out[rank] = s.put_stress(2000, 4096)
            s.close()
        except Exception:
            import traceback

            errs[rank] = traceback.format_exc()

    ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    assert not errs, errs
    r1 = out[1]
    assert r1["torn"] == 0 and r1["stale"] == 0 and r1["regress"] == 0, r1
    assert r1["observations"] >= 1
