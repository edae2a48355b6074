"""Multi-GPU RAS (one process per GPU): sync mode with NCCL halo exchange +
allreduce (parity with the oracle at 1e-10 per sweep), async mode with NVLink
P2P puts and both detectors (verified residual).  Skipped with < 2 GPUs."""
import multiprocessing as mp
import os

import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def _worker(rank, world, nccl_id, cfg, q):
    try:
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        import paper_2003_05361_b200 as R

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
        s = R.Solver(A, b, owner, gamma,
                     R.options(cfg["solver"], cfg["m"], detector=cfg.get("detector", "decentral"),
                               path=cfg.get("path", "auto"), async_persistent=cfg.get("persistent", 2)),
                     comm={"rank": rank, "world": world, "device": rank, "nccl_id": nccl_id})
        out = {}
        for k in cfg.get("ks", []):
            st, x = s.solve(1e-300, k, "sync")
            out[("sync", k)] = (st, x, s.stats()["sweeps"])
        if cfg.get("converge"):
            st, x = s.solve(1e-8, 20000, cfg["converge"])
            out[("conv", cfg["converge"])] = (st, x, s.stats())
        s.close()
        q.put((rank, "ok", out))
    except Exception as e:  # report instead of hanging the parent
        import traceback

        q.put((rank, "err", traceback.format_exc()))


def _run(world, cfg, timeout=300):
    import paper_2003_05361_b200 as R

    nid = R.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, nid, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, st, out = q.get(timeout=timeout)
        assert st == "ok", out
        res[r] = out
    for p in ps:
        p.join(60)
    return res


def _oracle(cfg, K):
    A = ri.laplace_2d(cfg["nx"], cfg["ny"])
    b = ri.rhs(cfg["nx"] * cfg["ny"], 0)
    subs = O.setup(A, b, cfg["owner"], cfg["gamma"])
    for s in subs:
        O.make_local_solver(s, cfg["solver"], cfg["m"])
    return A, b, O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("world,path", [(2, "auto"), (4, "auto"), (2, "resident"), (2, "tiled")])
def test_multi_gpu_sync_parity(world, path):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    nx, ny = 96, 80
    cfg = dict(nx=nx, ny=ny, P=8, gamma=3, solver="jacobi", m=12, ks=[1, 4],
               owner=ri.voronoi_partition(nx, ny, 8, seed=5), window=True, path=path)
    res = _run(world, cfg)
    A, b, ref = _oracle(cfg, 4)
    for r in range(world):
        for k in (1, 4):
            st, x, sw = res[r][("sync", k)]
            assert sw == k
            err = np.linalg.norm(x - ref.iterates[k]) / np.linalg.norm(ref.iterates[k])
            assert err <= 1e-10, (r, k, err)


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("detector", ["central", "decentral"])
@pytest.mark.parametrize("persistent", [0, 1])
def test_multi_gpu_async_p2p_converges(detector, persistent):
    # persistent = 1: the in-kernel NVLink puts, version bumps and cross-GPU detector
    # boards of k_async_persistent; 0: the per-subdomain stream driver
    nx, ny = 80, 80
    cfg = dict(nx=nx, ny=ny, P=6, gamma=4, solver="jacobi", m=10, converge="async", detector=detector,
               owner=ri.voronoi_partition(nx, ny, 6, seed=2), persistent=persistent)
    res = _run(2, cfg)
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    for r in range(2):
        st, x, stats = res[r][("conv", "async")]
        assert st == 0, stats
        assert O.verify_global(A, x, b, 1e-8)[0]
        assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 1e-6
        assert stats["fresh_halo_reads"] > 0  # peers' puts arrived over NVLink
    np.testing.assert_array_equal(res[0][("conv", "async")][1], res[1][("conv", "async")][1])


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
def test_multi_gpu_sync_converges():
    nx = ny = 64
    cfg = dict(nx=nx, ny=ny, P=4, gamma=2, solver="jacobi", m=20, converge="sync",
               owner=O.partition_regular(nx, ny, 1, 2, 2, 1))
    res = _run(2, cfg)
    A, b, _ = _oracle(cfg, 0)
    subs = O.setup(A, b, cfg["owner"], 2)
    for s in subs:
        O.make_local_solver(s, "jacobi", 20)
    ref = O.ras_sync(A, b, subs, 1e-8, 20000)
    for r in range(2):
        st, x, stats = res[r][("conv", "sync")]
        assert st == 0 and stats["sweeps"] == ref.sweeps
        assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-10


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
def test_multi_gpu_async_resident_sequential():
    # R34 on 2 GPUs: RESIDENT-sized subdomains, per-rank paired updates with
    # NVLink puts to the peer; converges and verifies
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
        assert stats["pcg_path"] == 3  # RESIDENT: the on-chip schedule ran (R34)


def _stress_worker(rank, world, nccl_id, q):
    try:
        import paper_2003_05361_b200 as R

        nx = ny = 256
        owner = O.partition_regular(nx, ny, 1, 1, 2, 1)
        s = R.Solver(ri.laplace_2d(nx, ny), ri.rhs(nx * ny, 0), owner, 2, R.options("jacobi", 4),
                     comm={"rank": rank, "world": world, "device": rank, "nccl_id": nccl_id})
        res = s.put_stress(20000, 30000)
        s.close()
        q.put((rank, "ok", res))
    except Exception:
        import traceback

        q.put((rank, "err", traceback.format_exc()))


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
def test_multi_gpu_nvlink_put_stress():
    # Q17 / R17 over NVLink: 20000 epochs of 30000 epoch-tagged 8-byte words stored
    # into the peer GPU's window, each published by fence + system-scope version
    # increment; the reader must never see a torn word, a stale word after an
    # acquired version, or a version going backwards
    import paper_2003_05361_b200 as R

    nid = R.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_stress_worker, args=(r, 2, nid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, st, out = q.get(timeout=600)
        assert st == "ok", out
        res[r] = out
    for p in ps:
        p.join(60)
    r1 = res[1]
    print("nvlink put stress:", r1)
    assert r1["torn"] == 0 and r1["stale"] == 0 and r1["regress"] == 0, r1
    assert r1["observations"] >= 100
