"""N>1 host logic on CPU: world-size-2 (and 3) gloo process groups build their
per-rank plans, exchange halo requests (what ras_setup does over NCCL), and run
one emulated halo exchange through the pack lists; every received value must
land in the right halo slot.  Plans are compared with the oracle's sets."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import ras_inputs as ri

R = pytest.importorskip("paper_2003_05361_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "voronoi":
            nx, ny, P, gamma = 45, 38, 10, 3
            owner = ri.voronoi_partition(nx, ny, P, seed=11)
        else:
            nx, ny, P, gamma = 40, 40, 8, 2
            owner = O.partition_regular(nx, ny, 1, 2, 4, 1)
        A = ri.laplace_2d(nx, ny)
        b = ri.rhs(nx * ny)
        pl = R.Plan(A, b, owner, gamma, rank=rank, world=world)
        # exchange requests: everyone learns what each peer needs from it
        reqs = [pl.halo_request(r) if r != rank else (np.zeros(0, np.int64), 0) for r in range(world)]
        gathered = [None] * world
        dist.all_gather_object(gathered, reqs)
        for qq in range(world):
            if qq != rank:
                g, off = gathered[qq][rank]
                pl.set_send(qq, g, off)
        pl.finalize()
        own_gids, halo_gids = pl.storage_gids()
        # emulated exchange: x[slot] = gid + 0.5 on owners, pack -> send -> land in halo
        x_own = own_gids.astype(np.float64) + 0.5
        halo = np.full(len(halo_gids), np.nan)
        ops = []
        bufs = []
        for qq in range(world):
            if qq == rank:
                continue
            g, slots, off = pl.send_list(qq)
            if len(g):
                t = torch.from_numpy(x_own[slots].copy())
                bufs.append(t)
                ops.append(dist.P2POp(dist.isend, t, qq))
            cnt = len(pl.halo_request(qq)[0])
            if cnt:
                rt = torch.empty(cnt, dtype=torch.float64)
                bufs.append((qq, rt))
                ops.append(dist.P2POp(dist.irecv, rt, qq))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for item in bufs:
            if isinstance(item, tuple):
                qq, rt = item
                g, off = pl.halo_request(qq)
                halo[off:off + len(g)] = rt.numpy()
        ok = np.array_equal(halo, halo_gids.astype(np.float64) + 0.5)
        # sets vs oracle
        subs = O.setup(A, b, owner, gamma)
        s2r = [(p * world) // P for p in range(P)]
        local = [s for s in subs if s2r[s.p] == rank]
        for li, s in enumerate(local):
            p, om, ow, gh = pl.subdomain(li)
            ok &= p == s.p and np.array_equal(om, s.omega) and np.array_equal(gh, s.ghosts)
        q.put((rank, bool(ok), len(halo_gids)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "regular"), (2, "voronoi"), (3, "voronoi")])
def test_gloo_multirank_exchange_plan(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert all(nh > 0 for _, _, nh in res)
