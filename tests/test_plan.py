"""Host-side setup plan (scope row a0) against the oracle, bit-exact, on CPU.

The plan is pure host C++ inside libras_b200.so (no CUDA call), so partitions,
overlap sets, ghosts, restrict/prolong/pack maps are checked here without a GPU.
Also: the library loads and exports every symbol include/*.h declares."""
import os
import re

import numpy as np
import pytest

import oracle as O
import ras_inputs as ri

R = pytest.importorskip("paper_2003_05361_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    names = set()
    for h in ("ras.h", "ras_plan.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^\s*(?:const char\*|ras_status|void|int32_t|int64_t)\s+\**(ras_\w+)\s*\(", src, re.M))
    lib = R._ffi.lib()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert {n for n, _, _ in R._ffi.SIGNATURES} == names
    assert lib.ras_abi_version() == R._ffi.ABI_VERSION == 4
    # provenance: the loaded library was built from exactly this tree
    from paper_2003_05361_b200.build import source_hash

    assert lib.ras_build_hash().decode() == source_hash()


@pytest.mark.parametrize("dims,parts", [((10, 1, 1), (3, 1, 1)), ((64, 64, 1), (2, 2, 1)), ((17, 9, 1), (4, 3, 1)),
                                        ((6, 5, 4), (2, 2, 2)), ((33, 12, 1), (1, 5, 1))])
def test_partition_regular_bit_exact(dims, parts):
    assert np.array_equal(R.partition_regular(*dims, *parts), O.partition_regular(*dims, *parts))


def test_partition_regular_rejects_empty_blocks():
    with pytest.raises(R.RasError):
        R.partition_regular(3, 3, 1, 4, 1, 1)


CASES = {
    "c1": (lambda: ri.laplace_2d(64), lambda: O.partition_regular(64, 64, 1, 2, 2, 1), 2),
    "voronoi": (lambda: ri.laplace_2d(41, 37), lambda: ri.voronoi_partition(41, 37, 9, seed=7), 3),
    "strips_g0": (lambda: ri.laplace_2d(20, 30), lambda: O.partition_regular1d(30, 4)[:600], 0),
    "3d": (lambda: ri.laplace_3d(9, 8, 7), lambda: O.partition_regular(9, 8, 7, 2, 2, 2), 2),
}


def _storage_order(subs_local, owner, sub_to_rank, rank):
    own = np.concatenate([s.omega[s.owned] for s in subs_local])
    need = set()
    for s in subs_local:
        need |= set(s.omega[~s.owned].tolist()) | set(s.ghosts.tolist())
    halo = [g for g in need if sub_to_rank[owner[g]] != rank]
    halo.sort(key=lambda g: (sub_to_rank[owner[g]], g))
    return own, np.array(halo, dtype=np.int64)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("world", [1, 2, 3])
def test_plan_maps_bit_exact_vs_oracle(case, world):
    mkA, mkown, gamma = CASES[case]
    A = mkA()
    owner = mkown()
    P = int(owner.max()) + 1
    if world > P:
        pytest.skip("more ranks than subdomains")
    b = ri.rhs(A.n, 0)
    subs = O.setup(A, b, owner, gamma)
    sub_to_rank = np.array([(p * world) // P for p in range(P)])
    plans = [R.Plan(A, b, owner, gamma, rank=r, world=world) for r in range(world)]
    # exchange halo requests in-process (what ras_setup does over NCCL)
    for q in range(world):
        for r in range(world):
            if q != r:
                g, off = plans[q].halo_request(r)
                plans[r].set_send(q, g, off)
    for pl in plans:
        pl.finalize()
    for r, pl in enumerate(plans):
        info = pl.info()
        local = [s for s in subs if sub_to_rank[s.p] == r]
        assert info["local_subdomains"] == len(local)
        own_gids, halo_gids = pl.storage_gids()
        want_own, want_halo = _storage_order(local, owner, sub_to_rank, r)
        assert np.array_equal(own_gids, want_own)
        assert np.array_equal(halo_gids, want_halo)
        slot = {int(g): i for i, g in enumerate(np.concatenate([own_gids, halo_gids]))}
        assert info["rows_local"] == sum(len(s.omega) for s in local)
        for li, s in enumerate(local):
            p, om, ow, gh = pl.subdomain(li)
            assert p == s.p
            assert np.array_equal(om, s.omega) and np.array_equal(ow, s.owned) and np.array_equal(gh, s.ghosts)
            rs, ps, gs = pl.maps(li)
            assert np.array_equal(rs, [slot[int(g)] for g in s.omega])
            assert np.array_equal(ps, np.where(s.owned, rs, -1))
            assert np.array_equal(gs, [slot[int(g)] for g in s.ghosts])
        # pack lists: what each peer q needs from r, in q's halo order, and where it lands
        for q in range(world):
            if q == r:
                continue
            g, sl, off = pl.send_list(q)
            qh, qoff = plans[q].halo_request(r)
            assert np.array_equal(g, qh) and off == qoff
            assert np.array_equal(own_gids[sl], g)
        assert info["nnz_residual"] == sum(A.to_scipy()[s.omega].nnz for s in local)
        assert info["nnz_local"] == sum(s.A.nnz for s in local)


def test_plan_c1_sizes():
    A = ri.laplace_2d(64)
    owner = O.partition_regular(64, 64, 1, 2, 2, 1)
    pl = R.Plan(A, ri.rhs(4096), owner, 2)
    pl.finalize()
    i = pl.info()
    assert i["rows_local"] == 4 * 1153 and i["nnz_local"] == 4 * 5629 and i["n_halo"] == 0


def test_plan_row_window():
    nx, ny = 30, 40
    owner = O.partition_regular(nx, ny, 1, 1, 4, 1)  # 4 strips of 10 grid rows
    full = R.Plan(ri.laplace_2d(nx, ny), None, owner, 2, rank=1, world=4)
    # rank 1 owns grid rows 10..19; Omega needs rows 8..21 -> window rows [8*nx, 22*nx)
    win = ri.laplace_2d_rows(nx, ny, 8 * nx, 22 * nx)
    wp = R.Plan(win, None, owner, 2, rank=1, world=4)
    assert np.array_equal(full.subdomain(0)[1], wp.subdomain(0)[1])
    small = ri.laplace_2d_rows(nx, ny, 9 * nx, 21 * nx)
    with pytest.raises(R.RasError, match="outside the CSR row window"):
        R.Plan(small, None, owner, 2, rank=1, world=4)


def test_plan_validation_errors():
    A = ri.laplace_2d(6)
    own = np.zeros(36, np.int32)
    with pytest.raises(R.RasError, match="owner"):
        bad = own.copy()
        bad[3] = 7
        R.Plan(A, None, bad, 1, num_subdomains=2)
    with pytest.raises(R.RasError, match="no subdomain"):
        R.Plan(A, None, own, 1, rank=1, world=2)
    B = ri.laplace_2d(6)
    B.indices[B.indptr[2]], B.indices[B.indptr[2] + 1] = B.indices[B.indptr[2] + 1], B.indices[B.indptr[2]]
    with pytest.raises(R.RasError, match="strictly increasing"):
        R.Plan(B, None, own, 1)


def _diameter(C):
    """Diameter of the subdomain graph p ~ q iff C[p, q] + C[q, p] > 0 (BFS from every node)."""
    P = C.shape[0]
    adj = [np.nonzero((C[p] + C[:, p]) > 0)[0] for p in range(P)]
    best = 0
    for s in range(P):
        dist = np.full(P, -1)
        dist[s] = 0
        frontier = [s]
        while frontier:
            nxt = []
            for u in frontier:
                for v in adj[u]:
                    if v != u and dist[v] < 0:
                        dist[v] = dist[u] + 1
                        nxt.append(v)
            frontier = nxt
        best = max(best, dist.max())
    return best


@pytest.mark.parametrize("scheme", ["regular1d", "regular2d", "graph"])
@pytest.mark.parametrize("gamma", [0, 2])
def test_comm_pattern_bit_exact(scheme, gamma):
    # NEXT f4 (PAPER §3.3 "Partitioning", Fig. 2, P257-290): the library's receive
    # counts equal the oracle's, computed independently from its own overlap sets
    N, P = 48, 9
    A = ri.laplace_2d(N)
    owner = {"regular1d": O.partition_regular1d(N, P), "regular2d": O.partition_regular2d(N, P),
             "graph": ri.voronoi_partition(N, N, P, seed=3)}[scheme]
    C = R.Plan(A, None, owner, gamma).comm_pattern()
    ref = O.comm_pattern(O.setup(A, np.zeros(N * N), owner, gamma), owner, P)
    assert C.dtype == np.int64 and np.array_equal(C, ref)
    assert np.all(np.diag(C) == 0)
    assert np.array_equal(C > 0, (C > 0).T)  # symmetric A: p needs q iff q needs p


def test_comm_pattern_multi_rank_rows_sum_to_the_whole():
    N, P, gamma = 40, 6, 1
    A = ri.laplace_2d(N)
    owner = ri.voronoi_partition(N, N, P, seed=7)
    ref = O.comm_pattern(O.setup(A, np.zeros(N * N), owner, gamma), owner, P)
    tot = np.zeros((P, P), np.int64)
    for rank in range(3):
        part = R.Plan(A, None, owner, gamma, rank=rank, world=3).comm_pattern()
        mine = [p for p in range(P) if (p * 3) // P == rank]
        assert not part[[p for p in range(P) if p not in mine]].any()
        tot += part
    assert np.array_equal(tot, ref)


@pytest.mark.parametrize("P", [4, 9, 16])
def test_information_propagation_distance(P):
    # P277-286: regular1d needs P - 1 exchanges between the farthest subdomains;
    # regular2d (px x py tiles) (px - 1) + (py - 1) with face neighbours only
    # (gamma = 0) and max(px, py) - 1 once the overlap adds the diagonal tiles (R3)
    N = 48
    A = ri.laplace_2d(N)
    px, py = O.factor_pair(P)
    d1 = _diameter(R.Plan(A, None, O.partition_regular1d(N, P), 1).comm_pattern())
    d2_face = _diameter(R.Plan(A, None, O.partition_regular2d(N, P), 0).comm_pattern())
    d2_diag = _diameter(R.Plan(A, None, O.partition_regular2d(N, P), 1).comm_pattern())
    assert d1 == P - 1
    assert d2_face == (px - 1) + (py - 1)
    assert d2_diag == max(px, py) - 1


@pytest.mark.parametrize("robin", [0.0, 0.6])
def test_band_cholesky_host_factor(robin):
    # NEXT f1 host part: the library's complete banded Cholesky factor of every
    # local A_p (ORAS-modified for robin > 0) reproduces A_p (L L^T) and equals
    # LAPACK's factor of the oracle's matrix (up to summation order)
    N, gamma = 30, 2
    A = ri.laplace_2d(N)
    owner = ri.voronoi_partition(N, N, 4, seed=2)
    pl = R.Plan(A, None, owner, gamma)
    pl.set_robin(robin)
    pl.finalize()
    subs = O.setup(A, np.zeros(N * N), owner, gamma, robin=robin)
    for lp in range(4):
        Lb, b = pl.band_cholesky(lp)
        n = Lb.shape[0]
        L = np.zeros((n, n))
        for i in range(n):
            for j in range(max(0, i - b), i + 1):
                L[i, j] = Lb[i, j - i + b]
        M = (subs[lp].Asolve if robin else subs[lp].A).toarray()
        m = M.shape[0]
        Mp = np.eye(n)
        Mp[:m, :m] = M  # padding rows are identity rows
        assert np.linalg.norm(L @ L.T - Mp) <= 1e-14 * np.linalg.norm(Mp)
        ref = np.linalg.cholesky(M)
        assert np.linalg.norm(L[:m, :m] - ref) <= 1e-13 * np.linalg.norm(ref)
        bw_ref = max(abs(i - j) for i, j in zip(*np.nonzero(M)))
        assert b == bw_ref
