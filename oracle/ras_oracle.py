"""Plain, slow, obviously-correct CPU oracle of the (a)synchronous RAS hot path.

TEST INFRASTRUCTURE ONLY: imported solely by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs.  Shares no code with the
CUDA path.  FP64 throughout (the paper states no precision; R16).

Citations: "P<n>" = /root/reference/PAPER.md line n (section / equation named),
"S<n>" = SPEC.md line n, "R<n>" = reading n in DESIGN.md (SURVEY §8c Q<n>).

What the method computes (PAPER §2.1, P114-153; Alg. 1, P233-245):
  solve A x = b (Eq. 1, P114-118) by Restricted Additive Schwarz: every
  subdomain p solves its overlapped local problem A_p d = R_p (b - A x^k)
  (local + interface matrix, P292-297) and writes back only the rows it owns
  ("considered as variables ... but discarded afterwards", P147-153).
The synchronous sweep is double-buffered (every p reads x^k; R5) and the
update is the residual-correction form with initial guess 0 (R4).

Parity status of every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py.  The only unpinned part
is the asynchronous iterate sequence, which is non-reproducible by design
(P170-172): "parity unpinned" for async iterates; only their end state
(verified residual, error vs the exact solution) is pinned.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "block_of",
    "factor_pair",
    "partition_regular",
    "partition_regular1d",
    "partition_regular2d",
    "overlap_sets",
    "Subdomain",
    "setup",
    "comm_pattern",
    "subdomain_graph",
    "cholesky_factor",
    "cholesky_solve",
    "pcg",
    "ic0",
    "ilu0",
    "level_sets",
    "make_local_solver",
    "local_residual",
    "local_converged",
    "RasResult",
    "ras_sync",
    "verify_global",
    "ras_schedule",
    "bfs_tree",
    "tree_depth",
    "tree_diameter",
    "detector_sim_centralized",
    "detector_sim_decentralized",
    "default_central_tree",
    "as_scipy",
]


def as_scipy(A):
    """Accept a ras_inputs.CSR or a scipy matrix; return scipy CSR (full matrix only)."""
    if sp.issparse(A):
        return sp.csr_matrix(A)
    if getattr(A, "row0", 0) != 0 or A.nrows != A.n:
        raise ValueError("oracle needs the full matrix")
    return sp.csr_matrix((A.data, A.indices, A.indptr), shape=(A.n, A.n))


# --------------------------------------------------------------------------
# Partitioning (PAPER §3.2.1 "Partitioning", P277-286; R23)
# --------------------------------------------------------------------------

def block_of(c: np.ndarray, n: int, p: int) -> np.ndarray:
    """Block index of coordinate c when n cells are cut into p blocks whose sizes
    differ by at most one, earlier blocks taking the remainder (S284, R23)."""
    if p < 1 or p > n:
        raise ValueError(f"cannot cut {n} cells into {p} non-empty blocks")
    q, rem = divmod(n, p)
    c = np.asarray(c, dtype=np.int64)
    big = rem * (q + 1)
    return np.where(c < big, c // (q + 1), rem + (c - big) // max(q, 1)).astype(np.int64)


def factor_pair(P: int) -> tuple[int, int]:
    """(px, py) with px*py = P, closest to square, py >= px (S225: P=2 -> 1x2)."""
    px = int(math.isqrt(P))
    while P % px:
        px -= 1
    return px, P // px


def partition_regular(nx: int, ny: int, nz: int, px: int, py: int, pz: int) -> np.ndarray:
    """Regular block partition of an nx*ny*nz grid (regular1d/regular2d, P277-286;
    its 3D extension for C4).  Point (x,y,z) -> id (bz*py + by)*px + bx (R23)."""
    n = nx * ny * nz
    g = np.arange(n, dtype=np.int64)
    x = g % nx
    y = (g // nx) % ny
    z = g // (nx * ny)
    bx = block_of(x, nx, px)
    by = block_of(y, ny, py)
    bz = block_of(z, nz, pz)
    return ((bz * py + by) * px + bx).astype(np.int32)


def partition_regular1d(N: int, P: int) -> np.ndarray:
    """regular1d: strips of whole grid rows, <= 2 neighbours (P277-282; S207-216)."""
    return partition_regular(N, N, 1, 1, P, 1)


def partition_regular2d(N: int, P: int) -> np.ndarray:
    """regular2d: tiles, factor pair closest to square (P284-286; S218-225)."""
    px, py = factor_pair(P)
    return partition_regular(N, N, 1, px, py, 1)


# --------------------------------------------------------------------------
# Overlap and subdomain extraction (PAPER §2.1 Fig. 1, P133-142; §3.2.2, P292-297)
# --------------------------------------------------------------------------

def _neighbours(A: sp.csr_matrix, rows: np.ndarray) -> np.ndarray:
    ip = A.indptr
    if len(rows) == 0:
        return np.zeros(0, dtype=np.int64)
    parts = [A.indices[ip[r]:ip[r + 1]] for r in rows]
    return np.unique(np.concatenate(parts).astype(np.int64))


def overlap_sets(A, owner: np.ndarray, p: int, gamma: int):
    """Omega_p = S_p plus gamma breadth-first layers in the graph of A (P136-140:
    overlap gamma = extra layers of "blue" points; R1), Gamma_p = the external
    interface ("red") points adjacent to Omega_p (P140-142).
    Returns (omega, owned_mask, ghosts), omega and ghosts ascending."""
    A = as_scipy(A)
    if gamma < 0:
        raise ValueError("overlap must be >= 0")
    n = A.shape[0]
    in_set = np.asarray(owner) == p
    frontier = np.nonzero(in_set)[0]
    for _ in range(gamma):
        nb = _neighbours(A, frontier)
        nb = nb[~in_set[nb]]
        in_set[nb] = True
        frontier = nb
    omega = np.nonzero(in_set)[0].astype(np.int64)
    nb = _neighbours(A, omega)
    ghosts = nb[~in_set[nb]]
    owned = np.asarray(owner)[omega] == p
    assert len(omega) <= n
    return omega, owned, ghosts


@dataclass
class Subdomain:
    """One subdomain's local problem (S188-S198): local matrix A_p over Omega_p,
    interface matrix B_p (rows of Omega_p x ghost columns), local RHS b~_p."""

    p: int
    omega: np.ndarray
    owned: np.ndarray
    ghosts: np.ndarray
    A: sp.csr_matrix
    B: sp.csr_matrix
    b: np.ndarray
    solver: object = None
    extra: dict = field(default_factory=dict)
    Asolve: sp.csr_matrix = None  # matrix of the local solve (A_p, or ORAS's A~_p); None = A

    @property
    def owned_global(self) -> np.ndarray:
        return self.omega[self.owned]


def setup(A, b, owner, gamma, P=None, robin=0.0):
    """Alg. 1 `initialization_and_setup` (P233-237, P247-303) minus factorization.

    robin > 0: Optimized RAS (NEXT f3; PAPER P760-763 names ORAS as future work
    and gives no formula -- DESIGN.md R30): a Robin-type transmission condition in
    algebraic form, the local matrix loses `robin` times the couplings it drops,
    A~_p = A_p - robin * diag(|B_p| 1)   (B_p = couplings to columns outside Omega_p),
    so robin = 0 is RAS's Dirichlet truncation and robin -> 1 a Neumann condition.
    Only the local solve uses A~_p; the residual b - A x keeps A."""
    A = as_scipy(A)
    owner = np.asarray(owner, dtype=np.int64)
    if P is None:
        P = int(owner.max()) + 1
    subs = []
    for p in range(P):
        if not (owner == p).any():
            raise ValueError(f"subdomain {p} is empty")
        omega, owned, ghosts = overlap_sets(A, owner, p, gamma)
        rows = A[omega]
        Ap = rows[:, omega].tocsr()
        Ap.sort_indices()
        Bp = rows[:, ghosts].tocsr()
        Bp.sort_indices()
        sub = Subdomain(p, omega, owned, ghosts, Ap, Bp, np.asarray(b)[omega].copy())
        if robin:
            dropped = np.asarray(abs(Bp).sum(axis=1)).ravel()
            sub.Asolve = (Ap - sp.diags(robin * dropped)).tocsr()
            sub.Asolve.sort_indices()
        subs.append(sub)
    return subs


def comm_pattern(subs, owner, P=None, include_overlap=True) -> np.ndarray:
    """P x P receive counts, row = receiver (Fig. 2, P257-275; S262-S266).
    include_overlap=True counts (Omega_p \\ S_p) u Gamma_p (what the RAS exchange
    carries under R4); False counts ghosts only (SPEC's CommPattern)."""
    owner = np.asarray(owner)
    P = len(subs) if P is None else P
    C = np.zeros((P, P), dtype=np.int64)
    for s in subs:
        need = s.ghosts
        if include_overlap:
            need = np.concatenate([s.omega[~s.owned], s.ghosts])
        q, c = np.unique(owner[need], return_counts=True)
        C[s.p, q] += c
    return C


def subdomain_graph(subs, owner, P=None):
    """Undirected neighbour lists: p~q iff p needs a value owned by q (or vice versa)."""
    C = comm_pattern(subs, owner, P)
    Csym = (C + C.T) > 0
    np.fill_diagonal(Csym, False)
    return [sorted(np.nonzero(Csym[p])[0].tolist()) for p in range(C.shape[0])]


# --------------------------------------------------------------------------
# Local solvers (PAPER §3.3.1 "Local solution", P309-323)
# --------------------------------------------------------------------------

class NotSPDError(ValueError):
    pass


def cholesky_factor(M):
    """Cholesky factor L (dense, lower) of the local matrix, computed once
    (P311-313, P317-318 CHOLMOD).  Dense up to 4096 rows, else banded storage."""
    M = sp.csr_matrix(M)
    n = M.shape[0]
    if n <= 4096:
        try:
            L = np.linalg.cholesky(M.toarray())
        except np.linalg.LinAlgError as e:
            raise NotSPDError(str(e))
        return ("dense", L)
    coo = M.tocoo()
    bw = int(np.max(np.abs(coo.row - coo.col))) if coo.nnz else 0
    ab = np.zeros((bw + 1, n))
    low = coo.row >= coo.col
    # lower banded storage: ab[i - j, j] = M[i, j]
    ab[coo.row[low] - coo.col[low], coo.col[low]] = coo.data[low]
    try:
        cb = sla.cholesky_banded(ab, lower=True)
    except np.linalg.LinAlgError as e:
        raise NotSPDError(str(e))
    return ("banded", cb)


def cholesky_solve(F, rhs):
    """Two triangular solves with the precomputed factor (P312-313)."""
    kind, L = F
    if kind == "dense":
        y = sla.solve_triangular(L, rhs, lower=True)
        return sla.solve_triangular(L.T, y, lower=False)
    return sla.cho_solve_banded((L, True), rhs)


def pcg(Ap, minv, rt, m, inner_tol=0.0):
    """Preconditioned CG on A_p d = r~ from d0 = 0, textbook recurrences (SURVEY
    §8c "Exact recurrences"; local iterative solve P313-315; R6, R7).

      d = 0; r = r~; z = M^-1 r; p = z; rho = r.z
      for it = 1..m:
        if rho == 0: break
        q = A p; sigma = p.q; if sigma == 0: break
        alpha = rho/sigma; d += alpha p; r -= alpha q
        if inner_tol > 0 and ||r|| <= inner_tol ||r~||: break
        z = M^-1 r; rho' = r.z; beta = rho'/rho; rho = rho'; p = z + beta p

    Returns (d, iterations performed)."""
    d = np.zeros_like(rt)
    r = rt.copy()
    z = minv(r)
    p = z.copy()
    rho = float(np.dot(r, z))
    rt_norm = float(np.sqrt(np.dot(rt, rt)))
    it = 0
    for _ in range(m):
        if rho == 0.0:
            break
        q = Ap @ p
        sigma = float(np.dot(p, q))
        if sigma == 0.0:
            break
        it += 1
        alpha = rho / sigma
        d = d + alpha * p
        r = r - alpha * q
        if inner_tol > 0.0 and float(np.sqrt(np.dot(r, r))) <= inner_tol * rt_norm:
            break
        z = minv(r)
        rho_new = float(np.dot(r, z))
        beta = rho_new / rho
        rho = rho_new
        p = z + beta * p
    return d, it


def ic0(Ap):
    """Incomplete Cholesky IC(0) of A_p in natural Omega_p order on the pattern
    of lower(A_p) (R9):
      for i ascending: for j < i in pattern ascending:
          L_ij = (a_ij - sum_{k<j, (i,k),(j,k) in pattern} L_ik L_jk) / L_jj
      L_ii = sqrt(a_ii - sum_{k<i} L_ik^2)      (<= 0 -> not SPD)
    Returns L as scipy CSR (lower, with diagonal)."""
    A = sp.csr_matrix(Ap)
    A.sort_indices()
    n = A.shape[0]
    rows = []  # rows[i] = dict col -> L_ij (j <= i)
    for i in range(n):
        cols = A.indices[A.indptr[i]:A.indptr[i + 1]]
        vals = A.data[A.indptr[i]:A.indptr[i + 1]]
        Li = {}
        aii = 0.0
        for j, a in zip(cols.tolist(), vals.tolist()):
            if j < i:
                Lj = rows[j]
                s = 0.0
                for k, lik in Li.items():  # k < j by construction (ascending)
                    ljk = Lj.get(k)
                    if ljk is not None:
                        s += lik * ljk
                Li[j] = (a - s) / Lj[j]
            elif j == i:
                aii = a
        piv = aii - sum(v * v for v in Li.values())
        if not piv > 0.0:
            raise NotSPDError(f"IC(0) pivot {piv} <= 0 at local row {i}")
        Li[i] = math.sqrt(piv)
        rows.append(Li)
    indptr = [0]
    indices = []
    data = []
    for Li in rows:
        ks = sorted(Li)
        indices += ks
        data += [Li[k] for k in ks]
        indptr.append(len(indices))
    return sp.csr_matrix((np.array(data), np.array(indices, dtype=np.int64), np.array(indptr)), shape=(n, n))


def ilu0(Ap):
    """ILU(0) of A_p on its own pattern, IKJ variant (Saad, Alg. 10.4; R10):
      for i: for k < i in pattern(i): a_ik /= a_kk;
                 for j > k in pattern(i): a_ij -= a_ik a_kj
    Returns (L unit-lower strict part + I, U upper with diagonal) as scipy CSR."""
    A = sp.csr_matrix(Ap, copy=True)
    A.sort_indices()
    n = A.shape[0]
    rows = []
    for i in range(n):
        cols = A.indices[A.indptr[i]:A.indptr[i + 1]].tolist()
        vals = A.data[A.indptr[i]:A.indptr[i + 1]].tolist()
        w = dict(zip(cols, vals))
        for k in cols:
            if k >= i:
                break
            Uk = rows[k]
            ukk = Uk[k]
            w[k] = w[k] / ukk
            lik = w[k]
            for j, ukj in Uk.items():
                if j > k and j in w:
                    w[j] -= lik * ukj
        if not w.get(i, 0.0) > 0.0:
            raise NotSPDError(f"ILU(0) pivot {w.get(i, 0.0)} <= 0 at local row {i}")
        rows.append(w)
    Li, Lj, Lv, Ui, Uj, Uv = [], [], [], [], [], []
    for i, w in enumerate(rows):
        for j in sorted(w):
            if j < i:
                Li.append(i); Lj.append(j); Lv.append(w[j])
            else:
                Ui.append(i); Uj.append(j); Uv.append(w[j])
        Li.append(i); Lj.append(i); Lv.append(1.0)
    L = sp.csr_matrix((Lv, (Li, Lj)), shape=(n, n))
    U = sp.csr_matrix((Uv, (Ui, Uj)), shape=(n, n))
    L.sort_indices(); U.sort_indices()
    return L, U


def level_sets(T, lower=True) -> np.ndarray:
    """Level of every row of a triangular matrix for a level-scheduled solve
    (cuSPARSE csrsm2 "level-set strategy", P320-323): level[i] = 0 if row i has
    no off-diagonal dependency, else 1 + max level of its dependencies."""
    T = sp.csr_matrix(T)
    n = T.shape[0]
    lev = np.zeros(n, dtype=np.int64)
    order = range(n) if lower else range(n - 1, -1, -1)
    for i in order:
        cols = T.indices[T.indptr[i]:T.indptr[i + 1]]
        dep = cols[cols < i] if lower else cols[cols > i]
        if len(dep):
            lev[i] = 1 + lev[dep].max()
    return lev


def make_local_solver(sub: Subdomain, kind: str, inner_iters: int = 20, inner_tol: float = 0.0):
    """Attach the local solve of Alg. 1 line "Locally solve the matrix" (P240):
    'exact' (Cholesky once + triangular solves, P311-318), 'jacobi' (Jacobi-PCG,
    R8), 'ic0' / 'ilu0' (incomplete-factor PCG, R9/R10).  Returns a callable
    r~ -> d and records the inner iteration count in sub.extra['inner']."""
    sub.extra["inner"] = 0
    M = sub.A if sub.Asolve is None else sub.Asolve  # ORAS: A~_p (R30)
    if kind == "exact":
        F = cholesky_factor(M)

        def solve(rt):
            return cholesky_solve(F, rt)
    elif kind in ("jacobi", "ic0", "ilu0"):
        if kind == "jacobi":
            diag = M.diagonal()
            if (diag <= 0).any():
                raise NotSPDError(f"non-positive diagonal in subdomain {sub.p}")
            dinv = 1.0 / diag

            def minv(r):
                return dinv * r
        elif kind == "ic0":
            L = ic0(M).tocsr()
            Lt = L.T.tocsr()
            sub.extra["L"] = L

            def minv(r):
                y = spla.spsolve_triangular(L, r, lower=True)
                return spla.spsolve_triangular(Lt, y, lower=False)
        else:
            L, U = ilu0(M)
            sub.extra["L"], sub.extra["U"] = L, U

            def minv(r):
                y = spla.spsolve_triangular(L, r, lower=True, unit_diagonal=True)
                return spla.spsolve_triangular(U, y, lower=False)

        def solve(rt):
            d, it = pcg(M, minv, rt, inner_iters, inner_tol)
            sub.extra["inner"] += it
            return d
    else:
        raise ValueError(f"unknown local solver {kind!r}")
    sub.solver = solve
    return solve


def local_residual(sub: Subdomain, x: np.ndarray) -> np.ndarray:
    """r~_p = b~_p - A_p x[Omega_p] - B_p x[Gamma_p]: the local residual with the
    boundary data entering through the interface-matrix SpMV (P294-297)."""
    return sub.b - sub.A @ x[sub.omega] - sub.B @ x[sub.ghosts]


def local_converged(r2: float, b2: float, tol: float) -> bool:
    """Eq. 2 (P337-340): ||r~_p||^2 < tau^2 ||b~_p||^2; if ||b~_p|| = 0 the
    subdomain is converged iff ||r~_p|| = 0 (R11; S438)."""
    if b2 == 0.0:
        return r2 == 0.0
    return r2 < tol * tol * b2


@dataclass
class RasResult:
    x: np.ndarray
    sweeps: int
    converged: bool
    history: list
    inner_total: int = 0


def ras_sync(A, b, subs, tol, max_iters, x0=None, record_iterates=False):
    """Synchronous RAS, Alg. 1 (P233-245) in lock-step (P155-161), double-buffered
    (R5).  At the start of sweep k: rel_k = ||b - A x^k|| / ||b||; stop at the
    first k with rel_k < tol (global criterion, P344-346; R13) returning x^k;
    return x^k with converged=False once k == max_iters (S78/S498, R21).
    Sweep: for every p, d_p = LocalSolve_p(r~_p) and
    x^{k+1}[S_p] = x^k[S_p] + d_p[S_p]  (restricted prolongation, P147-153)."""
    A = as_scipy(A)
    b = np.asarray(b, dtype=np.float64)
    n = A.shape[0]
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    bnorm = float(np.linalg.norm(b))
    hist = []
    iterates = [x.copy()] if record_iterates else None
    k = 0
    while True:
        r = b - A @ x
        rn = float(np.linalg.norm(r))
        rel = rn / bnorm if bnorm > 0 else (0.0 if rn == 0 else math.inf)
        hist.append(rel)
        if (rel < tol) if bnorm > 0 else (rn == 0.0):
            break
        if k >= max_iters:
            res = RasResult(x, k, False, hist, sum(s.extra.get("inner", 0) for s in subs))
            res.iterates = iterates
            return res
        x_new = x.copy()
        for s in subs:
            rt = local_residual(s, x)
            d = s.solver(rt)
            og = s.owned_global
            x_new[og] = x[og] + d[s.owned]
        x = x_new
        k += 1
        if record_iterates:
            iterates.append(x.copy())
    res = RasResult(x, k, True, hist, sum(s.extra.get("inner", 0) for s in subs))
    res.iterates = iterates
    return res


def ras_schedule(A, b, subs, schedule, x0=None):
    """One admissible ASYNCHRONOUS schedule of RAS updates (P163-176: every
    process updates with the data available to it, no waiting), written out as a
    sequence: `schedule` is a list of steps, each a list of subdomain indices that
    read the same current x and then all write their owned rows:

        for step in schedule:
            x_read = x                           (the data available at the step)
            for p in step: d_p = LocalSolve_p(r~_p(x_read))
            for p in step: x[S_p] = x_read[S_p] + d_p[S_p]

    [[0..P-1]] * K is K synchronous sweeps (ras_sync without the stopping test);
    [[0], [1], ..., [P-1]] * K is the sequential (multiplicative-Schwarz ordered)
    schedule that one processor updating its subdomains one after another in
    subdomain order produces (R34).  Returns x after the schedule."""
    A = as_scipy(A)
    n = A.shape[0]
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    for step in schedule:
        x_read = x.copy()
        for p in step:
            s = subs[p]
            d = s.solver(local_residual(s, x_read))
            og = s.owned_global
            x[og] = x_read[og] + d[s.owned]
    return x


def verify_global(A, x, b, tol):
    """Global criterion ||b - A x|| < tau ||b||, checked post termination (P344-348)."""
    A = as_scipy(A)
    rn = float(np.linalg.norm(b - A @ x))
    bn = float(np.linalg.norm(b))
    rel = rn / bn if bn > 0 else (0.0 if rn == 0 else math.inf)
    return ((rel < tol) if bn > 0 else rn == 0.0), rel


# --------------------------------------------------------------------------
# Convergence detection (PAPER §3.3.2, P326-357; §2.2, P186-196; R19)
# Both detectors as level-flag fixpoints under a lock-step scripted schedule:
# a report written in sweep k is visible in sweep k+1.
# --------------------------------------------------------------------------

def bfs_tree(adj, root=0):
    """BFS spanning tree of the subdomain graph (neighbours visited ascending).
    Returns parent array (parent[root] = -1; unreachable -> -2)."""
    P = len(adj)
    parent = [-2] * P
    parent[root] = -1
    q = [root]
    for v in q:
        for w in adj[v]:
            if parent[w] == -2:
                parent[w] = v
                q.append(w)
    return parent


def _children(parent):
    ch = [[] for _ in parent]
    for v, u in enumerate(parent):
        if u >= 0:
            ch[u].append(v)
    return ch


def tree_depth(parent) -> int:
    d = 0
    for v in range(len(parent)):
        k, u = 0, v
        while parent[u] >= 0:
            u = parent[u]
            k += 1
        d = max(d, k)
    return d


def tree_diameter(parent) -> int:
    P = len(parent)
    nb = [[] for _ in range(P)]
    for v, u in enumerate(parent):
        if u >= 0:
            nb[v].append(u)
            nb[u].append(v)

    def far(s):
        dist = [-1] * P
        dist[s] = 0
        q = [s]
        for v in q:
            for w in nb[v]:
                if dist[w] < 0:
                    dist[w] = dist[v] + 1
                    q.append(w)
        m = max(range(P), key=lambda i: dist[i])
        return m, dist[m]

    a, _ = far(0)
    _, d = far(a)
    return d


def default_central_tree(sub_to_rank):
    """Centralized tree (P331-335, Yamazaki 2019): the subdomains of a GPU are
    children of that GPU's first subdomain; GPU leaders are children of
    subdomain 0 (SURVEY §8c "Detectors")."""
    P = len(sub_to_rank)
    leader = {}
    for p in range(P):
        leader.setdefault(int(sub_to_rank[p]), p)
    parent = []
    for p in range(P):
        L = leader[int(sub_to_rank[p])]
        if p == 0:
            parent.append(-1)
        elif p == L:
            parent.append(0)
        else:
            parent.append(L)
    return parent


def detector_sim_centralized(parent, flags):
    """Centralized tree detection (P331-335).  flags[k][v] = c_v at sweep k.
    R_v(k) = c_v(k) and AND_{children w} R_w(k-1)   (R(-1) = False);
    the root stops at the first k with c_root(k) and all children R_w(k-1);
    node v stops one sweep after its parent.  Returns stop sweep per node (-1 = never)."""
    flags = np.asarray(flags, dtype=bool)
    K, P = flags.shape
    ch = _children(parent)
    root = parent.index(-1)
    R_prev = np.zeros(P, dtype=bool)
    stop = [-1] * P
    for k in range(K):
        R = np.zeros(P, dtype=bool)
        for v in range(P):
            R[v] = flags[k, v] and all(R_prev[w] for w in ch[v])
        if stop[root] < 0 and R[root]:
            stop[root] = k
        for v in range(P):
            if stop[v] < 0 and parent[v] >= 0 and 0 <= stop[parent[v]] <= k - 1:
                stop[v] = k
        R_prev = R
    return stop


def detector_sim_decentralized(parent, flags):
    """Decentralized detection (P350-357; Bahi 2005) as saturation on a spanning
    tree T with no designated root (R19):
      R_{v->u}(k) = c_v(k) and AND_{w in N_T(v)\\{u}} R_{w->v}(k-1);
      v declares global convergence at k if c_v(k) and AND_{w in N_T(v)} R_{w->v}(k-1)
      and floods STOP over T (a node stops one sweep after a tree neighbour).
    Returns stop sweep per node (-1 = never)."""
    flags = np.asarray(flags, dtype=bool)
    K, P = flags.shape
    nb = [[] for _ in range(P)]
    for v, u in enumerate(parent):
        if u >= 0:
            nb[v].append(u)
            nb[u].append(v)
    Rp = {(v, u): False for v in range(P) for u in nb[v]}
    stop = [-1] * P
    for k in range(K):
        Rn = {}
        for v in range(P):
            for u in nb[v]:
                Rn[(v, u)] = bool(flags[k, v]) and all(Rp[(w, v)] for w in nb[v] if w != u)
        newly = []
        for v in range(P):
            if stop[v] >= 0:
                continue
            declare = bool(flags[k, v]) and all(Rp[(w, v)] for w in nb[v])
            heard = any(0 <= stop[w] <= k - 1 for w in nb[v])
            if declare or heard:
                newly.append(v)
        for v in newly:
            stop[v] = k
        Rp = Rn
    return stop
