#!/usr/bin/env python
"""B200 analogues of the paper's experiments (PAPER §4), one JSON
line per configuration, through the C ABI:

  overlap   E4/E5 (P574-598): sweeps / updates and time-to-solution vs overlap
  regime    E3/E9 + NEXT f2 (P527-546, P716-735): the paper's latency regime, 4096
            unknowns per subdomain, many subdomains per GPU: sync vs async
  detector  E8 (P678-691): centralized vs decentralized detection (async)
  partition NEXT f4 / E2 (P257-290, P513-546, Figs. 2-3): regular1d vs regular2d vs
            graph partitions at 4096 unknowns per subdomain: communication
            pattern (heat map, volume, neighbours, propagation distance) and
            sweeps / time-to-solution, sync and async

  direct    NEXT f1 (P311-318): direct (banded Cholesky) vs Jacobi-PCG local solves in the
            4096-unknowns-per-subdomain regime: sweeps, time-to-solution, sync and async
  oras      NEXT f3 (P760-763, R30): sweeps / time-to-solution vs the Robin parameter

  python tools/experiments.py overlap|regime|detector|partition|direct|oras [--tol 1e-8] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ras_inputs as ri  # noqa: E402


ASYNC_PERSISTENT = 2  # ras_options.async_persistent (--persistent)


def run(nx, ny, px, py, gamma, mode, tol, m=20, solver="jacobi", detector="decentral", max_iters=200000, reps=1,
        owner=None, robin=0.0):
    import paper_2003_05361_b200 as R

    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    if owner is None:
        owner = R.partition_regular(nx, ny, 1, px, py, 1)
    s = R.Solver(A, b, owner, gamma, R.options(solver, m, detector=detector, robin=robin,
                                               async_persistent=ASYNC_PERSISTENT))
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        st, x = s.solve(tol, max_iters, mode, gather=False)
        wall = time.perf_counter() - t0
        d = s.stats()
        out.append({"status": int(st), "wall_s": wall, "tts_s": d["time_to_solution_s"], "sweeps": d["sweeps"],
                    "updates_min": d["updates_min"], "updates_median": d["updates_median"],
                    "updates_max": d["updates_max"], "inner_iters": d["inner_iters_total"],
                    "rel_residual": d["final_rel_residual"], "resumes": d["resumes"],
                    "launches": d["kernel_launches"]})
    s.close()
    rec = {"grid": [nx, ny], "subdomains": px * py, "tiles": [px, py], "unknowns_per_subdomain": nx * ny // (px * py),
           "overlap": gamma, "mode": mode, "tol": tol, "local_solver": solver if solver == "cholesky" else f"{solver}-PCG m={m}", "detector": detector,
           "runs": out}
    if reps > 1:
        t = [r["tts_s"] for r in out]
        rec["tts_mean_s"], rec["tts_sd_s"] = float(np.mean(t)), float(np.std(t))
    return rec


def heatmap(C):
    """Fig. 2 style text heat map of receive counts (row = receiver): '.' none, 1-9 = decile of the max."""
    mx = max(int(C.max()), 1)
    rows = []
    for p in range(C.shape[0]):
        rows.append("".join("." if v == 0 else str(min(9, 1 + (9 * int(v)) // (mx + 1))) for v in C[p]))
    return rows


def diameter(C):
    P = C.shape[0]
    adj = [np.nonzero((C[p] + C[:, p]) > 0)[0] for p in range(P)]
    best = 0
    for s0 in range(P):
        dist = np.full(P, -1)
        dist[s0] = 0
        fr = [s0]
        while fr:
            nx = []
            for u in fr:
                for v in adj[u]:
                    if v != u and dist[v] < 0:
                        dist[v] = dist[u] + 1
                        nx.append(v)
            fr = nx
        best = max(best, int(dist.max()))
    return best


def partition_study(tol, reps, gamma=4, sub=64, Ps=(4, 16, 36, 64, 100)):
    """f4: three partitioners at `sub`^2 unknowns per subdomain (P x sub^2 unknowns)."""
    import paper_2003_05361_b200 as R

    recs = []
    for P in Ps:
        k = int(round(P ** 0.5))
        N = k * sub
        px, py = R_factor(P)
        owners = {"regular1d": R.partition_regular(N, N, 1, 1, P, 1),
                  "regular2d": R.partition_regular(N, N, 1, px, py, 1),
                  "graph": voronoi_valid(N, P)}
        A = ri.laplace_2d(N)
        for name, owner in owners.items():
            C = R.Plan(A, None, owner, gamma).comm_pattern()
            stats = {"partition": name, "P": P, "grid": [N, N], "overlap": gamma,
                     "comm_values_per_sweep": int(C.sum()), "max_neighbours": int(((C > 0).sum(1)).max()),
                     "max_recv_per_subdomain": int(C.sum(1).max()), "propagation_distance": diameter(C)}
            if P <= 16:
                stats["heatmap"] = heatmap(C)
            for mode in ("sync", "async"):
                r = run(N, N, 1, P, gamma, mode, tol, reps=1 if mode == "sync" else reps, owner=owner)
                recs.append({**stats, **{k2: v for k2, v in r.items() if k2 not in ("grid", "tiles", "subdomains")}})
    return recs


def voronoi_valid(N, P):
    """First seed >= 1 whose Voronoi cells are all non-empty and 4-connected."""
    for seed in range(1, 100):
        try:
            return ri.voronoi_partition(N, N, P, seed=seed)
        except ValueError:
            continue
    raise RuntimeError("no valid Voronoi partition")


def R_factor(P):
    """(px, py), px * py = P, closest to square with py >= px (R23)."""
    px = int(P ** 0.5)
    while P % px:
        px -= 1
    return px, P // px


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["overlap", "regime", "detector", "partition", "direct", "oras"])
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--persistent", type=int, default=2, help="ras_options.async_persistent (0, 1, 2)")
    a = ap.parse_args()
    global ASYNC_PERSISTENT
    ASYNC_PERSISTENT = a.persistent
    recs = []
    if a.which == "overlap":
        # 1024^2, 4x4 subdomains of 256^2 (E4 shape: few subdomains, growing overlap)
        for g in (1, 2, 4, 8, 16):
            for mode in ("sync", "async"):
                recs.append(run(1024, 1024, 4, 4, g, mode, a.tol, reps=1 if mode == "sync" else a.reps))
    elif a.which == "regime":
        # 64^2 = 4096 unknowns per subdomain, overlap 16 (the paper's best async overlap, P594-598)
        for (px, py) in ((2, 2), (4, 4), (6, 6), (8, 8), (12, 8), (12, 12)):
            for mode in ("sync", "async"):
                recs.append(run(64 * px, 64 * py, px, py, 16, mode, a.tol, reps=1 if mode == "sync" else a.reps))
    elif a.which == "partition":
        recs = partition_study(a.tol, a.reps)
    elif a.which == "direct":
        for (px, py) in ((4, 4), (8, 8), (12, 12)):
            for solver in ("cholesky", "jacobi"):
                for mode in ("sync", "async"):
                    recs.append(run(64 * px, 64 * py, px, py, 4, mode, a.tol, solver=solver,
                                    reps=1 if mode == "sync" else a.reps))
    elif a.which == "oras":
        for solver, m in (("cholesky", 1), ("jacobi", 20)):
            for w in (0.0, 0.3, 0.5, 0.7, 0.8, 0.9):
                recs.append({"robin": w, **run(256, 256, 4, 4, 2, "sync", a.tol, m=m, solver=solver, robin=w)})
    else:
        for det in ("central", "decentral"):
            recs.append(run(512, 512, 8, 8, 16, "async", a.tol, detector=det, reps=a.reps))
    lines = [json.dumps({"experiment": a.which, **r}) for r in recs]
    for ln in lines:
        print(ln, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
