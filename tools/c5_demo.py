#!/usr/bin/env python
"""BASELINE configs[4] shape (C5) at reduced scale: 2D Laplacian, graph-
partitioned (seeded Voronoi stand-in for METIS, P217) irregular subdomains, 8 per
GPU, overlap 8, Jacobi-PCG m=20; sync (NCCL) vs async (NVLink puts) with the
centralized and decentralized detectors (P481-484, E8).  A fixed sweep / update
budget gives iteration rates (a 1e-8 solve of this size needs ~1e5 sweeps).
Each rank builds only its row window of A.  Launch with torchrun:

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/c5_demo.py --side 7072 --iters 100
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=7072)
    ap.add_argument("--per-gpu", type=int, default=8)
    ap.add_argument("--gamma", type=int, default=8)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--modes", default="sync,async:central,async:decentral")
    ap.add_argument("--robin", type=float, default=0.0)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--unbalanced", action="store_true", help="plain Voronoi cells (default: Lloyd + power-diagram balanced)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2003_05361_b200 as R

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N, P, g = a.side, a.per_gpu * world, a.gamma
    t0 = time.perf_counter()
    owner = None
    for seed in range(1, 50):
        try:
            owner = (ri.voronoi_partition(N, N, P, seed=seed) if a.unbalanced
                     else ri.voronoi_partition(N, N, P, seed=seed, lloyd=8, balance=60))
            break
        except ValueError:
            continue
    s2r = np.array([(p * world) // P for p in range(P)], dtype=np.int32)
    rows = np.nonzero(s2r[owner] == rank)[0]
    r0 = max(0, int(rows.min()) - (g + 1) * N)
    r1 = min(N * N, int(rows.max()) + 1 + (g + 1) * N)
    A = ri.laplace_2d_rows(N, N, r0, r1)
    b = ri.rhs(N * N, 0)[r0:r1]
    t_inputs = time.perf_counter() - t0
    res = []
    for spec in a.modes.split(","):
        mode, _, det = spec.partition(":")
        det = det or "central"
        obj = [R.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        t1 = time.perf_counter()
        s = R.Solver(A, b, owner, g, R.options("jacobi", 20, detector=det, robin=a.robin, async_timeout_s=3000.0),
                     comm={"rank": rank, "world": world, "device": local, "nccl_id": obj[0]})
        t_setup = time.perf_counter() - t1
        if world > 1:
            dist.barrier()
        st, _ = s.solve(a.tol, a.iters, mode, gather=False)
        d = s.stats()
        t = torch.tensor([d["time_to_solution_s"]], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res.append({"mode": mode, "detector": det if mode == "async" else None, "status": int(st), "robin": a.robin,
                    "time_s": float(t[0]), "sweeps_or_max_updates": d["sweeps"], "updates_min": d["updates_min"],
                    "rel_residual": d["final_rel_residual"], "pcg_path": d["pcg_path"], "setup_s": t_setup,
                    "resident_lanes": d["resident_lanes"], "resident_pattern": d["resident_pattern"],
                    "verified": d["verified"], "phase_s": {k: d[k] for k in ("t_residual", "t_local_solve",
                                                                            "t_exchange", "t_convcheck")},
                    "resumes": d["resumes"], "per_sweep_ms": 1e3 * float(t[0]) / max(d["sweeps"], 1)})
        s.close()
    if rank == 0:
        for r in res:
            print(json.dumps({"experiment": "c5_demo", "gpus": world, "grid": [N, N], "unknowns": N * N,
                              "subdomains": P, "overlap": g, "inputs_s": t_inputs, **r}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
