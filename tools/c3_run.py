#!/usr/bin/env python
"""BASELINE configs[2] as specified (C3): 2D 5-point Laplacian with 2^24 unknowns
per GPU and ONE subdomain per GPU (4096^2 at G=1, 4096 x 8192 at G=2, 8192^2 at
G=4, 8192 x 16384 at G=8), overlap gamma in {1, 2, 4, 8}, Jacobi-PCG m = 20, sync
(NCCL) and async (NVLink puts); time per sweep (sync) / per subdomain update
(async) over a fixed number of sweeps (P574-598: the overlap study; a one-level
method with 2^24-row subdomains does not reach 1e-8 in a bounded run).  Launch
with torchrun, one process per GPU:

  python -m torch.distributed.run --nproc-per-node G tools/c3_run.py
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ras_inputs as ri  # noqa: E402

GRIDS = {1: (4096, 4096, 1, 1), 2: (4096, 8192, 1, 2), 4: (8192, 8192, 2, 2), 8: (8192, 16384, 2, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gammas", default="1,2,4,8")
    ap.add_argument("--modes", default="sync,async")
    ap.add_argument("--sweeps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2003_05361_b200 as R

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx, ny, px, py = GRIDS[world]
    owner = R.partition_regular(nx, ny, 1, px, py, 1)
    rows = np.nonzero(owner == rank)[0]  # one subdomain per GPU: subdomain id = rank
    out = []
    for g in (int(x) for x in a.gammas.split(",")):
        r0 = max(0, int(rows.min()) - (g + 1) * nx)
        r1 = min(nx * ny, int(rows.max()) + 1 + (g + 1) * nx)
        A = ri.laplace_2d_rows(nx, ny, r0, r1)
        b = ri.rhs(nx * ny, 0)[r0:r1]
        for mode in a.modes.split(","):
            obj = [R.nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            s = R.Solver(A, b, owner, g, R.options("jacobi", 20),
                         comm={"rank": rank, "world": world, "device": local, "nccl_id": obj[0]})
            s.solve(1e-300, 2, mode, gather=False)  # warm-up
            if world > 1:
                dist.barrier()
            st, _ = s.solve(1e-300, a.sweeps, mode, gather=False)
            d = s.stats()
            t = torch.tensor([d["time_to_solution_s"]], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            n_upd = max(d["sweeps"], 1)
            out.append({"overlap": g, "mode": mode, "status": int(st), "time_s": float(t[0]), "sweeps_or_max_updates": d["sweeps"],
                        "updates_min": d["updates_min"], "ms_per_sweep_or_update": 1e3 * float(t[0]) / n_upd,
                        "rel_residual": d["final_rel_residual"], "pcg_path": d["pcg_path"],
                        "phase_s": {k: d[k] for k in ("t_residual", "t_local_solve", "t_exchange", "t_convcheck")}})
            s.close()
    if rank == 0:
        for r in out:
            print(json.dumps({"experiment": "c3_run", "gpus": world, "grid": [nx, ny], "subdomains": world,
                              "unknowns_per_gpu": nx * ny // world, "local_solver": "jacobi-PCG m=20", **r}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
