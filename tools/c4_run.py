#!/usr/bin/env python
"""BASELINE configs[3] shape (C4): 3D 7-point Laplacian, regular box subdomains,
overlap 4, IC(0)-PCG (level-scheduled triangular solves, a3') or Jacobi-PCG,
solved to rel. residual 1e-8 in sync (NCCL) and async (NVLink puts) mode; weak
scaling with one 256^3 subdomain per GPU.  Launch with torchrun (1..8 GPUs):

  python -m torch.distributed.run --nproc-per-node G tools/c4_run.py --grid 512 256 256 --parts 2 1 1
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
    ap.add_argument("--grid", type=int, nargs=3, default=[256, 256, 256])
    ap.add_argument("--parts", type=int, nargs=3, default=[1, 1, 1])
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--solvers", default="ic0:10")
    ap.add_argument("--modes", default="sync,async")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--iters", type=int, default=100000)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2003_05361_b200 as R

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx, ny, nz = a.grid
    px, py, pz = a.parts
    P = px * py * pz
    owner = R.partition_regular(nx, ny, nz, px, py, pz)
    s2r = np.array([(p * world) // P for p in range(P)], dtype=np.int32)
    rows = np.nonzero(s2r[owner] == rank)[0]
    plane = nx * ny
    r0 = max(0, int(rows.min()) - (a.gamma + 1) * plane)
    r1 = min(nx * ny * nz, int(rows.max()) + 1 + (a.gamma + 1) * plane)
    A = ri.laplace_3d_rows(nx, ny, nz, r0, r1)
    b = ri.rhs(nx * ny * nz, 0)[r0:r1]
    out = []
    for sv in a.solvers.split(","):
        kind, _, m = sv.partition(":")
        for mode in a.modes.split(","):
            obj = [R.nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            t1 = time.perf_counter()
            s = R.Solver(A, b, owner, a.gamma, R.options(kind, int(m or 10), async_timeout_s=3000.0),
                         comm={"rank": rank, "world": world, "device": local, "nccl_id": obj[0]})
            t_setup = time.perf_counter() - t1
            if world > 1:
                dist.barrier()
            st, _ = s.solve(a.tol, a.iters, mode, gather=False)
            d = s.stats()
            t = torch.tensor([d["time_to_solution_s"]], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out.append({"solver": f"{kind}-PCG m={m or 10}", "mode": mode, "status": int(st), "time_s": float(t[0]),
                        "sweeps_or_max_updates": d["sweeps"], "updates_min": d["updates_min"],
                        "inner_iters_total": d["inner_iters_total"], "rel_residual": d["final_rel_residual"],
                        "verified": d["verified"], "resumes": d["resumes"], "pcg_path": d["pcg_path"],
                        "setup_s": t_setup, "per_sweep_ms": 1e3 * float(t[0]) / max(d["sweeps"], 1),
                        "phase_s": {k: d[k] for k in ("t_residual", "t_local_solve", "t_exchange", "t_convcheck")}})
            s.close()
    if rank == 0:
        for r in out:
            print(json.dumps({"experiment": "c4_run", "gpus": world, "grid": [nx, ny, nz], "parts": [px, py, pz],
                              "unknowns": nx * ny * nz, "overlap": a.gamma, **r}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
