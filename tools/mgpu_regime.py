#!/usr/bin/env python
"""Multi-GPU sync vs async in the paper's latency regime (NEXT f2, PAPER E9,
P716-735): 64^2 = 4096 unknowns per subdomain, overlap 16, Jacobi-PCG m=20,
regular tiles, contiguous subdomain blocks per GPU.  Launch with torchrun:

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_regime.py [--tiles 12x12]
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
    ap.add_argument("--tiles", default="12x12")
    ap.add_argument("--gamma", type=int, default=16)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-8)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2003_05361_b200 as R

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    def nccl_id():  # a fresh NCCL communicator id per solver context
        obj = [R.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return obj[0]
    px, py = (int(v) for v in a.tiles.split("x"))
    nx, ny = 64 * px, 64 * py
    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    owner = R.partition_regular(nx, ny, 1, px, py, 1)
    out = []
    for persistent in (1, 0):  # 1: force the persistent kernel for the fixed-m solves (opt-in, R33)
        s = R.Solver(A, b, owner, a.gamma, R.options("jacobi", 20, async_persistent=persistent),
                     comm={"rank": rank, "world": world, "device": local, "nccl_id": nccl_id()})
        for mode in ("sync", "async"):
            if mode == "sync" and persistent == 0:
                continue
            for _ in range(a.reps if mode == "async" else 1):
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                st, x = s.solve(a.tol, 200000, mode, gather=False)
                wall = time.perf_counter() - t0
                d = s.stats()
                t = torch.tensor([d["time_to_solution_s"], float(d["updates_max"]), float(d["updates_min"])],
                                 dtype=torch.float64, device="cuda")
                if world > 1:
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                out.append({"mode": mode, "driver": ("persistent" if persistent else "streams") if mode == "async"
                            else "sync", "status": int(st), "tts_s_max_over_ranks": float(t[0]),
                            "updates_max": int(t[1]), "rel_residual": d["final_rel_residual"],
                            "resumes": d["resumes"], "launches": d["kernel_launches"], "wall_s": wall})
        s.close()
    if rank == 0:
        for r in out:
            print(json.dumps({"experiment": "mgpu_regime", "gpus": world, "tiles": [px, py], "subdomains": px * py,
                              "unknowns_per_subdomain": 4096, "overlap": a.gamma, **r}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
