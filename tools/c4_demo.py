#!/usr/bin/env python
"""BASELINE configs[3] shape (C4) on one GPU at reduced scale: 3D 7-point
Laplacian N^3, 2x2x2 subdomains, overlap 4, IC(0)-PCG m=10 with level-scheduled
triangular solves (a3'), sync: per-sweep time and per-kernel split.

  python tools/c4_demo.py [--side 256] [--sweeps 10]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ras_inputs as ri  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--sweeps", type=int, default=10)
    ap.add_argument("--solver", default="ic0")
    a = ap.parse_args()
    import paper_2003_05361_b200 as R

    N = a.side
    t0 = time.perf_counter()
    A = ri.laplace_3d(N)
    b = ri.rhs(N ** 3, 0)
    owner = R.partition_regular(N, N, N, 2, 2, 2)
    t1 = time.perf_counter()
    s = R.Solver(A, b, owner, 4, R.options(a.solver, 10))
    t2 = time.perf_counter()
    s.solve(1e-300, 2, "sync", gather=False)
    s.kernel_timing(True)
    s.solve(1e-300, a.sweeps, "sync", gather=False)
    kt = s.kernel_times()
    st = s.stats()
    tot = sum(v[1] for v in kt.values())
    # levels of one triangular solve of a corner subdomain (natural order on the
    # gamma-hop Omega_p of a box: deepest row x+y+z = 3(N/2 - 1) + gamma)
    levels = 3 * (N // 2 - 1) + 4 + 1
    print(json.dumps({"experiment": "c4_demo", "grid": [N, N, N], "unknowns": N ** 3, "subdomains": 8, "overlap": 4,
                      "local_solver": f"{a.solver}-PCG m=10", "inputs_s": t1 - t0, "setup_s": t2 - t1,
                      "ms_per_sweep": tot / a.sweeps, "pcg_path": st["pcg_path"],
                      "trsv": os.environ.get("RAS_TRSV", "ds"), "levels_per_solve": levels,
                      "us_per_level": (1e3 * kt["k_trsv"][1] / kt["k_trsv"][0] / levels) if kt.get("k_trsv", (0,))[0] else None,
                      "kernels": {k: {"launches": v[0], "ms_per_sweep": v[1] / a.sweeps, "share": v[1] / tot}
                                  for k, v in kt.items() if v[0]}}), flush=True)


if __name__ == "__main__":
    main()
