#!/usr/bin/env python
"""Small solves through every kernel path, for compute-sanitizer (SURVEY §4
layer 6): memcheck / racecheck / synccheck on C1-size problems.

  compute-sanitizer --tool memcheck python tools/sanitize_paths.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_05361_b200 as R  # noqa: E402
import ras_inputs as ri  # noqa: E402


def check(A, b, x, tol):
    r = b - A.to_scipy() @ x
    rel = np.linalg.norm(r) / np.linalg.norm(b)
    assert rel < tol, rel
    return rel


def main():
    N = 48
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = ri.voronoi_partition(N, N, 4, seed=2)
    cases = [("jacobi", "tiled", {}), ("jacobi", "block", {}), ("jacobi", "resident", {}),
             ("exact", "resident", {}), ("ic0", "auto", {}), ("cholesky", "auto", {}),
             ("jacobi", "auto", {"robin": 0.5})]
    for kind, path, kw in cases:
        s = R.Solver(A, b, owner, 2, R.options(kind, 10, path=path, **kw))
        st, x = s.solve(1e-8, 5000, "sync")
        print(kind, path, kw, "sync", st, s.stats()["sweeps"], check(A, b, x, 1e-8), flush=True)
        s.close()
    for persistent in (1, 0):
        s = R.Solver(A, b, owner, 2, R.options("jacobi", 10, async_persistent=persistent))
        st, x = s.solve(1e-8, 20000, "async")
        print("async persistent" if persistent else "async streams", st, check(A, b, x, 1e-8), flush=True)
        s.close()
    print("ok")


if __name__ == "__main__":
    main()
