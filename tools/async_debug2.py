"""R33 evidence, step 1 (R33, profiles/r02_r33_investigation.md): 256^2 Laplacian,
16 strips, overlap 4, async to 1e-8 -- the persistent kernel vs the stream driver with fixed-m
Jacobi-PCG (m = 5, 20, 60) and with exact local solves, and the sync sweep count beside them."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2003_05361_b200 as R, ras_inputs as ri
N = 256
A = ri.laplace_2d(N); b = ri.rhs(N * N, 0)
owner = R.partition_regular(N, N, 1, 1, 16, 1)
for kind, m, pers in (("jacobi", 20, 1), ("jacobi", 20, 0), ("jacobi", 60, 1), ("jacobi", 5, 1), ("exact", 20, 1), ("exact", 20, 0)):
    s = R.Solver(A, b, owner, 4, R.options(kind, m, async_persistent=pers))
    st, x = s.solve(1e-8, 5000, "async", gather=False)
    d = s.stats()
    print(json.dumps({"kind": kind, "m": m, "persistent": pers, "status": int(st), "max": d["updates_max"],
                      "min": d["updates_min"], "rel": d["final_rel_residual"], "inner": d["inner_iters_total"]}), flush=True)
    s.close()
# sync reference
s = R.Solver(A, b, owner, 4, R.options("jacobi", 20))
st, x = s.solve(1e-8, 5000, "sync", gather=False)
print(json.dumps({"sync": True, "status": int(st), "sweeps": s.stats()["sweeps"]}))
