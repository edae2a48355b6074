"""R33 diagnosis: persistent async kernel on the thin-strip configuration with the
CTA count capped (persistent_grid), fixed-m PCG vs exact local solves."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_2003_05361_b200 as R  # noqa: E402
import ras_inputs as ri  # noqa: E402

N = 256
A = ri.laplace_2d(N)
b = ri.rhs(N * N, 0)
owner = R.partition_regular(N, N, 1, 1, 16, 1)
for kind, m in (("jacobi", 20), ("exact", 20)):
    for G in (1, 2, 4, 8, 16):
        s = R.Solver(A, b, owner, 4, R.options(kind, m, async_persistent=1, persistent_grid=G, max_resumes=0))
        st, x = s.solve(1e-8, 4000, "async", gather=False)
        d = s.stats()
        print(json.dumps({"kind": kind, "m": m, "G": G, "status": int(st), "max": d["updates_max"],
                          "min": d["updates_min"], "rel": d["final_rel_residual"],
                          "tts": round(d["time_to_solution_s"], 4)}), flush=True)
        s.close()
