import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2003_05361_b200 as R, ras_inputs as ri
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from experiments import voronoi_valid
N = 256
A = ri.laplace_2d(N); b = ri.rhs(N * N, 0)
cases = {"r1d16": R.partition_regular(N, N, 1, 1, 16, 1), "graph16": voronoi_valid(N, 16)}
for name, owner in cases.items():
    for pers in (1, 0):
        for det in ("decentral", "central"):
            s = R.Solver(A, b, owner, 4, R.options("jacobi", 20, detector=det, async_persistent=pers))
            st, x = s.solve(1e-8, 20000, "async", gather=False)
            d = s.stats()
            print(json.dumps({"case": name, "persistent": pers, "det": det, "status": int(st), "max": d["updates_max"],
                              "min": d["updates_min"], "med": d["updates_median"], "rel": d["final_rel_residual"],
                              "resumes": d["resumes"], "tts": round(d["time_to_solution_s"], 3)}), flush=True)
            s.close()
