"""R33 diagnosis, step 2: the persistent kernel with one CTA per strip made
synchronous by grid barriers (RAS_PERSISTENT_LOCKSTEP=1) must BE the synchronous
sweep: iterate parity with the oracle's ras_sync after K rounds, and the sync sweep
count to 1e-8.  If it is, the kernel computes correctly with one CTA per subdomain
and the free-running divergence comes from the asynchronous schedule itself."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
os.environ["RAS_PERSISTENT_LOCKSTEP"] = "1"
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2003_05361_b200 as R  # noqa: E402
import ras_inputs as ri  # noqa: E402

N = 256
A = ri.laplace_2d(N)
b = ri.rhs(N * N, 0)
owner = R.partition_regular(N, N, 1, 1, 16, 1)
subs = O.setup(A, b, np.asarray(owner), 4)
for s_ in subs:
    O.make_local_solver(s_, "jacobi", 20)
K = 5
ref = O.ras_sync(A, b, subs, 1e-300, K, record_iterates=True)
s = R.Solver(A, b, owner, 4, R.options("jacobi", 20, async_persistent=1, persistent_grid=16, max_resumes=0))
st, x = s.solve(1e-300, K, "async")
err = float(np.linalg.norm(x - ref.iterates[K]) / np.linalg.norm(ref.iterates[K]))
print(json.dumps({"lockstep_rounds": K, "rel_diff_vs_oracle_sync": err, "updates": s.stats()["updates_max"]}), flush=True)
st, x = s.solve(1e-8, 5000, "async")
d = s.stats()
print(json.dumps({"lockstep_to_1e-8": int(st), "updates": d["updates_max"], "rel": d["final_rel_residual"]}), flush=True)
s.close()
