"""R33 diagnosis, step 3: the persistent kernel with one CTA per strip (the diverging
configuration) with whole-update neighbour snapshots (RAS_PERSISTENT_SEQLOCK=1: a
residual is recomputed until no data neighbour wrote x[S_q] during it), next to the
free-running kernel (RAS_PERSISTENT_SEQLOCK=0).  If the snapshots converge,
the divergence comes from residuals that mix a neighbour's old and new values."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1:  # child: one configuration (the env vars are read at context setup)
    sys.path.insert(0, os.getcwd())
    import paper_2003_05361_b200 as R  # noqa: E402
    import ras_inputs as ri  # noqa: E402

    N = 256
    A = ri.laplace_2d(N)
    b = ri.rhs(N * N, 0)
    owner = R.partition_regular(N, N, 1, 1, 16, 1)
    kind, m, G = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    s = R.Solver(A, b, owner, 4, R.options(kind, m, async_persistent=1, persistent_grid=G, max_resumes=0))
    st, x = s.solve(1e-8, 4000, "async", gather=False)
    d = s.stats()
    print(json.dumps({"mode": os.environ.get("R33_MODE"), "kind": kind, "m": m, "G": G, "status": int(st),
                      "max": d["updates_max"], "min": d["updates_min"], "rel": d["final_rel_residual"],
                      "tts": round(d["time_to_solution_s"], 4)}), flush=True)
    s.close()
    sys.exit(0)

for mode, env in (("free", {"RAS_PERSISTENT_SEQLOCK": "0"}), ("seqlock", {"RAS_PERSISTENT_SEQLOCK": "1"})):
    for kind, m, G in (("jacobi", 20, 16), ("jacobi", 20, 8), ("jacobi", 5, 16), ("exact", 20, 16)):
        e = dict(os.environ, R33_MODE=mode, **env)
        subprocess.run([sys.executable, __file__, kind, str(m), str(G)], env=e, timeout=600)
