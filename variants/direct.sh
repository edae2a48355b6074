#!/bin/bash
# direct local solve timing (16 subdomains of 64^2, overlap 4, 100 sweeps) for the listed builds
for v in "$@"; do
RAS_LIB_PATH=$PWD/variants/lib_$v.so python - <<'PY'
import os, time, sys
sys.path.insert(0, os.getcwd())
import paper_2003_05361_b200 as R, ras_inputs as ri
nx = ny = 256
A = ri.laplace_2d(nx, ny); b = ri.rhs(nx * ny, 0)
owner = R.partition_regular(nx, ny, 1, 4, 4, 1)
s = R.Solver(A, b, owner, 4, R.options("cholesky"))
s.solve(1e-300, 5, "sync", gather=False)
s.kernel_timing(True)
s.solve(1e-300, 100, "sync", gather=False)
kt = s.kernel_times()
print(os.environ["RAS_LIB_PATH"].split("/")[-1], "k_band_chol avg us", round(kt["k_band_chol"][1] / kt["k_band_chol"][0] * 1e3, 1))
PY
done
