"""Small driver for one-launch ncu captures of the latency-regime kernels: the
direct banded-Cholesky local solve (k_band_chol, row f1) and the BLOCK Jacobi-PCG
(k_small_pcg, row f2) on the paper's 4096-unknown subdomains (512^2, 8x8
subdomains, overlap 4), a few sync sweeps each.

  ncu ... -k regex:k_band_chol python tools/ncu_small.py cholesky
  ncu ... -k regex:k_small_pcg python tools/ncu_small.py jacobi
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_2003_05361_b200 as R  # noqa: E402
import ras_inputs as ri  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "jacobi"
N = 512
A = ri.laplace_2d(N)
b = ri.rhs(N * N, 0)
owner = R.partition_regular(N, N, 1, 8, 8, 1)
s = R.Solver(A, b, owner, 4, R.options(kind, 20))
st, _ = s.solve(1e-300, 4, "sync", gather=False)
print(kind, s.stats()["pcg_path"], s.stats()["sweeps"])
s.close()
