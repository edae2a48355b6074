import os, sys
sys.path.insert(0, os.getcwd())
import paper_2003_05361_b200 as R, ras_inputs as ri
A = ri.laplace_2d(256); b = ri.rhs(256 * 256, 0)
owner = R.partition_regular(256, 256, 1, 4, 4, 1)
s = R.Solver(A, b, owner, 4, R.options("cholesky"))
s.solve(1e-300, 3, "sync", gather=False)
print("ok")
