import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, paper_2003_05361_b200 as R, ras_inputs as ri
N=1024; A=ri.laplace_2d(N); b=ri.rhs(N*N,0); owner=R.partition_regular(N,N,1,4,4,1)
xs={}
for name, env, path in (("v2",None,"resident"),("v1","1","resident"),("tiled",None,"tiled")):
    if env: os.environ["RAS_RESIDENT_KERNEL"]=env
    else: os.environ.pop("RAS_RESIDENT_KERNEL", None)
    s=R.Solver(A,b,owner,8,R.options("jacobi",20,path=path))
    st,x=s.solve(1e-300, 400, "sync"); xs[name]=x; t=s.stats(); print(name, t["resident_lanes"], t["final_rel_residual"]); 
    st,x=s.solve(1e-8, 100000, "sync", gather=False); print(name, "sweeps to 1e-8:", s.stats()["sweeps"]); s.close()
for a in ("v1","tiled"): print("v2 vs", a, np.linalg.norm(xs["v2"]-xs[a])/np.linalg.norm(xs[a]))
