import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["RAS_SETUP_TRACE"]="1"
import numpy as np, paper_2003_05361_b200 as R, ras_inputs as ri
A=ri.laplace_2d(4096); b=ri.rhs(4096*4096,0); owner=R.partition_regular(4096,4096,1,4,4,1)
for dev in (1,0):
    t=time.time(); s=R.Solver(A,b,owner,8,R.options("jacobi",20,device_setup=dev)); print("device_setup",dev,"setup_s",s.stats()["setup_s"] if False else time.time()-t, flush=True); s.close()
