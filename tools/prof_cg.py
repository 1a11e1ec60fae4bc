"""ncu driver: a short fixed-iteration PCG on the C2 mesh."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import semgen
from paper_2405_05640_b200 import sem
per = int(os.environ.get("PER", "32"))
xi, _ = sem.sem_gll(7)
m = semgen.box_mesh((per, per, per), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, 7, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
f = torch.from_numpy(semgen.tgv_source(m["coords"]).reshape(E, -1)).cuda()
b = torch.empty_like(f); mesh.rhs(f, b); x = torch.zeros_like(f)
mesh.cg_solve(b, x, tol=0.0, maxit=int(os.environ.get("ITERS", "3")))
torch.cuda.synchronize()
print("done")
