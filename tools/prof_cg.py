"""ncu driver: a short fixed-iteration PCG on a periodic box (PER^3 elements,
order NORD, Helmholtz h2 = H2 if set)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch
import semgen
from paper_2405_05640_b200 import sem
per = int(os.environ.get("PER", "32"))
N = int(os.environ.get("NORD", "7"))
h2 = float(os.environ.get("H2", "0"))
xi, _ = sem.sem_gll(N)
m = semgen.box_mesh((per, per, per), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
mesh.set_options(graph=int(os.environ.get("GRAPH", "0")),  # stream order under ncu
                 cg_layout=int(os.environ.get("CG_LAYOUT", "1")))
f = torch.from_numpy(semgen.tgv_source(m["coords"]).reshape(E, -1)).cuda()
b = torch.empty_like(f); mesh.rhs(f, b); x = torch.zeros_like(f)
mesh.cg_solve(b, x, h2c=h2, tol=0.0, maxit=int(os.environ.get("ITERS", "3")))
torch.cuda.synchronize()
print("done")
