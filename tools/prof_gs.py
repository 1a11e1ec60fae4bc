"""ncu driver: standalone gs_op and ax_dssum on the c2 mesh."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch
import semgen
from paper_2405_05640_b200 import sem
xi, _ = sem.sem_gll(7)
m = semgen.box_mesh((32, 32, 32), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, 7, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
u = torch.from_numpy(semgen.random_field((E, 512), 1)).cuda()
w = torch.empty_like(u)
for _ in range(2):
    mesh.gs_op(w)
for _ in range(2):
    mesh.ax_dssum(u, w)
torch.cuda.synchronize()
print("done")
