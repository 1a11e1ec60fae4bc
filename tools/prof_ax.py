"""Small driver for ncu: builds the C2 mesh and runs the fused operator
(standalone Ax+dssum, local Ax, and a short fixed-iteration PCG)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch  # noqa: E402

import semgen  # noqa: E402
from paper_2405_05640_b200 import sem  # noqa: E402

per = int(os.environ.get("PER", "32"))
N = int(os.environ.get("NORD", "7"))
reps = int(os.environ.get("REPS", "3"))
xi, _ = sem.sem_gll(N)
m = semgen.box_mesh((per, per, per), xi, deform=float(os.environ.get("DEFORM", "0")))
E = m["conn"].shape[0]
mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
u = torch.from_numpy(semgen.random_field((E, (N + 1) ** 3), 1)).cuda()
w = torch.empty_like(u)
for _ in range(reps):
    mesh.ax_dssum(u, w)
for _ in range(reps):
    mesh.ax(u, w)
b = torch.empty_like(u)
mesh.rhs(u, b)
x = torch.zeros_like(u)
mesh.cg_solve(b, x, tol=0.0, maxit=reps)
torch.cuda.synchronize()
print("done", E)
for _ in range(reps):
    mesh.gs_op(w, sem.SEM_GS_ADD)
torch.cuda.synchronize()
