"""ncu/timing driver for the lx = 10 cylinder (C5 shape, fewer layers)."""
import math, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch
import semgen
from paper_2405_05640_b200 import sem
nz = int(os.environ.get("NZ", "32"))
xi, _ = sem.sem_gll(9)
m = semgen.cylinder_mesh(xi, nc=32, nr=16, nz=nz)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, 9, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
mesh.set_options(graph=int(os.environ.get("GRAPH", "1")))
h1c, h2c = math.sqrt(1e-11), (11 / 6) / 1e-3
u = torch.from_numpy(semgen.random_field((E, 1000), 1)).cuda()
w = torch.empty_like(u)
def t(f, reps=10):
    for _ in range(2): f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
res = {"E": E, "ax_us": t(lambda: mesh.ax(u, w, h1c=h1c, h2c=h2c)), "gs_us": t(lambda: mesh.gs_op(w)),
       "ax_dssum_us": t(lambda: mesh.ax_dssum(u, w, h1c=h1c, h2c=h2c))}
b = torch.empty_like(u); mesh.rhs(u, b); x = torch.zeros_like(u)
res["cg10_ms"] = t(lambda: mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=0.0, maxit=10), reps=2) / 1e3
res["cg_ms_per_iter"] = (t(lambda: mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=0.0, maxit=60), reps=2) - t(lambda: mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=0.0, maxit=10), reps=2)) / 50 / 1e3
print(json.dumps(res))
