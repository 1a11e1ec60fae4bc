"""Real-run (not under ncu) timing of the operator pieces on C2 with CUDA events."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import semgen
from paper_2405_05640_b200 import sem
per = int(os.environ.get("PER", "32")); N = int(os.environ.get("NORD", "7"))
xi, _ = sem.sem_gll(N)
m = semgen.box_mesh((per, per, per), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
u = torch.from_numpy(semgen.random_field((E, (N + 1) ** 3), 1)).cuda()
w = torch.empty_like(u)
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
res = {"env": {k: os.environ.get(k) for k in ("SEM_CHUNK_SHIFT", "SEM_GS_OVERLAP", "SEM_LANES", "SEM_GRAPH")},
       "ax_us": t(lambda: mesh.ax(u, w)), "gs_us": t(lambda: mesh.gs_op(w)),
       "ax_dssum_us": t(lambda: mesh.ax_dssum(u, w))}
b = torch.empty_like(u); mesh.rhs(u, b); x = torch.zeros_like(u)
res["cg100_ms"] = t(lambda: mesh.cg_solve(b, x, tol=0.0, maxit=100), reps=3) / 1e3
res["variant"] = os.environ.get("SEM_CG_VARIANT")
print(json.dumps(res))
