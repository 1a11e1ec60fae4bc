"""ncu / timing driver: restarted GMRES on a periodic box (PER^3 elements,
order NORD), STEPS Arnoldi steps with restart RESTART, tol TOL (0), preconditioner
PC (jacobi | hsmg).  Prints the
event-timed ms per Arnoldi step (second run; the first is warm-up)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch
import semgen
from paper_2405_05640_b200 import sem
per = int(os.environ.get("PER", "32"))
N = int(os.environ.get("NORD", "7"))
steps = int(os.environ.get("STEPS", "30"))
restart = int(os.environ.get("RESTART", "30"))
xi, _ = sem.sem_gll(N)
m = semgen.box_mesh((per, per, per), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
mesh.set_options(gmres_precond=os.environ.get("PC", "jacobi"), hsmg_coarse_iters=int(os.environ.get("COARSE", "20")))
f = torch.from_numpy(semgen.tgv_source(m["coords"]).reshape(E, -1)).cuda()
b = torch.empty_like(f); mesh.rhs(f, b); x = torch.zeros_like(f)
for rep in range(int(os.environ.get("REPS", "2"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    it, rr, _ = mesh.gmres_solve(b, x, tol=float(os.environ.get("TOL", "0")), maxit=steps, restart=restart)
    e1.record(); torch.cuda.synchronize()
    print(f"rep {rep}: {it} steps, {e0.elapsed_time(e1) / it:.4f} ms/step, rel_res {rr:.3e}", flush=True)
