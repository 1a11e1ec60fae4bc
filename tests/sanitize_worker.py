"""Every kernel of the library on small meshes, for compute-sanitizer
(tests/test_gpu_sanitize.py runs this under memcheck, racecheck, synccheck
and initcheck).  Exercises: geometry, multiplicity/mask, the operator (all
coefficient modes, CG fusion, affine variant), Ax+dssum, standalone
gather-scatter, RHS, Jacobi, standard PCG (conditional-graph loop,
per-iteration graphs, stream order), the single-reduction PCG, the
host-buffer path, restarted GMRES and the splitting time step.  Exit 0
when every call returned SEM_OK and the results are finite."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import semgen  # noqa: E402
from paper_2405_05640_b200 import sem  # noqa: E402


def run_case(kind):
    if kind == "box":
        N = 7
        xl, _ = sem.sem_gll(N)
        m = semgen.box_mesh((3, 3, 4), xl, periodic=(True, False, True), deform=0.2)
    else:
        N = 9
        xl, _ = sem.sem_gll(N)
        m = semgen.cylinder_mesh(xl, nc=2, nr=1, nz=3)
    E = m["conn"].shape[0]
    n3 = (N + 1) ** 3
    mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
    mesh.geom_factors()
    rng = np.random.default_rng(1)
    u = torch.from_numpy(rng.uniform(-1, 1, (E, n3))).cuda()
    h1 = torch.from_numpy(rng.uniform(0.5, 1.5, (E, n3))).cuda()
    h2 = torch.from_numpy(rng.uniform(0.5, 1.5, (E, n3))).cuda()
    w = torch.empty_like(u)
    outs = []
    mesh.ax(u, w)
    mesh.ax(u, w, h1c=0.5, h2c=2.0)
    mesh.ax(u, w, h1=h1, h2=h2)
    for _ in range(2):
        mesh.ax_dssum(u, w)
        mesh.ax_dssum(u, w, h1c=0.5, h2c=2.0)
        outs.append(w.clone())
    d = u.clone()
    mesh.gs_op(d, sem.SEM_GS_ADD)
    mesh.gs_op(d, sem.SEM_GS_MASK)
    b = torch.empty_like(u)
    mesh.rhs(u, b)
    dinv = torch.empty_like(u)
    mesh.jacobi(dinv, h1=h1, h2=h2)
    x = torch.zeros_like(u)
    for graph in (1, 0):
        mesh.set_options(graph=graph)
        mesh.cg_solve(b, x, tol=1e-8, maxit=200)
        mesh.cg_solve(b, x, h1=h1, h2=h2, tol=0.0, maxit=5)
    mesh.set_options(graph=1)
    mesh.profile_enable(True)
    mesh.cg_solve(b, x, tol=0.0, maxit=4)
    mesh.profile_get()
    mesh.profile_enable(False)
    mesh.set_options(cg_variant="pipelined")
    mesh.cg_solve(b, x, tol=1e-8, maxit=200)
    mesh.set_options(cg_variant="standard")
    bh = b.cpu().pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    mesh.cg_solve_host(bh, xh, tol=0.0, maxit=3)
    mesh.gmres_solve(b, x, h1=h1, h2=h2, tol=1e-8, maxit=40, restart=8)
    mesh.gmres_solve(b, x, tol=0.0, maxit=12, restart=5)
    if kind == "box":
        mesh.set_options(affine=1)  # deformed: detection runs, general path stays
    torch.cuda.synchronize()
    ok = all(bool(torch.isfinite(o).all()) for o in outs + [x, d, dinv])
    mesh.close()
    return ok


def main():
    torch.cuda.set_device(0)
    ok = True
    for kind in ("box", "cyl"):
        ok = run_case(kind) and ok
    # an undeformed box: the affine-element operator
    xl, _ = sem.sem_gll(5)
    m = semgen.box_mesh((3, 3, 3), xl)
    mesh = sem.Mesh(27, 5, m["coords"], m["conn"], m["bc"])
    mesh.geom_factors()
    mesh.set_options(affine=1)
    u = torch.ones((27, 216), dtype=torch.float64, device="cuda")
    w = torch.empty_like(u)
    mesh.ax_dssum(u, w)
    x = torch.zeros_like(u)
    mesh.cg_solve(w, x, tol=0.0, maxit=3)
    torch.cuda.synchronize()
    mesh.close()
    # a periodic box: the splitting time step (metrics, convection, weak
    # divergence, gradient, four PCG solves)
    m = semgen.box_mesh((3, 3, 3), xl, periodic=(True, True, True), deform=0.1)
    mesh = sem.Mesh(27, 5, m["coords"], m["conn"], m["bc"])
    mesh.geom_factors()
    uvw = torch.from_numpy(semgen.tgv_velocity(m["coords"]).reshape(3, 27, 216)).cuda().contiguous()
    p = torch.zeros((27, 216), dtype=torch.float64, device="cuda")
    mesh.pnpn_step(uvw, p, dt=1e-2, nu=1e-2, tol=1e-8, maxit=200)
    torch.cuda.synchronize()
    ok = ok and bool(torch.isfinite(uvw).all()) and bool(torch.isfinite(p).all())
    mesh.close()
    print("sanitize worker ok" if ok else "sanitize worker: non-finite results", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
