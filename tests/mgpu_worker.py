"""Multi-GPU parity worker, launched by tests/test_gpu_multi.py as
    python -m torch.distributed.run --nproc-per-node P tests/mgpu_worker.py CASE
        [--p2p 0|1] [--variant standard|pipelined] [--repeat K] [--solver cg|gmres|hsmg]
Each rank builds its element block, creates the NCCL communicator through the
C ABI and compares the distributed results with the oracle on the global
mesh (restricted to its elements).  On fully periodic Poisson cases the
right-hand side has a non-zero mean (f + 0.7), so the singular-system
projections of b and x (reading R10) act across ranks.  --repeat K runs K
solves on the same communicator (sequence counters of the peer-memory
paths must stay in step; the communicator must report healthy after).
Exit code 0 = all checks passed."""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import semgen  # noqa: E402
from paper_2405_05640_b200 import sem  # noqa: E402

CASES = {
    "box2": dict(nel=(6, 3, 3), N=5, periodic=(True, True, True), grid=(2, 1, 1), deform=0.2),
    "walled2": dict(nel=(4, 4, 4), N=7, periodic=(False, False, False), grid=(2, 1, 1), deform=0.0),
    "box4": dict(nel=(6, 6, 3), N=4, periodic=(True, False, True), grid=(2, 2, 1), deform=0.1),
    "box8": dict(nel=(6, 6, 6), N=3, periodic=(True, True, True), grid=(2, 2, 2), deform=0.1),
}


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / (nb if nb else 1.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--p2p", type=int, default=1)
    ap.add_argument("--variant", default="standard")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--solver", default="cg", choices=["cg", "gmres", "hsmg"])
    ap.add_argument("--layout", type=int, default=1, help="option cg_layout")
    args = ap.parse_args()
    case = CASES[args.case]
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    uid = [sem.sem_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.sem_comm_create(uid[0], rank, ws, lr, p2p=bool(args.p2p))
    nel, N, per, grid = case["nel"], case["N"], case["periodic"], case["grid"]
    lx, n3 = N + 1, (N + 1) ** 3
    elems = semgen.box_partition(nel, grid, rank)
    xl, _ = sem.sem_gll(N)
    ml = semgen.box_mesh(nel, xl, periodic=per, deform=case["deform"], elems=elems)
    mesh = sem.Mesh(len(elems), N, ml["coords"], ml["conn"], ml["bc"], comm)
    mesh.geom_factors()
    mesh.set_options(cg_variant=args.variant, cg_layout=args.layout)
    # oracle on the global mesh
    xo, _ = oracle.gll(N)
    mo = semgen.box_mesh(nel, xo, periodic=per, deform=case["deform"])
    G, B = oracle.geom(N, mo["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, per)
    mask = oracle.mask_from_bc(N, mo["bc"], ids, nuniq).reshape(-1, n3)
    mult = oracle.mult(ids, nuniq).reshape(-1, n3)
    lat = {tuple(p): q for q, p in enumerate(semgen.box_partition(nel, (1, 1, 1), 0))}
    gi = np.array([lat[tuple(p)] for p in elems])
    res = {}
    info = mesh.info()
    res["n_unique"] = (int(info.n_unique), int(nuniq))
    dm, dk = mesh.mult_mask()
    res["mult"] = rel(dm.cpu().numpy(), mult[gi])
    res["mask"] = rel(dk.cpu().numpy(), mask[gi])
    # Ax + dssum (fused) on the same global random field
    ug = semgen.random_field((G.shape[0], n3), 5)
    ref = oracle.ax_dssum(N, G, B, ids, ug, mask=mask, nuniq=nuniq)
    u = torch.from_numpy(np.ascontiguousarray(ug[gi])).cuda()
    w = torch.empty_like(u)
    for _ in range(2):
        mesh.ax_dssum(u, w)
    torch.cuda.synchronize()
    res["ax_dssum"] = rel(w.cpu().numpy(), ref[gi])
    d = torch.from_numpy(np.ascontiguousarray(ug[gi])).cuda()
    mesh.gs_op(d, sem.SEM_GS_ADD)
    res["gs"] = rel(d.cpu().numpy(), oracle.dssum(ids, ug.ravel(), nuniq).reshape(-1, n3)[gi])
    # all copies of a global node identical across ranks: checked by the
    # oracle comparison above at 1e-15; CG next
    fg = semgen.random_field((G.shape[0], n3), 6)
    h1c, h2c = 1.0, (0.5 if not all(per) else 0.0)
    if all(per):
        fg = fg + 0.7  # non-zero mean: the singular projections act
    bo = oracle.dssum(ids, (B * fg).ravel(), nuniq) * mask.ravel()
    if args.solver == "hsmg":  # FGMRES + hybrid-Schwarz multigrid (oracle/hsmg.py)
        from oracle import hsmg as H
        levels = H.setup(N, mo["coords"], mo["bc"], lambda Nl, cl: oracle.lattice_ids(nel, Nl, per))
        xo_, it_o, _, _ = H.fgmres(levels, bo, h1c, h2c, tol=1e-10, maxit=500, restart=20)
        zo = H.vcycle(levels, bo, h1c, h2c)
        mesh.set_options(gmres_precond="hsmg")
    elif args.solver == "gmres":
        xo_, it_o, _, _ = oracle.gmres(N, G, B, ids, bo, mask=mask.ravel(), h1c=h1c, h2c=h2c, tol=1e-10,
                                       maxit=2000, restart=20, nuniq=nuniq)
    else:
        xo_, it_o, _, _ = oracle.pcg(N, G, B, ids, bo, mask=mask.ravel(), h1c=h1c, h2c=h2c, tol=1e-10, maxit=2000,
                                     nuniq=nuniq)
    b = torch.empty_like(u)
    mesh.rhs(torch.from_numpy(np.ascontiguousarray(fg[gi])).cuda(), b)
    if args.solver == "hsmg":  # one V-cycle across the ranks
        z = torch.empty_like(b)
        mesh.hsmg_apply(b, z, h1c=h1c, h2c=h2c)
        res["vcycle"] = rel(z.cpu().numpy(), zo.reshape(-1, n3)[gi])
    xs = []
    for _ in range(args.repeat):
        x = torch.zeros_like(u)
        if args.solver in ("gmres", "hsmg"):
            it, rr, conv = mesh.gmres_solve(b, x, h1c=h1c, h2c=h2c, tol=1e-10, maxit=2000, restart=20)
        else:
            it, rr, conv = mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=1e-10, maxit=2000)
        xs.append(x.cpu().numpy())
    res["cg_x"] = rel(xs[-1], xo_.reshape(-1, n3)[gi])
    res["cg_iters"] = (it, it_o)
    res["repeat_identical"] = all(np.array_equal(xs[0], xk) for xk in xs)
    res["comm_status"] = list(comm.status())
    ok = (res["n_unique"][0] == res["n_unique"][1] and res["mult"] == 0.0 and res["mask"] == 0.0
          and res["ax_dssum"] <= 1e-12 and res["gs"] <= 1e-14 and res["cg_x"] <= 1e-10
          and abs(it - it_o) <= 1 and conv and res["repeat_identical"] and res.get("vcycle", 0.0) <= 1e-10)
    print(json.dumps({"rank": rank, "ok": ok, "args": vars(args), **res}), flush=True)
    mesh.close()
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
