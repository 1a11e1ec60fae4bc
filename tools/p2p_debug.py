"""Debug: distributed ax_dssum repeated, error per call on each rank."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, torch.distributed as dist
import oracle, semgen
from paper_2405_05640_b200 import sem
from mgpu_worker import CASES, rel
case = CASES[sys.argv[1]]
rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
uid = [sem.sem_comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = sem.sem_comm_create(uid[0], rank, ws, rank)
nel, N, per, grid = case["nel"], case["N"], case["periodic"], case["grid"]
n3 = (N + 1) ** 3
elems = semgen.box_partition(nel, grid, rank)
xl, _ = sem.sem_gll(N)
ml = semgen.box_mesh(nel, xl, periodic=per, deform=case["deform"], elems=elems)
mesh = sem.Mesh(len(elems), N, ml["coords"], ml["conn"], ml["bc"], comm)
mesh.geom_factors()
xo, _ = oracle.gll(N)
mo = semgen.box_mesh(nel, xo, periodic=per, deform=case["deform"])
G, B = oracle.geom(N, mo["coords"])
ids, nuniq = oracle.lattice_ids(nel, N, per)
mask = oracle.mask_from_bc(N, mo["bc"], ids, nuniq).reshape(-1, n3)
lat = {tuple(p): q for q, p in enumerate(semgen.box_partition(nel, (1, 1, 1), 0))}
gi = np.array([lat[tuple(p)] for p in elems])
ug = semgen.random_field((G.shape[0], n3), 5)
ref = oracle.ax_dssum(N, G, B, ids, ug, mask=mask, nuniq=nuniq)[gi]
u = torch.from_numpy(np.ascontiguousarray(ug[gi])).cuda()
w = torch.empty_like(u)
out = []
for k in range(4):
    if os.environ.get("SYNC"): dist.barrier(); torch.cuda.synchronize()
    mesh.ax_dssum(u, w)
    torch.cuda.synchronize()
    d = np.abs(w.cpu().numpy() - ref)
    bad = np.argwhere(d > 1e-9 * np.abs(ref).max())
    out.append((k, rel(w.cpu().numpy(), ref), len(bad), bad[:3].tolist()))
print(json.dumps({"rank": rank, "info": [int(mesh.info().n_peers)], "calls": out}), flush=True)
mesh.close(); comm.close()
