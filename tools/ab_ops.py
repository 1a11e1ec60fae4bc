"""A/B timing (CUDA events, not under ncu) of the operator, the gather-scatter
pass, Ax+dssum and 100 PCG iterations on a periodic box, for option
combinations (sem_mesh_set_options).  Developer tool.
usage: python tools/ab_ops.py [per] [N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch  # noqa: E402

import semgen  # noqa: E402
from paper_2405_05640_b200 import sem  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 7
xi, _ = sem.sem_gll(N)
m = semgen.box_mesh((per, per, per), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
u = torch.from_numpy(semgen.random_field((E, (N + 1) ** 3), 1)).cuda()
w = torch.empty_like(u)


def t(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps * 1e3, 1)


b = torch.empty_like(u)
mesh.rhs(u, b)
x = torch.zeros_like(u)
OPTS = ({"graph": 1}, {"graph": 1, "cg_layout": 0}, {"graph": 1, "pdl": 1}, {"graph": 0}, {"graph": 0, "pdl": 1},
        {"graph": 1, "cg_variant": "pipelined"}, {"graph": 1, "affine": 1})
for opts in (OPTS[:2] if os.environ.get("AB_QUICK") else OPTS):
    mesh.set_options(cg_variant="standard", affine=0, pdl=0, cg_layout=1)
    mesh.set_options(**opts)
    res = dict(opts, ax_us=t(lambda: mesh.ax(u, w)), gs_us=t(lambda: mesh.gs_op(w)),
               ax_dssum_us=t(lambda: mesh.ax_dssum(u, w)),
               cg_ms_per_iter=round(t(lambda: mesh.cg_solve(b, x, tol=0.0, maxit=100), reps=3) / 1e5, 4))
    print(json.dumps(res), flush=True)
