"""Interleaved A/B of the PCG iteration time over option sets on one mesh
(CUDA events; each round runs every option set once, in rotating order, so
clock drift spreads evenly).  Developer tool.
usage: python tools/ab_cg.py '{"cg_layout":1}' '{"cg_layout":0}' [...]
env: PER (32), NORD (7), ROUNDS (6), ITERS (100)"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
import torch  # noqa: E402

import semgen  # noqa: E402
from paper_2405_05640_b200 import sem  # noqa: E402

per = int(os.environ.get("PER", "32"))
N = int(os.environ.get("NORD", "7"))
rounds = int(os.environ.get("ROUNDS", "6"))
iters = int(os.environ.get("ITERS", "100"))
opts = [json.loads(a) for a in sys.argv[1:]] or [{}]
xi, _ = sem.sem_gll(N)
m = semgen.box_mesh((per, per, per), xi)
E = m["conn"].shape[0]
mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"])
mesh.geom_factors()
base = mesh.options()
f = torch.from_numpy(semgen.tgv_source(m["coords"]).reshape(E, -1)).cuda()
b = torch.empty_like(f)
mesh.rhs(f, b)
x = torch.zeros_like(f)
times = [[] for _ in opts]
for r in range(rounds + 1):
    order = list(range(len(opts)))
    order = order[r % len(opts):] + order[:r % len(opts)]
    for k in order:
        mesh.set_options(base)
        mesh.set_options(**opts[k])
        mesh.cg_solve(b, x, tol=0.0, maxit=iters)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        mesh.cg_solve(b, x, tol=0.0, maxit=iters)
        a1.record()
        torch.cuda.synchronize()
        if r > 0:
            times[k].append(a0.elapsed_time(a1) / iters)
for k, o in enumerate(opts):
    print(json.dumps({"opts": o, "ms_per_iter_median": round(statistics.median(times[k]), 5),
                      "min": round(min(times[k]), 5), "max": round(max(times[k]), 5)}))
