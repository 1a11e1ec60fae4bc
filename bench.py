#!/usr/bin/env python
"""Benchmark of the SEM hot path (arXiv 2405.05640): fixed-iteration
Jacobi-PCG on a Taylor-Green-vortex box, Poisson (pressure) operator.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4] [--iters 100]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference     # the CPU oracle on the same workload

One STEP = one sem_cg_solve(tol = 0, maxit = --iters) over the whole mesh:
Jacobi set-up (R9), r = mask b, and --iters iterations of
[p = dinv r + beta p -> w = mask dssum(A p) -> pAp -> x, r update -> rtr, rtz],
i.e. every row of SURVEY.md 8(a) that runs per solve.  value = Ax+dssum
GDOF/s through the solver = iters * (local DOF over all ranks) / step time;
ms_per_step / iters = pressure-CG ms per iteration (BASELINE.json metric).
Multi-GPU: weak scaling, the per-GPU element block is fixed (c2: 32^3
elements per GPU on a (px,py,pz) process grid).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (elements per GPU per axis, N, description)
    "c2": (32, 7, "tgv-box-32^3-per-gpu-lx8 (BASELINE configs[1]; N GPUs: weak-scaled periodic box)"),
    "c3": (64, 7, "tgv-box-64^3-lx8 (BASELINE configs[2])"),
    "c4": (48, 7, "tgv-box-48^3-per-gpu-lx8 (BASELINE configs[3] weak scaling)"),
}
GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
BYTES_PER_DOF_CG_AX = 88   # fused CG operator: r, dinv, p in; p, w out; G x 6 in
BYTES_PER_DOF_AXDSSUM = 64  # standalone Ax+dssum: u, G x 6 in; w out


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def _mesh_for_rank(cfg, nranks, rank, xi):
    import semgen
    per, N, _ = CONFIGS[cfg]
    grid = GRIDS[nranks] if cfg != "c3" else GRIDS[nranks]
    if cfg == "c3":
        nel = (per, per, per)
    else:
        nel = (per * grid[0], per * grid[1], per * grid[2])
    elems = semgen.box_partition(nel, grid, rank)
    lengths = tuple(2 * math.pi * nel[a] / nel[0] for a in range(3))  # isotropic elements
    m = semgen.box_mesh(nel, xi, lengths=lengths, periodic=(True, True, True), elems=elems)
    return m, nel, N


def run_ours(args):
    import torch
    ws, rank, lrank = _dist_env()
    n = args.gpus
    if ws != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={ws}")
    torch.cuda.set_device(lrank)
    from paper_2405_05640_b200 import sem
    import semgen
    comm = None
    if n > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
        uid = sem.sem_comm_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        comm = sem.sem_comm_create(obj[0], rank, n, lrank)
    per, N, desc = CONFIGS[args.config]
    xi, _ = sem.sem_gll(N)
    m, nel, N = _mesh_for_rank(args.config, n, rank, xi)
    E = m["conn"].shape[0]
    lx = N + 1
    mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"], comm)
    mesh.geom_factors()
    coords = m["coords"]
    f = torch.from_numpy(semgen.tgv_source(coords).reshape(E, lx ** 3)).cuda()
    del m, coords
    b = torch.empty_like(f)
    mesh.rhs(f, b)
    x = torch.zeros_like(f)
    stream = torch.cuda.current_stream()
    iters = args.iters

    def barrier():
        if n > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up
    for _ in range(args.warmup):
        mesh.cg_solve(b, x, tol=0.0, maxit=iters)
    torch.cuda.synchronize()
    mesh.profile_enable(True)
    _, _, kl0 = mesh.profile_get()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(lrank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            it, rr, conv = mesh.cg_solve(b, x, tol=0.0, maxit=iters)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    ax_launches, ax_ms, kl1 = mesh.profile_get()
    mesh.profile_enable(False)
    gpu_launches = kl1 - kl0

    # standalone fused Ax+dssum (the benchmarked operator, 64 B/DOF)
    u = torch.from_numpy(semgen.random_field((E, lx ** 3), 7)).cuda()
    w = torch.empty_like(u)
    for _ in range(3):
        mesh.ax_dssum(u, w)
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = max(10, args.steps)
    e0.record(stream)
    for _ in range(reps):
        mesh.ax_dssum(u, w)
    e1.record(stream)
    torch.cuda.synchronize()
    ax_alone_ms = e0.elapsed_time(e1) / reps

    # end-to-end through the public API with HOST buffers (pinned)
    bh = b.cpu().pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    mesh.cg_solve_host(bh, xh, tol=0.0, maxit=iters)
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 5))
    t0.record(stream)
    for _ in range(e2e_steps):
        mesh.cg_solve_host(bh, xh, tol=0.0, maxit=iters)
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1) / e2e_steps

    nloc = E * lx ** 3
    vals = torch.tensor([ms, ax_ms / max(ax_launches, 1), ax_alone_ms, e2e_ms], dtype=torch.float64,
                        device="cuda")
    if n > 1:
        import torch.distributed as dist
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, ax_avg_ms, ax_alone_ms, e2e_ms = vals.tolist()
    ms_step = ms / args.steps
    dof_total = nloc * n
    value = iters * dof_total / (ms_step * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    achieved = BYTES_PER_DOF_CG_AX * nloc / (ax_avg_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(f"{args.config}_cg_ax")
            if tr:
                traffic = tr
    except Exception:
        pass
    res = None
    if rank == 0:
        cpu = None if (n > 1 or args.no_cpu_baseline) else cpu_baseline(args, budget_s=args.cpu_budget)
        res = {
            "metric": "Ax+dssum fp64 GDOF/s through Jacobi-PCG (pressure, TGV box); CG ms/iter",
            "value": round(value, 3),
            "unit": "GDOF/s",
            "n_gpus": n,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "cg_ms_per_iter": round(ms_step / iters, 5),
            "iters_per_step": iters,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (TGV pressure source on a periodic box, seeded)",
            "config": {"workload": CONFIGS[args.config][2], "elements_global": int(E * n),
                       "elements_per_gpu": int(E), "lx": lx, "dof_local_per_gpu": int(nloc),
                       "process_grid": list(GRIDS[n]), "l2": "inputs larger than L2 (working set "
                       f"{(nloc * 11 * 8) / 1e9:.2f} GB per GPU >> 126 MB)", "solver": "tol=0 fixed iterations"},
            "roofline": {"kernel": "k_ax<8,0,GS,CG> (fused p-update + Ax + dssum + mask + pAp)",
                         "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "bytes_per_dof": BYTES_PER_DOF_CG_AX,
                         "avg_launch_ms": round(ax_avg_ms, 5), "launches_timed": ax_launches},
            "ax_dssum_standalone": {"gdofs": round(nloc / (ax_alone_ms * 1e-3) / 1e9, 3),
                                    "ms": round(ax_alone_ms, 5), "bytes_per_dof": BYTES_PER_DOF_AXDSSUM,
                                    "achieved_gbs": round(BYTES_PER_DOF_AXDSSUM * nloc / (ax_alone_ms * 1e-3) / 1e9, 1),
                                    "frac": round(BYTES_PER_DOF_AXDSSUM * nloc / (ax_alone_ms * 1e-3) / 1e9 / peak, 4)},
            "e2e": {"value": round(iters * dof_total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GDOF/s",
                    "h2d_bytes_per_step": int(nloc * 8), "d2h_bytes_per_step": int(nloc * 8),
                    "ms_per_step": round(e2e_ms, 4)},
            "gpu_launches": int(gpu_launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(res), flush=True)
    mesh.close()
    if comm is not None:
        comm.close()
    if n > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return res


def _oracle_setup(cfg, max_elems=None):
    """Oracle-side mesh for the CPU legs (its own GLL, geometry, numbering)."""
    import oracle
    import semgen
    per, N, _ = CONFIGS[cfg]
    nel = (per, per, per)
    xo, _ = oracle.gll(N)
    m = semgen.box_mesh(nel, xo, periodic=(True, True, True))
    G, B = oracle.geom(N, m["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, (True, True, True))
    f = semgen.tgv_source(m["coords"]).reshape(G.shape[0], -1)
    b = oracle.dssum(ids, (B * f).ravel(), nuniq)
    dinv = oracle.jacobi(N, G, B, ids, None, nuniq=nuniq)
    return N, G, B, ids, nuniq, b, dinv


def cpu_baseline(args, budget_s=20.0):
    """The oracle (as it stands) on the host cores: PCG iterations of the same
    workload (full mesh of --config at N=1), set-up excluded."""
    import oracle
    t0 = time.time()
    N, G, B, ids, nuniq, b, dinv = _oracle_setup(args.config)
    setup_s = time.time() - t0
    E = G.shape[0]
    nloc = E * (N + 1) ** 3
    k = 2
    t0 = time.time()
    oracle.pcg(N, G, B, ids, b, tol=0.0, maxit=k, nuniq=nuniq, dinv=dinv)
    dt = time.time() - t0
    cores = len(os.sched_getaffinity(0))
    return {"value": round(k * nloc / dt / 1e9, 4), "unit": "GDOF/s", "cores": cores, "kind": "oracle",
            "ms_per_iter": round(dt / k * 1e3, 2),
            "sample": f"{k} oracle PCG iterations (tol=0) on the full {args.config} mesh "
                      f"({E} elements, {nloc} local DOF), set-up ({setup_s:.1f} s) excluded; "
                      f"OpenMP threads = {os.environ.get('OMP_NUM_THREADS', cores)}"}


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return None
    import oracle
    N, G, B, ids, nuniq, b, dinv = _oracle_setup(args.config)
    E = G.shape[0]
    nloc = E * (N + 1) ** 3
    # each step: one PCG iteration of the full mesh (bounded sample of the
    # 100-iteration GPU step); warm-up untimed
    for _ in range(args.warmup):
        oracle.pcg(N, G, B, ids, b, tol=0.0, maxit=1, nuniq=nuniq, dinv=dinv)
    t0 = time.time()
    for _ in range(args.steps):
        oracle.pcg(N, G, B, ids, b, tol=0.0, maxit=1, nuniq=nuniq, dinv=dinv)
    dt = time.time() - t0
    ms_step = dt / args.steps * 1e3
    value = nloc / (ms_step * 1e-3) / 1e9
    cores = len(os.sched_getaffinity(0))
    res = {
        "impl": "reference",
        "metric": "Ax+dssum fp64 GDOF/s through Jacobi-PCG (pressure, TGV box); CG ms/iter",
        "value": round(value, 4), "unit": "GDOF/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "cg_ms_per_iter": round(ms_step, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (TGV pressure source on a periodic box, seeded)",
        "config": {"workload": CONFIGS[args.config][2], "elements_global": int(E), "lx": N + 1},
        "cpu_baseline": {"kind": "oracle", "cores": cores, "value": round(value, 4), "unit": "GDOF/s",
                         "sample": f"each step = 1 oracle PCG iteration of the full {args.config} mesh "
                                   f"({nloc} local DOF); set-up excluded"},
        "e2e": {"value": round(value, 4), "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res), flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
