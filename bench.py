#!/usr/bin/env python
"""Benchmark of the SEM hot path (arXiv 2405.05640): fixed-iteration
Jacobi-PCG through the C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5] [--iters 100]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference     # the CPU oracle on the same workload

One STEP = one sem_cg_solve(tol = 0, maxit = --iters) over the whole mesh:
Jacobi set-up (R9), r = mask b, and --iters iterations of
[p = dinv r + beta p -> w = mask dssum(A p) -> pAp -> x, r update -> rtr, rtz],
i.e. every row of SURVEY.md 8(a) that runs per solve.  value = Ax+dssum
GDOF/s through the solver = iters * (local DOF over all ranks) / step time;
ms_per_step / iters = CG ms per iteration (BASELINE.json metric).

Configs (BASELINE.json configs[1..4]):
  c2  TGV pressure (Poisson), periodic box 32^3 elements per GPU, lx = 8
      (N GPUs: weak scaling on a (2,1,1)/(2,2,1)/(2,2,2) process grid)  [default]
  c3  TGV pressure, 64^3 elements global (strong scaling), lx = 8
  c4  TGV pressure, 48^3 elements per GPU (weak scaling), lx = 8
  c5  RBC-like O-grid cylinder, lx = 10, 393,216 elements global (axial
      slabs over GPUs), velocity Helmholtz h1 = sqrt(Pr/Ra), h2 = (11/6)/dt
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
    "c2": "tgv-box-32^3-per-gpu-lx8 (BASELINE configs[1]; N GPUs: weak-scaled periodic box)",
    "c3": "tgv-box-64^3-lx8 (BASELINE configs[2]; N GPUs: strong scaling)",
    "c4": "tgv-box-48^3-per-gpu-lx8 (BASELINE configs[3]; weak scaling)",
    "c5": "rbc-cylinder-ogrid-lx10-393216el (BASELINE configs[4]; Helmholtz velocity solve, axial slabs)",
}
GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
H1_C5 = math.sqrt(1.0 / 1e11)        # sqrt(Pr/Ra), Ra = 1e11, Pr = 1
H2_C5 = (11.0 / 6.0) / 1e-3          # BDF3 coefficient / dt (dt proposed)


def _bytes_per_dof(helmholtz, affine=False):
    """Algorithmic bytes per local DOF (
    no gather-scatter surcharge: a fused dssum moves no mandatory HBM bytes,
    so gs traffic LOWERS the fraction): the fused CG operator, the standalone
    Ax+dssum, and one whole CG iteration (x update deferred into the
    operator: 136 instead of SURVEY's 152)."""
    hb = 8 if helmholtz else 0
    g = 0 if affine else 48  # affine variant: 6 constants per element instead of G per node
    cg_op = 56 + g + hb   # G x 6, r, dinv, p, x in; p, x, w out (+ B)
    axd = 16 + g + hb     # u, G x 6 (+ B) in; w out
    cg_iter = cg_op + 32  # + the update pass: r, w, dinv in; r out
    return cg_op, axd, cg_iter


NOMINAL_HBM_GBS = 8000.0  # BASELINE.json north star "~8 TB/s"


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

    def __init__(self, devices, active=True):
        # one sampler (rank 0) queries every GPU of the job: fewer process
        # spawns competing with the ranks' launch threads
        self.devs = ",".join(str(d) for d in devices)
        self.active = active
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", self.devs, f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                for line in out.splitlines():
                    if line.strip():
                        self.samples.append([s.strip() for s in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.active:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
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


def problem(cfg, nranks, rank, xi, reduced=False):
    """Mesh block of `rank`, its source f and coefficients.  `reduced`: a
    bounded sample of the same workload for the CPU oracle legs."""
    import semgen
    if cfg == "c5":
        nz = 128
        layers = semgen.cylinder_partition(nz, nranks, rank)
        if reduced:
            layers = (0, 2)
        m = semgen.cylinder_mesh(xi, nc=32, nr=16, nz=nz, layers=layers)
        E = m["conn"].shape[0]
        f = semgen.cyl_source(m["coords"], h1=H1_C5, h2=H2_C5).reshape(E, -1)
        return dict(mesh=m, N=9, h1c=H1_C5, h2c=H2_C5, f=f, scaling="strong", grid=(1, 1, nranks),
                    periods=(None, None, None), nel=None)
    per = {"c2": 32, "c3": 64, "c4": 48}[cfg]
    grid = GRIDS[nranks]
    if cfg == "c3":
        nel, scaling = (per, per, per), "strong"
    else:
        nel, scaling = (per * grid[0], per * grid[1], per * grid[2]), "weak"
    if reduced:
        nel, grid, rank = (per, per, per), (1, 1, 1), 0
    elems = semgen.box_partition(nel, grid, rank)
    lengths = tuple(2 * math.pi * nel[a] / nel[0] for a in range(3))  # isotropic elements
    m = semgen.box_mesh(nel, xi, lengths=lengths, periodic=(True, True, True), elems=elems)
    E = m["conn"].shape[0]
    f = semgen.tgv_source(m["coords"]).reshape(E, -1)
    return dict(mesh=m, N=7, h1c=1.0, h2c=0.0, f=f, scaling=scaling, grid=grid, periods=m["periods"], nel=nel)


def _bind_near_gpu(dev):
    """Bind this process's thread to the host cores NVML reports as local to
    GPU `dev` (the e2e leg's pinned host buffers are then first-touched on
    the GPU's NUMA node).  Returns (cores now, cores before) or None."""
    import torch
    try:
        import pynvml
        before = sorted(os.sched_getaffinity(0))
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(dev).uuid))
        pynvml.nvmlDeviceSetCpuAffinity(h)
        return sorted(os.sched_getaffinity(0)), before
    except Exception:
        return None


def run_ours(args):
    import torch
    ws, rank, lrank = _dist_env()
    n = args.gpus
    if ws != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={ws}")
    torch.cuda.set_device(lrank)
    binding = _bind_near_gpu(lrank)
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
    N0 = 9 if args.config == "c5" else 7
    xi, _ = sem.sem_gll(N0)
    pb = problem(args.config, n, rank, xi)
    m, N = pb["mesh"], pb["N"]
    h1c, h2c = pb["h1c"], pb["h2c"]
    helm = h2c != 0.0
    E = m["conn"].shape[0]
    lx = N + 1
    mesh = sem.Mesh(E, N, m["coords"], m["conn"], m["bc"], comm)
    mesh.geom_factors()
    mesh.set_options(affine=int(args.affine), graph=int(not args.no_graph),
                     cg_variant="pipelined" if args.pipelined else "standard")
    f = torch.from_numpy(np.ascontiguousarray(pb["f"])).cuda()
    pb_coords = m["coords"] if (n == 1 and args.config in ("c2", "c3", "c4")) else None
    del m, pb
    b = torch.empty_like(f)
    mesh.rhs(f, b)
    x = torch.zeros_like(f)
    stream = torch.cuda.current_stream()
    iters = args.iters

    def barrier():
        if n > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=0.0, maxit=iters)
    torch.cuda.synchronize()
    # the timed region: the production path (the whole CG loop is one CUDA
    # graph with a conditional WHILE node; no profiling events)
    _, _, kl0 = mesh.profile_get()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev_step = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(range(n), active=(rank == 0)) as clk:
        ev0.record(stream)
        for s_ in range(args.steps):
            mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=0.0, maxit=iters)
            ev_step[s_].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    step_ms = [ev0.elapsed_time(ev_step[0])] + [ev_step[q - 1].elapsed_time(ev_step[q]) for q in range(1, args.steps)]
    _, _, kl1 = mesh.profile_get()
    gpu_launches = kl1 - kl0
    # the roofline's kernel timing: CUDA events around every operator launch
    # on its stream, in a profiled pass of the same steps right after (the
    # events need one graph launch per iteration, which would slow the
    # headline region)
    prof_steps = max(2, min(args.steps, 5))
    mesh.profile_enable(True)
    barrier()
    torch.cuda.synchronize()
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(prof_steps):
        mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=0.0, maxit=iters)
    pe1.record(stream)
    torch.cuda.synchronize()
    prof_ms_step = pe0.elapsed_time(pe1) / prof_steps
    ax_launches, ax_ms, _ = mesh.profile_get()
    mesh.profile_enable(False)

    # standalone fused Ax+dssum (the benchmarked operator)
    u = torch.from_numpy(semgen.random_field((E, lx ** 3), 7)).cuda()
    w = torch.empty_like(u)
    for _ in range(3):
        mesh.ax_dssum(u, w, h1c=h1c, h2c=h2c)
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = max(10, args.steps)
    e0.record(stream)
    for _ in range(reps):
        mesh.ax_dssum(u, w, h1c=h1c, h2c=h2c)
    e1.record(stream)
    torch.cuda.synchronize()
    ax_alone_ms = e0.elapsed_time(e1) / reps

    # end-to-end through the public API with HOST buffers (pinned)
    bh = b.cpu().pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    mesh.cg_solve_host(bh, xh, h1c=h1c, h2c=h2c, tol=0.0, maxit=iters)
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 5))
    t0.record(stream)
    for _ in range(e2e_steps):
        mesh.cg_solve_host(bh, xh, h1c=h1c, h2c=h2c, tol=0.0, maxit=iters)
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1) / e2e_steps

    # restarted GMRES on the same system: ms per Arnoldi step
    # (tol = 0: exactly 2 cycles of restart 30), one GPU, box configs only
    # (the basis is 31 vectors of the local size)
    gmres = None
    if n == 1 and args.config in ("c2", "c4") and not args.no_gmres:
        def _timed_gmres(pc, tol, maxit, restart=30):
            mesh.set_options(gmres_precond=pc)
            mesh.gmres_solve(b, x, h1c=h1c, h2c=h2c, tol=tol, maxit=min(maxit, 60), restart=restart)  # warm-up
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            it_g, rr_g, conv_g = mesh.gmres_solve(b, x, h1c=h1c, h2c=h2c, tol=tol, maxit=maxit, restart=restart)
            g1.record(stream)
            torch.cuda.synchronize()
            return it_g, rr_g, conv_g, g0.elapsed_time(g1)
        steps_g, restart_g = 60, 30
        it_g, rr_g, _, gms = _timed_gmres("jacobi", 0.0, steps_g)
        gmres = {"restart": restart_g, "arnoldi_steps": it_g, "ms_per_step": round(gms / it_g, 5),
                 "gdofs": round(it_g * E * lx ** 3 / (gms * 1e-3) / 1e9, 3), "rel_res": rr_g,
                 "what": "sem_gmres_solve, right Jacobi preconditioning, CGS2 Arnoldi (TMA-staged vector passes); "
                         "the set-up (Jacobi) included"}
        # the paper's pressure solver: FGMRES + hybrid-Schwarz
        # multigrid, time to a 1e-8 residual, against Jacobi-GMRES and
        # Jacobi-PCG on the same system
        if h2c == 0.0:
            tol_s = 1e-8
            it_h, rr_h, cv_h, ms_h = _timed_gmres("hsmg", tol_s, 500)
            it_j, rr_j, cv_j, ms_j = _timed_gmres("jacobi", tol_s, 5000)
            mesh.set_options(gmres_precond="jacobi")
            c0 = torch.cuda.Event(enable_timing=True)
            c1 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            it_c, rr_c, cv_c = mesh.cg_solve(b, x, h1c=h1c, h2c=h2c, tol=tol_s, maxit=20000)
            c1.record(stream)
            torch.cuda.synchronize()
            gmres["time_to_solution"] = {
                "tol": tol_s,
                "fgmres_hsmg": {"steps": it_h, "ms": round(ms_h, 3), "ms_per_step": round(ms_h / max(it_h, 1), 4),
                                "converged": cv_h, "coarse_iters": mesh.options().hsmg_coarse_iters},
                "gmres_jacobi": {"steps": it_j, "ms": round(ms_j, 3), "converged": cv_j},
                "pcg_jacobi": {"iterations": it_c, "ms": round(c0.elapsed_time(c1), 3), "converged": cv_c},
                "what": "the set-up (levels built on the first call, outside) excluded; Jacobi set-up included"}
    # one velocity-pressure splitting time step (the paper's
    # "time per time step") from the 3D Taylor-Green field of
    # PAPER.md:96 on the same periodic box: ms per step, the solves at 1e-8
    pnpn = None
    if n == 1 and args.config in ("c2", "c3", "c4") and not args.no_pnpn:
        xg = torch.from_numpy(np.ascontiguousarray(semgen.tgv_velocity(pb_coords).reshape(3, E, lx ** 3))).cuda()
        pp = torch.zeros_like(b)
        dt_, nu_ = 1e-3, 1.0 / 1600.0  # Re = 1600
        mesh.pnpn_step(xg, pp, dt_, nu_, tol=1e-8, maxit=2000)
        xg.copy_(torch.from_numpy(np.ascontiguousarray(semgen.tgv_velocity(pb_coords).reshape(3, E, lx ** 3))))
        pp.zero_()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        nsteps = 3
        its_all = []
        q0.record(stream)
        for _ in range(nsteps):
            its_all.append(mesh.pnpn_step(xg, pp, dt_, nu_, tol=1e-8, maxit=2000))
        q1.record(stream)
        torch.cuda.synchronize()
        pnpn = {"ms_per_step": round(q0.elapsed_time(q1) / nsteps, 3), "steps": nsteps, "dt": dt_, "Re": 1600,
                "iterations_per_step": its_all[-1],
                "what": "sem_pnpn_step: BDF1/EXT1 splitting, convection + pressure PCG + 3 velocity Helmholtz PCG "
                        "to tol 1e-8, 3D TGV initial field"}
        # the paper's solver configuration: pressure by FGMRES +
        # hybrid-Schwarz multigrid, velocity by Jacobi-PCG
        xg.copy_(torch.from_numpy(np.ascontiguousarray(semgen.tgv_velocity(pb_coords).reshape(3, E, lx ** 3))))
        pp.zero_()
        mesh.set_options(pnpn_pressure="gmres", gmres_precond="hsmg")
        # warm-up: the same steps from the same state (every Arnoldi step graph
        # the timed steps replay is captured here), then the state is reset
        for _ in range(nsteps):
            mesh.pnpn_step(xg, pp, dt_, nu_, tol=1e-8, maxit=2000)
        xg.copy_(torch.from_numpy(np.ascontiguousarray(semgen.tgv_velocity(pb_coords).reshape(3, E, lx ** 3))))
        pp.zero_()
        torch.cuda.synchronize()
        its_h = []
        q0.record(stream)
        for _ in range(nsteps):
            its_h.append(mesh.pnpn_step(xg, pp, dt_, nu_, tol=1e-8, maxit=2000))
        q1.record(stream)
        torch.cuda.synchronize()
        mesh.set_options(pnpn_pressure="cg", gmres_precond="jacobi")
        pnpn["papers_solvers"] = {"ms_per_step": round(q0.elapsed_time(q1) / nsteps, 3),
                                  "iterations_per_step": its_h[-1],
                                  "what": "pressure: FGMRES(30) + hybrid-Schwarz multigrid V-cycle; velocity: "
                                          "Jacobi-PCG (PAPER.md:72)"}
        del xg, pp
    nloc = E * lx ** 3
    info = mesh.info()
    vals = torch.tensor([ms, ax_ms / max(ax_launches, 1), ax_alone_ms, e2e_ms], dtype=torch.float64,
                        device="cuda")
    tots = torch.tensor([nloc, gpu_launches], dtype=torch.float64, device="cuda")
    if n > 1:
        import torch.distributed as dist
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(tots, op=dist.ReduceOp.SUM)
    ms, ax_avg_ms, ax_alone_ms, e2e_ms = vals.tolist()
    st = torch.tensor(step_ms, dtype=torch.float64, device="cuda")
    if n > 1:
        import torch.distributed as dist
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
    st = st.tolist()
    step_stats = {"median_ms": round(statistics.median(st), 4), "mean_ms": round(statistics.mean(st), 4),
                  "ci95_ms": round(1.96 * statistics.stdev(st) / math.sqrt(len(st)), 4) if len(st) > 1 else None,
                  "n": len(st), "what": "per-step device time (max over ranks per step)"}
    dof_total = int(tots[0].item())
    ms_step = ms / args.steps
    value = iters * dof_total / (ms_step * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    b_cg, b_axd, b_it = _bytes_per_dof(helm, bool(info.affine))
    achieved = b_cg * nloc / (ax_avg_ms * 1e-3) / 1e9
    traffic = traffic_ratio = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(args.config)
        if tr and n == 1:
            traffic = int(tr["bytes_per_launch"])
            traffic_ratio = round(traffic / (b_cg * nloc), 3)
    except Exception:
        pass
    kname = ("fused CG operator: k_ax<CG> (deferred x update + p update + Ax + pAp partials), then the nodal "
             "gather-scatter k_gs_nodal (mask . dssum, pAp reduced in its last block)")
    res = None
    if rank == 0:
        if binding:  # the CPU legs use every host core again
            os.sched_setaffinity(0, binding[1])
        cpu = None if (n > 1 or args.no_cpu_baseline) else cpu_baseline(args.config)
        res = {
            "metric": "Ax+dssum fp64 GDOF/s through Jacobi-PCG; CG ms/iter",
            "value": round(value, 3),
            "unit": "GDOF/s",
            "n_gpus": n,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "cg_ms_per_iter": round(ms_step / iters, 5),
            "step_stats": step_stats,
            "iters_per_step": iters,
            "higher_is_better": True,
            "scaling": "strong" if args.config in ("c3", "c5") else "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded mesh and manufactured source; no datasets)",
            "config": {"workload": CONFIGS[args.config], "elements_global": int(info.E) * n if args.config in ("c2", "c4") else None,
                       "elements_per_gpu": int(E), "lx": lx, "dof_local_total": dof_total,
                       "unique_dof_global": int(info.n_unique), "operator": "helmholtz" if helm else "poisson",
                       "n_peers": int(info.n_peers),
                       "l2": "inputs larger than L2 (working set "
                             f"{(nloc * 12 * 8) / 1e9:.2f} GB per GPU >> 126 MB)",
                       "solver": "tol=0 fixed iterations, Jacobi-PCG",
                       "host_binding": (f"{len(binding[0])} host cores NVML reports local to the GPU (pinned e2e "
                                        f"buffers on its NUMA node)" if binding else "none")},
            "roofline": {"kernel": kname,
                         "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind + " (MEASURED_PEAKS.json hbm_gbs, copy burst)", "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "frac_vs_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                         "traffic": traffic, "traffic_over_algorithmic": traffic_ratio,
                         "bytes_per_dof": b_cg, "bytes_per_dof_source": "SURVEY 8(d), no gs surcharge",
                         "avg_launch_ms": round(ax_avg_ms, 5), "launches_timed": ax_launches,
                         "timing": f"CUDA events around every operator launch on its stream, over a profiled pass "
                                   f"of {prof_steps} steps right after the timed region ({round(prof_ms_step, 3)} "
                                   f"ms per step with the events)"},
            "cg_iteration": {"bytes_per_dof": b_it, "ms": round(ms_step / iters, 5),
                             "achieved_gbs": round(b_it * nloc / (ms_step / iters * 1e-3) / 1e9, 1),
                             "frac": round(b_it * nloc / (ms_step / iters * 1e-3) / 1e9 / peak, 4),
                             "frac_vs_8tbs": round(b_it * nloc / (ms_step / iters * 1e-3) / 1e9 / NOMINAL_HBM_GBS, 4)},
            "ax_dssum_standalone": {"gdofs": round(nloc / (ax_alone_ms * 1e-3) / 1e9, 3),
                                    "ms": round(ax_alone_ms, 5), "bytes_per_dof": b_axd,
                                    "achieved_gbs": round(b_axd * nloc / (ax_alone_ms * 1e-3) / 1e9, 1),
                                    "frac": round(b_axd * nloc / (ax_alone_ms * 1e-3) / 1e9 / peak, 4),
                                    "frac_vs_8tbs": round(b_axd * nloc / (ax_alone_ms * 1e-3) / 1e9 / NOMINAL_HBM_GBS, 4),
                                    "target_gdofs_70pct_of_8tbs": round(0.7 * NOMINAL_HBM_GBS / b_axd, 2)},
            "e2e": {"value": round(iters * dof_total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GDOF/s",
                    "h2d_bytes_per_step": int(nloc * 8), "d2h_bytes_per_step": int(nloc * 8),
                    "ms_per_step": round(e2e_ms, 4)},
            "gpu_launches": int(tots[1].item()),
            "gmres": gmres,
            "pnpn_step": pnpn,
            "variant": ("affine elements: 6 metric constants per element instead of G per node "
                        "(SURVEY 8(f) f3; bytes_per_dof without G)" if info.affine else "general (G per node)")
                       + ("; single-reduction PCG (SURVEY 8(f) f1)" if args.pipelined else ""),
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


def _oracle_setup(cfg, full=False):
    """Oracle-side problem for the CPU legs (its own GLL, geometry and
    numbering); unless full, c3/c5 use a bounded sample (c3: the 32^3 box,
    c5: two axial layers of the cylinder)."""
    import oracle
    N0 = 9 if cfg == "c5" else 7
    xo, _ = oracle.gll(N0)
    reduced = cfg in ("c3", "c5") and not full
    pb = problem("c2" if (cfg == "c3" and reduced) else cfg, 1, 0, xo, reduced=(cfg == "c5" and reduced))
    m, N = pb["mesh"], pb["N"]
    G, B = oracle.geom(N, m["coords"])
    if pb["nel"] is not None:
        ids, nuniq = oracle.lattice_ids(pb["nel"], N, (True, True, True))
    else:
        ids, nuniq = oracle.geometric_ids(m["coords"], tol=1e-9)
    mask = oracle.mask_from_bc(N, m["bc"], ids, nuniq)
    b = oracle.dssum(ids, (B * pb["f"]).ravel(), nuniq) * mask
    dinv = oracle.jacobi(N, G, B, ids, mask, h1c=pb["h1c"], h2c=pb["h2c"], nuniq=nuniq)
    desc = ("c2 32^3 box (bounded sample of c3)" if (cfg == "c3" and reduced) else
            "2 of 128 axial layers of the c5 cylinder" if (cfg == "c5" and reduced) else f"the full {cfg} mesh")
    return N, G, B, ids, nuniq, b, dinv, mask, pb["h1c"], pb["h2c"], desc, reduced


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _median_time(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def cpu_leg(cfg, what):
    """One group of oracle legs on the host cores (run in a subprocess by
    cpu_baseline, so the GPU bench process never loads the oracle):
    'ax' = Ax+dssum single application (median of 3), 'cg:K' = K PCG
    iterations (tol = 0), 'cgfull' = PCG to tol 1e-12 (C1's manufactured
    problem).  Set-up (geometry, numbering, Jacobi) is excluded."""
    import oracle
    t0 = time.time()
    if cfg == "c1":
        xo, _ = oracle.gll(7)
        import semgen
        m = semgen.box_mesh((4, 4, 4), xo)
        N = 7
        G, B = oracle.geom(N, m["coords"])
        ids, nuniq = oracle.lattice_ids((4, 4, 4), N, (True,) * 3)
        mask = oracle.mask_from_bc(N, m["bc"], ids, nuniq)
        f = semgen.sin3_source(m["coords"])
        b = oracle.dssum(ids, (B * f).ravel(), nuniq)
        dinv = oracle.jacobi(N, G, B, ids, mask, nuniq=nuniq)
        h1c, h2c, desc = 1.0, 0.0, "C1 periodic 4^3 box, lx = 8, manufactured sin"
    else:
        N, G, B, ids, nuniq, b, dinv, mask, h1c, h2c, desc, _ = _oracle_setup(cfg, full=(what == "ax"))
    setup_s = time.time() - t0
    E = G.shape[0]
    nloc = E * (N + 1) ** 3
    out = {"config": cfg, "desc": desc, "local_dof": int(nloc), "setup_s": round(setup_s, 1),
           "threads": int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))}
    if what == "ax":
        u = np.random.default_rng(7).uniform(-1, 1, (E, (N + 1) ** 3))
        dt = _median_time(lambda: oracle.ax_dssum(N, G, B, ids, u, mask=mask, h1c=h1c, h2c=h2c, nuniq=nuniq), 3)
        out.update(leg="Ax+dssum single application (median of 3)", s=round(dt, 4),
                   gdofs=round(nloc / dt / 1e9, 5))
    elif what.startswith("cg:"):
        k = int(what[3:])
        t1 = time.perf_counter()
        oracle.pcg(N, G, B, ids, b, mask=mask, h1c=h1c, h2c=h2c, tol=0.0, maxit=k, nuniq=nuniq, dinv=dinv)
        dt = time.perf_counter() - t1
        out.update(leg=f"{k} PCG iterations (tol = 0)", s=round(dt, 4), ms_per_iter=round(dt / k * 1e3, 2),
                   gdofs=round(k * nloc / dt / 1e9, 5))
    elif what == "cgfull":
        t1 = time.perf_counter()
        _, it, rr, conv = oracle.pcg(N, G, B, ids, b, mask=mask, h1c=h1c, h2c=h2c, tol=1e-12, maxit=3000,
                                     nuniq=nuniq, dinv=dinv)
        dt = time.perf_counter() - t1
        out.update(leg="PCG to tol 1e-12", s=round(dt, 4), iters=int(it), converged=bool(conv),
                   ms_per_iter=round(dt / max(it, 1) * 1e3, 2), gdofs=round(it * nloc / dt / 1e9, 5))
    return out


# (config, leg, threads: "all" | 1): the default set finishes in ~1-2 min of
# host time; --cpu-legs all adds the full-size C3/C5 Ax+dssum legs
CPU_LEGS_DEFAULT = [("c1", "cgfull", "all"), ("c1", "ax", "all"), ("c2", "cg:10", "all"), ("c2", "ax", "all"),
                    ("c2", "ax", 1)]
CPU_LEGS_ALL = CPU_LEGS_DEFAULT + [("c3", "ax", "all"), ("c5", "ax", "all")]


def cpu_baseline(cfg, legs=None):
    """The oracle, as it stands, on the box's host cores (SURVEY 8(d) "Oracle
    timing"): each leg group in its own subprocess (OMP_NUM_THREADS = the
    affinity count, or 1).  value = PCG GDOF/s of the configuration's own
    workload (c2: 10 iterations on the full mesh; c3/c5: a bounded sample)."""
    cores = len(os.sched_getaffinity(0))
    legs = list(legs or CPU_LEGS_DEFAULT)
    main_leg = (cfg, "cg:10" if cfg in ("c2", "c4") else "cg:2", "all")
    if main_leg not in legs:
        legs.append(main_leg)
    results = []
    for c, what, th in legs:
        env = dict(os.environ, OMP_NUM_THREADS=str(cores if th == "all" else th))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--cpu-leg", f"{c}:{what}"],
                           capture_output=True, text=True, env=env, timeout=3600)
        try:
            results.append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            results.append({"config": c, "leg": what, "error": (r.stderr or r.stdout)[-300:]})
    main = next((x for x in results if x.get("config") == cfg and x.get("leg", "").startswith(
        main_leg[1][3:] + " PCG")), None)
    value = main["gdofs"] if main and "gdofs" in main else None
    return {"value": value, "unit": "GDOF/s", "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": (f"{main['leg']} on {main['desc']} ({main['local_dof']} local DOF), set-up excluded, "
                       f"{main['threads']} OpenMP threads" if main else "unavailable"),
            "legs": results}


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return None
    import oracle
    N, G, B, ids, nuniq, b, dinv, mask, h1c, h2c, desc, _ = _oracle_setup(args.config)
    E = G.shape[0]
    nloc = E * (N + 1) ** 3
    # each step: one PCG iteration (a bounded sample of the GPU step's
    # --iters iterations); warm-up untimed
    for _ in range(args.warmup):
        oracle.pcg(N, G, B, ids, b, mask=mask, h1c=h1c, h2c=h2c, tol=0.0, maxit=1, nuniq=nuniq, dinv=dinv)
    t0 = time.time()
    for _ in range(args.steps):
        oracle.pcg(N, G, B, ids, b, mask=mask, h1c=h1c, h2c=h2c, tol=0.0, maxit=1, nuniq=nuniq, dinv=dinv)
    dt = time.time() - t0
    ms_step = dt / args.steps * 1e3
    value = nloc / (ms_step * 1e-3) / 1e9
    cores = len(os.sched_getaffinity(0))
    res = {
        "impl": "reference",
        "metric": "Ax+dssum fp64 GDOF/s through Jacobi-PCG; CG ms/iter",
        "value": round(value, 4), "unit": "GDOF/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "cg_ms_per_iter": round(ms_step, 3),
        "higher_is_better": True, "scaling": "strong" if args.config in ("c3", "c5") else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded mesh and manufactured source; no datasets)",
        "config": {"workload": CONFIGS[args.config], "sample": desc, "elements": int(E), "lx": N + 1},
        "cpu_baseline": {"kind": "oracle", "cores": cores, "value": round(value, 4), "unit": "GDOF/s",
                         "sample": f"each step = 1 oracle PCG iteration on {desc} ({nloc} local DOF); "
                                   "set-up excluded"},
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
    ap.add_argument("--no-gmres", action="store_true", help="skip the GMRES leg")
    ap.add_argument("--no-pnpn", action="store_true", help="skip the time-step leg")
    ap.add_argument("--pipelined", action="store_true",
                    help="single-reduction (Chronopoulos-Gear) PCG, SURVEY 8(f) f1 (option cg_variant)")
    ap.add_argument("--no-graph", action="store_true",
                    help="issue the CG iterations in stream order (option graph = 0; for ncu launch lists)")
    ap.add_argument("--cpu-leg", default=None, help=argparse.SUPPRESS)  # internal: one oracle leg group
    ap.add_argument("--cpu-legs", default=None, choices=["default", "all"],
                    help="only run the oracle CPU legs (all: + full-size C3/C5 Ax+dssum) and print them")
    ap.add_argument("--affine", action="store_true",
                    help="affine-element operator variant (SURVEY 8(f) f3; never the headline line)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.cpu_leg:
        c, what = args.cpu_leg.split(":", 1)
        print(json.dumps(cpu_leg(c, what)), flush=True)
        return
    if args.cpu_legs:
        print(json.dumps(cpu_baseline(args.config, CPU_LEGS_ALL if args.cpu_legs == "all" else None)), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
