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


def _bytes_per_dof(helmholtz):
    """Algorithmic bytes per local DOF before the
    gather-scatter's share: the fused CG operator, the standalone Ax+dssum,
    and one whole CG iteration."""
    hb = 8 if helmholtz else 0
    cg_op = 104 + hb   # G x 6, r, dinv, p, x in; p, x, w out (+ B)
    axd = 64 + hb      # u, G x 6 (+ B) in; w out
    cg_iter = cg_op + 32  # + the update pass: r, w, dinv in; r out
    return cg_op, axd, cg_iter


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
    # gather-scatter traffic (BASELINE north star: "plus gs traffic"): every
    # local copy of a shared node is read and written once, a masked single
    # copy written once
    mult_, mask_ = mesh.mult_mask()
    gs_bytes = float(16 * (mult_ < 1.0).sum().item() + 8 * ((mult_ == 1.0) & (mask_ == 0.0)).sum().item())
    del mult_, mask_
    f = torch.from_numpy(np.ascontiguousarray(pb["f"])).cuda()
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
    mesh.profile_enable(True)
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
    ax_launches, ax_ms, kl1 = mesh.profile_get()
    mesh.profile_enable(False)
    gpu_launches = kl1 - kl0

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
    b_cg, b_axd, b_it = _bytes_per_dof(helm)
    b_gs = gs_bytes / nloc             # per local DOF, this rank's mesh
    b_cg, b_axd, b_it = b_cg + b_gs, b_axd + b_gs, b_it + b_gs
    if info.affine:  # the affine variant reads 48 B per element instead of G x 6 per node
        b_cg, b_axd, b_it = b_cg - 48, b_axd - 48, b_it - 48
    achieved = b_cg * nloc / (ax_avg_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(args.config)
    except Exception:
        pass
    res = None
    if rank == 0:
        cpu = None if (n > 1 or args.no_cpu_baseline) else cpu_baseline(args)
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
                       "solver": "tol=0 fixed iterations, Jacobi-PCG"},
            "roofline": {"kernel": "fused CG operator: k_ax<CG> (deferred x update + p update + Ax + pAp partials), "
                                   "then the nodal gather-scatter k_gs_nodal (mask . dssum)",
                         "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "bytes_per_dof": round(b_cg, 2), "gs_bytes_per_dof": round(b_gs, 2),
                         "avg_launch_ms": round(ax_avg_ms, 5), "launches_timed": ax_launches},
            "cg_iteration": {"bytes_per_dof": round(b_it, 2), "ms": round(ms_step / iters, 5),
                             "achieved_gbs": round(b_it * nloc / (ms_step / iters * 1e-3) / 1e9, 1),
                             "frac": round(b_it * nloc / (ms_step / iters * 1e-3) / 1e9 / peak, 4)},
            "ax_dssum_standalone": {"gdofs": round(nloc / (ax_alone_ms * 1e-3) / 1e9, 3),
                                    "ms": round(ax_alone_ms, 5), "bytes_per_dof": round(b_axd, 2),
                                    "achieved_gbs": round(b_axd * nloc / (ax_alone_ms * 1e-3) / 1e9, 1),
                                    "frac": round(b_axd * nloc / (ax_alone_ms * 1e-3) / 1e9 / peak, 4)},
            "e2e": {"value": round(iters * dof_total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GDOF/s",
                    "h2d_bytes_per_step": int(nloc * 8), "d2h_bytes_per_step": int(nloc * 8),
                    "ms_per_step": round(e2e_ms, 4)},
            "gpu_launches": int(tots[1].item()),
            "variant": ("affine elements: 6 metric constants per element instead of G per node "
                        "(SURVEY 8(f) f3; bytes_per_dof without G)" if info.affine else "general (G per node)"),
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


def _oracle_setup(cfg):
    """Oracle-side problem for the CPU legs (its own GLL, geometry and
    numbering); c3/c5 use a bounded sample (c3: the 32^3 box, c5: two axial
    layers of the cylinder)."""
    import oracle
    N0 = 9 if cfg == "c5" else 7
    xo, _ = oracle.gll(N0)
    reduced = cfg in ("c3", "c5")
    pb = problem("c2" if cfg == "c3" else cfg, 1, 0, xo, reduced=(cfg == "c5"))
    m, N = pb["mesh"], pb["N"]
    G, B = oracle.geom(N, m["coords"])
    if pb["nel"] is not None:
        ids, nuniq = oracle.lattice_ids(pb["nel"], N, (True, True, True))
    else:
        ids, nuniq = oracle.geometric_ids(m["coords"], tol=1e-9)
    mask = oracle.mask_from_bc(N, m["bc"], ids, nuniq)
    b = oracle.dssum(ids, (B * pb["f"]).ravel(), nuniq) * mask
    dinv = oracle.jacobi(N, G, B, ids, mask, h1c=pb["h1c"], h2c=pb["h2c"], nuniq=nuniq)
    desc = ("c2 32^3 box (bounded sample of c3)" if cfg == "c3" else
            "2 of 128 axial layers of the c5 cylinder" if cfg == "c5" else f"the full {cfg} mesh")
    return N, G, B, ids, nuniq, b, dinv, mask, pb["h1c"], pb["h2c"], desc, reduced


def cpu_baseline(args):
    """The oracle (as it stands) on the host cores: PCG iterations of the same
    workload (or a bounded sample of it), set-up excluded."""
    import oracle
    t0 = time.time()
    N, G, B, ids, nuniq, b, dinv, mask, h1c, h2c, desc, _ = _oracle_setup(args.config)
    setup_s = time.time() - t0
    E = G.shape[0]
    nloc = E * (N + 1) ** 3
    k = 2
    t0 = time.time()
    oracle.pcg(N, G, B, ids, b, mask=mask, h1c=h1c, h2c=h2c, tol=0.0, maxit=k, nuniq=nuniq, dinv=dinv)
    dt = time.time() - t0
    cores = len(os.sched_getaffinity(0))
    return {"value": round(k * nloc / dt / 1e9, 4), "unit": "GDOF/s", "cores": cores, "kind": "oracle",
            "ms_per_iter": round(dt / k * 1e3, 2),
            "sample": f"{k} oracle PCG iterations (tol=0) on {desc} ({E} elements, {nloc} local DOF), "
                      f"set-up ({setup_s:.1f} s) excluded; OpenMP threads = "
                      f"{os.environ.get('OMP_NUM_THREADS', cores)}"}


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
    ap.add_argument("--affine", action="store_true",
                    help="affine-element operator variant (SURVEY 8(f) f3; never the headline line)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.affine:
        os.environ["SEM_AFFINE"] = "1"  # read by sem_geom_factors
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
