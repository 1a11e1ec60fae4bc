"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (bench.problem builds the same meshes, sources and coefficients).

- C2 (32^3, lx = 8): the fused Ax+dssum against the oracle on every element,
  and the fixed-iteration PCG (tol = 0, as timed; 10 iterations) against the
  oracle's PCG.
- C3 (64^3) and C5 (cylinder, lx = 10, Helmholtz): Ax+dssum on sampled
  elements.  Every copy of a node of a sampled element lies in an element
  sharing a vertex with it, so the oracle computes those elements' assembled
  values exactly from that closure alone (its own GLL, geometry and geometric
  numbering of the closure).
- C3: the solver's reported residual equals ||b - mask dssum(A x)|| / ||b||
  recomputed with the standalone operator (a property at any size).
Bars: 1e-12 relative (Ax/dssum), 1e-10 (CG solution); on C5's wall-clustered
axial layers (node spacing ~3e-6 at |z| ~ 1) the Ax/dssum bar follows the
geometry's conditioning (reading R13, `_geom_tol`).
"""
import numpy as np
import pytest

import oracle
import semgen
from gpu_common import rel_l2

pytestmark = pytest.mark.gpu


def _problem(cfg):
    import bench
    from paper_2405_05640_b200 import sem
    N0 = 9 if cfg == "c5" else 7
    xl, _ = sem.sem_gll(N0)
    pb = bench.problem(cfg, 1, 0, xl)
    m = pb["mesh"]
    mesh = sem.Mesh(m["conn"].shape[0], pb["N"], m["coords"], m["conn"], m["bc"])
    mesh.geom_factors()
    return pb, mesh


def _gpu_ax_dssum(mesh, u_host, h1c, h2c):
    import torch
    u = torch.from_numpy(u_host).cuda()
    w = torch.empty_like(u)
    mesh.ax_dssum(u, w, h1c=h1c, h2c=h2c)
    torch.cuda.synchronize()
    return u, w


def _geom_tol(coords):
    """Bar for meshes whose node spacing is tiny next to the coordinates
    (reading R13): both sides differentiate coordinates that carry
    an absolute rounding of eps |x|, so independent implementations of the
    geometric factors agree to ~eps |x|_max / h_min, not better.  The bar is
    max(1e-12, 40 eps |x|_max / h_min) with h_min the smallest distance
    between neighbouring nodes of the closure; 40 = 2 (both end points of a
    difference) x 3 (~sqrt(lx) rounding of a D row) x 3 (G ~ J R R^T depends
    quadratically on the inverse Jacobian) x 2 (margin)."""
    X = np.asarray(coords).reshape(3, -1, coords.shape[-1])
    n = X.shape[-1]
    lx = round(n ** (1 / 3))
    Y = X.reshape(3, -1, lx, lx, lx)
    h = min(float(np.min(np.linalg.norm(np.diff(Y, axis=ax), axis=0))) for ax in (2, 3, 4))
    return max(1e-12, 40 * np.finfo(float).eps * float(np.max(np.abs(X))) / h)


def _closure(conn, sample):
    """Elements sharing at least one vertex with a sampled element."""
    verts = np.unique(conn[sample].ravel())
    return np.flatnonzero(np.isin(conn, verts).any(axis=1))


def _oracle_closure(N, coords, bc, u, closure, sample, periods, h1c, h2c):
    G, B = oracle.geom(N, coords)
    ids, nuniq = oracle.geometric_ids(coords, periods=periods, tol=1e-9)
    n3 = (N + 1) ** 3
    ids = ids.reshape(-1, n3)
    mask = oracle.mask_from_bc(N, bc, ids, nuniq)
    w = oracle.ax_dssum(N, G, B, ids, u, mask=mask, h1c=h1c, h2c=h2c, nuniq=nuniq)
    pos = {int(e): q for q, e in enumerate(closure)}
    return w[[pos[int(e)] for e in sample]]


def test_c2_full_ax_dssum_and_fixed_iteration_cg():
    import torch
    pb, mesh = _problem("c2")
    N, E = pb["N"], pb["mesh"]["conn"].shape[0]
    n3 = (N + 1) ** 3
    xo, _ = oracle.gll(N)
    mo = semgen.box_mesh(pb["nel"], xo, lengths=tuple(2 * np.pi for _ in range(3)), periodic=(True,) * 3)
    G, B = oracle.geom(N, mo["coords"])
    ids, nuniq = oracle.lattice_ids(pb["nel"], N, (True,) * 3)
    u = semgen.random_field((E, n3), 11)
    _, w = _gpu_ax_dssum(mesh, u, 1.0, 0.0)
    wo = oracle.ax_dssum(N, G, B, ids, u, nuniq=nuniq)
    assert rel_l2(w.cpu().numpy(), wo) <= 1e-12
    # the timed configuration: tol = 0, fixed iterations (10 of the 100)
    bo = oracle.dssum(ids, (B * pb["f"]).ravel(), nuniq)
    xo_, it_o, _, _ = oracle.pcg(N, G, B, ids, bo, tol=0.0, maxit=10, nuniq=nuniq)
    b = torch.empty((E, n3), dtype=torch.float64, device="cuda")
    mesh.rhs(torch.from_numpy(np.ascontiguousarray(pb["f"])).cuda(), b)
    x = torch.zeros_like(b)
    it, _, conv = mesh.cg_solve(b, x, tol=0.0, maxit=10)
    assert it == it_o == 10 and not conv
    assert rel_l2(x.cpu().numpy(), xo_) <= 1e-10
    # a right-hand side with a non-zero mean (f ~ U(-1,1) + 0.7): the
    # singular-system projections of b and x at full size (reading R10)
    f2 = semgen.random_field((E, n3), 14) + 0.7
    bo2 = oracle.dssum(ids, (B * f2).ravel(), nuniq)
    xo2, it_o2, rr_o2, _ = oracle.pcg(N, G, B, ids, bo2, tol=0.0, maxit=10, nuniq=nuniq)
    mesh.rhs(torch.from_numpy(f2).cuda(), b)
    x.zero_()
    it2, rr2, _ = mesh.cg_solve(b, x, tol=0.0, maxit=10)
    assert it2 == it_o2 == 10
    assert rel_l2(x.cpu().numpy(), xo2) <= 1e-10 and abs(rr2 - rr_o2) <= 1e-12
    mesh.close()


def test_c3_full_sampled_ax_dssum_and_residual():
    import torch
    pb, mesh = _problem("c3")
    N, m = pb["N"], pb["mesh"]
    E, n3 = m["conn"].shape[0], (N + 1) ** 3
    u = semgen.random_field((E, n3), 12)
    ut, w = _gpu_ax_dssum(mesh, u, 1.0, 0.0)
    rng = np.random.default_rng(3)
    sample = np.sort(rng.choice(E, 8, replace=False))
    clo = _closure(m["conn"], sample)
    xo, _ = oracle.gll(N)
    per = m["periods"]
    # the oracle's own coordinates of the closure (same generator, its GLL)
    lat = semgen.box_partition(pb["nel"], (1, 1, 1), 0)
    mo = semgen.box_mesh(pb["nel"], xo, lengths=tuple(2 * np.pi for _ in range(3)), periodic=(True,) * 3,
                         elems=[lat[e] for e in clo])
    wo = _oracle_closure(N, mo["coords"], mo["bc"], u[clo], clo, sample, per, 1.0, 0.0)
    assert rel_l2(w.cpu().numpy()[sample], wo) <= 1e-12
    # residual property of the timed solve (tol = 0, fixed iterations)
    b = torch.empty_like(ut)
    mesh.rhs(torch.from_numpy(np.ascontiguousarray(pb["f"])).cuda(), b)
    x = torch.zeros_like(b)
    it, rr, _ = mesh.cg_solve(b, x, tol=0.0, maxit=20)
    ax = torch.empty_like(b)
    mesh.ax_dssum(x, ax)
    mult = mesh.mult_mask()[0]
    r = b - ax
    rn = torch.sqrt((mult * r * r).sum()).item()
    bn = torch.sqrt((mult * b * b).sum()).item()
    assert it == 20 and abs(rn / bn - rr) <= 1e-6 * rr
    mesh.close()


def test_c5_full_sampled_ax_dssum():
    pb, mesh = _problem("c5")
    N, m = pb["N"], pb["mesh"]
    E, n3 = m["conn"].shape[0], (N + 1) ** 3
    u = semgen.random_field((E, n3), 13)
    _, w = _gpu_ax_dssum(mesh, u, pb["h1c"], pb["h2c"])
    w = w.cpu().numpy()
    mesh.close()
    E2, nz = m["E_per_layer"], m["nz"]
    xo, _ = oracle.gll(N)
    rng = np.random.default_rng(4)
    for layer in (0, nz // 2, nz - 1):  # bottom wall, middle, top wall
        sample = layer * E2 + np.sort(rng.choice(E2, 3, replace=False))
        sample = np.concatenate([sample, [layer * E2 + E2 - 1]])  # an outer (side-wall) element
        clo = _closure(m["conn"], sample)
        k0, k1 = max(0, layer - 1), min(nz, layer + 2)
        mo = semgen.cylinder_mesh(xo, nc=m["nc"], nr=m["nr"], nz=nz, layers=(k0, k1))
        loc = clo - k0 * E2
        wo = _oracle_closure(N, mo["coords"][:, loc], mo["bc"][loc], u[clo], clo, sample, (None,) * 3,
                             pb["h1c"], pb["h2c"])
        errs = [rel_l2(w[s], o) for s, o in zip(sample, wo)]
        if layer == nz // 2:
            # mid-cell: the axial spacing is ~1e-2, no conditioning loss -> the
            # north-star bar itself
            assert max(errs) <= 1e-12, (layer, sample.tolist(), errs)
            continue
        # wall layers (reading R13): each sampled element against the bar
        # derived from ITS OWN closure's coordinates
        for s, err in zip(sample, errs):
            own = np.flatnonzero(clo == s)
            assert err <= _geom_tol(mo["coords"][:, loc[own]]), (layer, int(s), err)
