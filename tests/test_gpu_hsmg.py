"""GPU hybrid-Schwarz multigrid (sem_hsmg_apply) and flexible GMRES with it
(sem_gmres_solve, gmres_precond = SEM_PC_HSMG, PAPER.md:72,
reading R16) vs the oracle (oracle/hsmg.py, pinned in
tests/test_oracle_hsmg.py).  Each side builds its own levels: the oracle
from its GLL nodes and lattice / geometric numbering, the library from its
own nodes and topological numbering.

Bars: one V-cycle z = M r rel-L2 <= 1e-10 (the coarse PCG stops at
tol 1e-12, so the two sides may stop one step apart: a 1e-12-relative
difference of the coarse correction); the FGMRES solution <= 1e-10 and the
iteration count within max(1, 1 %) (reading R14: CGS2 vs MGS)."""
import math

import numpy as np
import pytest

import oracle
import semgen
from gpu_common import Case, rel_l2, to_dev, to_np
from oracle import hsmg as H

pytestmark = pytest.mark.gpu

CASES = {
    "box7-periodic": dict(kind="box", N=7, nel=(4, 3, 3), periodic=(True, True, True), deform=0.2),
    "box5-walls": dict(kind="box", N=5, nel=(3, 4, 3), periodic=(True, False, False), deform=0.15),
    "box3-two-levels": dict(kind="box", N=3, nel=(3, 3, 4), periodic=(False, True, True), deform=0.1),
    "box1-coarse-only": dict(kind="box", N=1, nel=(4, 3, 3), periodic=(True, True, False), deform=0.1),
    "cyl9": dict(kind="cyl", N=9, nc=2, nr=1, nz=3),
}


def _case(name):
    p = dict(CASES[name])
    kind, N = p.pop("kind"), p.pop("N")
    c = Case(kind, N, **p)
    if kind == "box":
        nel, per = p["nel"], p["periodic"]
        ids_fn = lambda Nl, cl: oracle.lattice_ids(nel, Nl, per)  # noqa: E731
    else:
        ids_fn = lambda Nl, cl: oracle.geometric_ids(cl, tol=1e-9)  # noqa: E731
    c.levels = H.setup(N, c.mo["coords"], c.mo["bc"], ids_fn)
    return c


def _rhs(c, f):
    bo = oracle.dssum(c.ids, (c.Bo * f).ravel(), c.nuniq) * c.mask.ravel()
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    return bo, b


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("h2c", [0.0, 0.8])
def test_vcycle_matches_oracle(name, h2c):
    c = _case(name)
    f = c.field(301) + 0.3
    bo, b = _rhs(c, f)
    zo = H.vcycle(c.levels, bo, 1.0, h2c, coarse_iters=5)
    z = to_dev(np.zeros_like(f))
    c.mesh.hsmg_apply(b, z, h1c=1.0, h2c=h2c)
    assert rel_l2(to_np(z), zo) <= 1e-10
    # a second application reuses the levels (and the cached coarse Jacobi)
    z2 = to_dev(np.zeros_like(f))
    c.mesh.hsmg_apply(b, z2, h1c=1.0, h2c=h2c)
    assert float((z2 - z).abs().max()) == 0.0


@pytest.mark.parametrize("name", ["box7-periodic", "box5-walls", "cyl9"])
def test_fgmres_hsmg_matches_oracle(name):
    c = _case(name)
    h2c = 0.0 if name != "box5-walls" else 0.6
    f = c.field(302) + 0.5  # non-zero mean: the singular projections act
    bo, b = _rhs(c, f)
    xo, it_o, rr_o, conv_o = H.fgmres(c.levels, bo, 1.0, h2c, tol=1e-10, maxit=300, restart=30)
    c.mesh.set_options(gmres_precond="hsmg")
    x = to_dev(np.zeros_like(f))
    it, rr, conv = c.mesh.gmres_solve(b, x, h2c=h2c, tol=1e-10, maxit=300, restart=30)
    assert conv and conv_o and abs(it - it_o) <= max(1, math.ceil(0.01 * it_o)), (it, it_o)
    assert rel_l2(to_np(x), xo.reshape(f.shape)) <= 1e-10
    assert rr <= 2e-10
    # far fewer iterations than the Jacobi-preconditioned GMRES
    c.mesh.set_options(gmres_precond="jacobi")
    xj = to_dev(np.zeros_like(f))
    itj, _, convj = c.mesh.gmres_solve(b, xj, h2c=h2c, tol=1e-10, maxit=5000, restart=30)
    assert convj and 4 * it <= itj, (it, itj)
    assert rel_l2(to_np(xj), to_np(x)) <= 1e-8


def test_fgmres_hsmg_fixed_iterations_and_restarts():
    c = _case("box5-walls")
    f = c.field(303)
    bo, b = _rhs(c, f)
    xo, it_o, rr_o, _ = H.fgmres(c.levels, bo, 1.0, 0.0, tol=0.0, maxit=9, restart=4)
    c.mesh.set_options(gmres_precond="hsmg")
    x = to_dev(np.zeros_like(f))
    it, rr, conv = c.mesh.gmres_solve(b, x, tol=0.0, maxit=9, restart=4)
    assert it == it_o == 9 and not conv
    assert rel_l2(to_np(x), xo.reshape(f.shape)) <= 1e-10
    assert abs(rr - rr_o) <= 1e-9 * max(rr_o, 1e-300) + 1e-13


def test_hsmg_contract():
    from paper_2405_05640_b200 import sem
    c = _case("box3-two-levels")
    f = c.field(304)
    _, b = _rhs(c, f)
    with pytest.raises(sem.SemError) as ei:
        c.mesh.hsmg_apply(b, b)
    assert ei.value.status == sem.SEM_EINVAL
    c.mesh.set_options(gmres_precond="hsmg")
    x = to_dev(np.zeros_like(f))
    with pytest.raises(sem.SemError) as ei:
        c.mesh.gmres_solve(b, x, h1=to_dev(np.ones_like(f)), tol=1e-8)
    assert ei.value.status == sem.SEM_EINVAL
    with pytest.raises(sem.SemError) as ei:
        c.mesh.set_options(hsmg_coarse_iters=0)
    assert ei.value.status == sem.SEM_EINVAL
    # zero right-hand side: zero solution, no iteration
    z = to_dev(np.zeros_like(f))
    it, rr, conv = c.mesh.gmres_solve(z, x, tol=1e-10, maxit=20)
    assert it == 0 and conv and float(x.abs().max()) == 0.0
    # the V-cycle of a zero residual is zero
    out = to_dev(np.ones_like(f))
    c.mesh.hsmg_apply(z, out)
    assert float(out.abs().max()) == 0.0


def test_vcycle_coarse_iterations_option():
    c = _case("box7-periodic")
    f = c.field(305)
    bo, b = _rhs(c, f)
    c.mesh.set_options(hsmg_coarse_iters=12)
    z = to_dev(np.zeros_like(f))
    c.mesh.hsmg_apply(b, z)
    assert rel_l2(to_np(z), H.vcycle(c.levels, bo, coarse_iters=12)) <= 1e-10
    assert rel_l2(to_np(z), H.vcycle(c.levels, bo, coarse_iters=5)) > 1e-8  # the option acts
