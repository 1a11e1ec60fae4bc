"""GPU restarted GMRES (sem_gmres_solve) vs the oracle's
GMRES (O12, itself pinned to the Krylov minimal-residual definition in
tests/test_oracle_gmres.py).  Bars: solution rel-L2 <= 1e-10 (as for CG);
iteration counts within max(1, 1 %) -- the GPU orthogonalises by classical
Gram-Schmidt with re-orthogonalisation, the oracle by modified Gram-Schmidt
(equal in exact arithmetic; reading R14), and over hundreds of
restarted iterations the rounding difference can move the stopping step by
a couple; fixed-iteration runs (tol = 0) compare iterate by iterate,
including restarts."""
import math

import numpy as np
import pytest

import oracle
import semgen
from gpu_common import Case, rel_l2, to_dev, to_np

pytestmark = pytest.mark.gpu


def _both(c, f, h1c=1.0, h2c=0.0, tol=1e-10, maxit=2000, restart=30):
    bo = oracle.dssum(c.ids, (c.Bo * f).ravel(), c.nuniq) * c.mask.ravel()
    xo, it_o, rr_o, conv_o = oracle.gmres(c.N, c.Go, c.Bo, c.ids, bo, mask=c.mask.ravel(), h1c=h1c, h2c=h2c,
                                          tol=tol, maxit=maxit, restart=restart, nuniq=c.nuniq)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    x = to_dev(np.zeros_like(f))
    it, rr, conv = c.mesh.gmres_solve(b, x, h1c=h1c, h2c=h2c, tol=tol, maxit=maxit, restart=restart)
    return to_np(x), it, rr, conv, xo.reshape(f.shape), it_o, rr_o, conv_o


@pytest.mark.parametrize("kind", ["walls-helm", "periodic-singular", "cyl"])
def test_gmres_converged(kind):
    if kind == "walls-helm":
        c = Case("box", 5, nel=(3, 4, 3), periodic=(True, False, False), deform=0.2)
        f, h1c, h2c, restart = c.field(91), 1.0, 0.7, 20
    elif kind == "periodic-singular":
        c = Case("box", 7, nel=(4, 4, 3), deform=0.2)
        f, h1c, h2c, restart = c.field(92) + 0.7, 1.0, 0.0, 30  # non-zero mean: projections act
    else:
        c = Case("cyl", 9, nc=2, nr=1, nz=3)
        f = semgen.cyl_source(c.ml["coords"]).reshape(c.E, -1)
        h1c, h2c, restart = 1.0, 0.0, 25
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _both(c, f, h1c, h2c, tol=1e-10, restart=restart)
    assert conv and conv_o and abs(it - it_o) <= max(1, math.ceil(0.01 * it_o)), (it, it_o)
    assert rel_l2(x, xo) <= 1e-10
    assert rr <= 2e-10


@pytest.mark.parametrize("restart,maxit", [(30, 12), (4, 11), (1, 5)])
def test_gmres_fixed_iterations(restart, maxit):
    # tol = 0: exactly maxit Arnoldi steps, restarts every `restart`
    c = Case("box", 7, nel=(4, 3, 3), periodic=(True, False, True), deform=0.2)
    f = c.field(93)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _both(c, f, tol=0.0, maxit=maxit, restart=restart)
    assert it == it_o == maxit and not conv
    assert rel_l2(x, xo) <= 1e-10
    assert abs(rr - rr_o) <= 1e-10 * max(1.0, rr_o) + 1e-6 * rr_o


def test_gmres_matches_cg_solution():
    # both Krylov methods solve the same SPD system: same x to the tolerance
    c = Case("box", 7, nel=(4, 4, 4), deform=0.2)
    f = semgen.sin3_source(c.ml["coords"]).reshape(c.E, -1)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    x1 = to_dev(np.zeros_like(f))
    x2 = to_dev(np.zeros_like(f))
    c.mesh.cg_solve(b, x1, tol=1e-12, maxit=3000)
    it, rr, conv = c.mesh.gmres_solve(b, x2, tol=1e-12, maxit=3000, restart=30)
    assert conv
    assert rel_l2(to_np(x2), to_np(x1)) <= 1e-9


def test_gmres_contract():
    from paper_2405_05640_b200 import sem
    c = Case("box", 3, nel=(3, 3, 3), periodic=(False,) * 3)
    z = to_dev(np.zeros((c.E, c.lx ** 3)))
    x = to_dev(np.zeros((c.E, c.lx ** 3)))
    it, rr, conv = c.mesh.gmres_solve(z, x, tol=1e-10, maxit=50)
    assert it == 0 and conv and float(x.abs().max()) == 0.0
    with pytest.raises(sem.SemError) as ei:
        c.mesh.gmres_solve(z, x, restart=31)
    assert ei.value.status == sem.SEM_EINVAL
    f = c.field(94)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    it, rr, conv = c.mesh.gmres_solve(b, x, tol=1e-14, maxit=3, restart=2)
    assert it == 3 and not conv and rr > 0
