"""GPU Jacobi-PCG (sem_cg_solve) vs the oracle's PCG (O10/R10).

Bar (BASELINE.json north_star): solution rel-L2 <= 1e-10, iteration counts
within +-1.  Each side assembles its own right-hand side b = mask dssum(B f)
from the same seeded / manufactured f.
"""
import math

import numpy as np
import pytest

import oracle
import semgen
from gpu_common import Case, rel_l2, to_dev, to_np

pytestmark = pytest.mark.gpu


def _solve_both(c, f, h1=None, h2=None, h1c=1.0, h2c=0.0, tol=1e-10, maxit=3000):
    bo = oracle.dssum(c.ids, (c.Bo * f).ravel(), c.nuniq) * c.mask.ravel()
    xo, it_o, rr_o, conv_o = oracle.pcg(c.N, c.Go, c.Bo, c.ids, bo, mask=c.mask.ravel(), h1=h1, h2=h2,
                                        h1c=h1c, h2c=h2c, tol=tol, maxit=maxit, nuniq=c.nuniq)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    x = to_dev(np.zeros_like(f))
    it, rr, conv = c.mesh.cg_solve(b, x, None if h1 is None else to_dev(h1),
                                   None if h2 is None else to_dev(h2), h1c, h2c, tol=tol, maxit=maxit)
    return to_np(x), it, rr, conv, xo.reshape(f.shape), it_o, rr_o, conv_o


@pytest.mark.parametrize("deform", [0.0, 0.2])
def test_c1_poisson_manufactured(deform):
    c = Case("box", 7, nel=(4, 4, 4), deform=deform)
    f = semgen.sin3_source(c.ml["coords"]).reshape(c.E, -1)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, tol=1e-12)
    assert conv and conv_o and abs(it - it_o) <= 1
    assert rel_l2(x, xo) <= 1e-10
    # and the manufactured solution itself (spectral accuracy at N=7)
    ue = semgen.sin3(c.ml["coords"]).reshape(c.E, -1)
    B = c.Bo
    xm = x - np.sum(B * x) / B.sum()
    um = ue - np.sum(B * ue) / B.sum()
    assert np.max(np.abs(xm - um)) < (1e-7 if deform == 0 else 1e-4)


@pytest.mark.parametrize("deform", [0.0, 0.2])
def test_singular_random_rhs_projection(deform):
    """Periodic Poisson with a right-hand side whose weighted mean is NOT zero
    (f ~ U(-1,1) + 0.7): exercises the singular-system projections of b and x
    (reading R10 / SURVEY 8(c) O10, G15) with a non-trivial mean, which the
    symmetric manufactured sources never do.  x, iteration count and the
    reported residual against the oracle."""
    c = Case("box", 7, nel=(4, 4, 3), deform=deform)
    f = c.field(35) + 0.7
    bo = oracle.dssum(c.ids, (c.Bo * f).ravel(), c.nuniq)
    assert abs(np.sum(c.mult.ravel() * bo)) > 0.01 * np.sum(c.mult.ravel() * np.abs(bo))
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, tol=1e-10)
    assert conv and conv_o and abs(it - it_o) <= 1, (it, it_o)
    assert rel_l2(x, xo) <= 1e-10
    if it == it_o:
        # at rel_res ~ 1e-10 both recursive residuals are mostly rounding
        # history: agreement to a few per cent, not to 1e-12
        assert abs(rr - rr_o) <= 0.1 * rr_o
    # the solution is mean-zero over unique nodes on both sides
    assert abs(np.sum(c.mult * x)) <= 1e-12 * np.sum(c.mult * np.abs(x))
    # fixed-iteration mode: the same projections, iterate by iterate
    x10, it10, rr10, _, xo10, it_o10, rr_o10, _ = _solve_both(c, f, tol=0.0, maxit=10)
    assert it10 == it_o10 == 10
    assert rel_l2(x10, xo10) <= 1e-10 and abs(rr10 - rr_o10) <= 1e-12


def test_helmholtz_walls_arrays():
    c = Case("box", 5, nel=(3, 4, 3), periodic=(True, False, False), deform=0.2)
    f = c.field(31)
    h1 = semgen.positive_field(f.shape, 32)
    h2 = semgen.positive_field(f.shape, 33)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, h1=h1, h2=h2, tol=1e-10)
    assert conv and conv_o and abs(it - it_o) <= 1
    assert rel_l2(x, xo) <= 1e-10


def test_cylinder_helmholtz_c5_coefficients():
    # C5 velocity Helmholtz: h1 = sqrt(Pr/Ra) (Ra = 1e11, Pr = 1),
    # h2 = (11/6)/dt with dt = 1e-3 (BDF3), all walls Dirichlet, lx = 10
    c = Case("cyl", 9, nc=2, nr=1, nz=3)
    h1c = math.sqrt(1.0 / 1e11)
    h2c = (11.0 / 6.0) / 1e-3
    f = semgen.cyl_source(c.ml["coords"], h1=h1c, h2=h2c).reshape(c.E, -1)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, h1c=h1c, h2c=h2c, tol=1e-10)
    assert conv and conv_o and abs(it - it_o) <= 1
    assert rel_l2(x, xo) <= 1e-10


def test_cylinder_poisson_manufactured():
    c = Case("cyl", 9, nc=2, nr=1, nz=3)
    f = semgen.cyl_source(c.ml["coords"]).reshape(c.E, -1)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, tol=1e-11)
    assert conv and conv_o and abs(it - it_o) <= 1
    assert rel_l2(x, xo) <= 1e-10
    ue = semgen.cyl_exact(c.ml["coords"]).reshape(c.E, -1)
    assert np.max(np.abs(x - ue)) < 1e-2


def test_tgv_pressure_small():
    c = Case("box", 7, nel=(6, 6, 6))
    f = semgen.tgv_source(c.ml["coords"]).reshape(c.E, -1)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, tol=1e-10)
    assert conv and abs(it - it_o) <= 1
    assert rel_l2(x, xo) <= 1e-10


def test_contract_cases():
    from paper_2405_05640_b200 import sem
    c = Case("box", 3, nel=(3, 3, 3), periodic=(False,) * 3)
    z = to_dev(np.zeros((c.E, c.lx ** 3)))
    x = to_dev(np.zeros((c.E, c.lx ** 3)))
    it, rr, conv = c.mesh.cg_solve(z, x, tol=1e-10, maxit=50)
    assert it == 0 and conv and float(x.abs().max()) == 0.0
    f = c.field(41)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    it, rr, conv = c.mesh.cg_solve(b, x, tol=1e-14, maxit=3)
    assert it == 3 and not conv and rr > 0
    it, rr, conv = c.mesh.cg_solve(b, x, tol=0.0, maxit=11)  # fixed-iteration mode
    assert it == 11 and not conv
    bo = oracle.dssum(c.ids, (c.Bo * f).ravel(), c.nuniq) * c.mask.ravel()
    xo, it_o, _, _ = oracle.pcg(c.N, c.Go, c.Bo, c.ids, bo, mask=c.mask.ravel(), tol=0.0, maxit=11,
                                nuniq=c.nuniq)
    assert rel_l2(to_np(x), xo) <= 1e-10
    with pytest.raises(sem.SemError) as ei:
        c.mesh.cg_solve(b, x, h1c=1.0, h2c=-1e4, tol=1e-10, maxit=50)
    assert ei.value.status == sem.SEM_EBREAKDOWN


def test_host_buffer_path_matches_device_path():
    import torch
    c = Case("box", 7, nel=(4, 4, 4), deform=0.2)
    f = semgen.sin3_source(c.ml["coords"]).reshape(c.E, -1)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    x = to_dev(np.zeros_like(f))
    r1 = c.mesh.cg_solve(b, x, tol=1e-10, maxit=500)
    bh = b.cpu().pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    r2 = c.mesh.cg_solve_host(bh, xh, tol=1e-10, maxit=500)
    assert r1[0] == r2[0]
    np.testing.assert_array_equal(xh.numpy(), to_np(x))


def test_deterministic_repeat():
    c = Case("box", 7, nel=(4, 4, 4), deform=0.2)
    f = c.field(51)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    xs = []
    for _ in range(2):
        x = to_dev(np.zeros_like(f))
        c.mesh.cg_solve(b, x, tol=1e-10, maxit=500)
        xs.append(to_np(x))
    np.testing.assert_array_equal(xs[0], xs[1])


@pytest.mark.parametrize("kind", ["c1", "c1def", "walls", "cyl-c5", "lx4"])
def test_pipelined_cg(kind):
    # single-reduction (Chronopoulos-Gear) PCG, SURVEY 8(f) f1 (option
    # cg_variant): same iterates as the oracle's standard PCG up to rounding
    # -> same bar
    h1 = h2 = None
    h1c, h2c = 1.0, 0.0
    if kind in ("c1", "c1def"):
        c = Case("box", 7, nel=(4, 4, 4), deform=0.0 if kind == "c1" else 0.2)
        f = semgen.sin3_source(c.ml["coords"]).reshape(c.E, -1)
    elif kind == "walls":
        c = Case("box", 5, nel=(3, 4, 3), periodic=(True, False, False), deform=0.2)
        f = c.field(71)
        h1 = semgen.positive_field(f.shape, 72)
        h2 = semgen.positive_field(f.shape, 73)
    elif kind == "cyl-c5":
        c = Case("cyl", 9, nc=2, nr=1, nz=3)
        h1c, h2c = math.sqrt(1.0 / 1e11), (11.0 / 6.0) / 1e-3
        f = semgen.cyl_source(c.ml["coords"], h1=h1c, h2=h2c).reshape(c.E, -1)
    else:
        c = Case("box", 3, nel=(3, 3, 4), periodic=(False, True, True), deform=0.1)
        f = c.field(74)
    c.mesh.set_options(cg_variant="pipelined")
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, h1=h1, h2=h2, h1c=h1c, h2c=h2c, tol=1e-10)
    assert conv and conv_o and abs(it - it_o) <= 1, (it, it_o)
    assert rel_l2(x, xo) <= 1e-10


def test_graph_replay_matches_stream_order():
    # the CUDA-graph replay of the CG iteration (option graph, default on)
    # must be bit-identical to issuing the same launches in stream order
    c = Case("box", 7, nel=(4, 4, 4), deform=0.2)
    f = c.field(81)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    xs = []
    for g in (1, 0):
        c.mesh.set_options(graph=g)
        x = to_dev(np.zeros_like(f))
        r = c.mesh.cg_solve(b, x, tol=1e-10, maxit=500)
        xs.append((r[0], to_np(x)))
    assert xs[0][0] == xs[1][0]
    np.testing.assert_array_equal(xs[0][1], xs[1][1])


@pytest.mark.parametrize("graph", [1, 0])
def test_pdl_matches_plain_launches(graph):
    # option pdl (programmatic dependent launch of the iteration's kernels):
    # the same kernels in the same order -> bit-identical iterates
    c = Case("box", 7, nel=(4, 4, 4), deform=0.2)
    f = c.field(82) + 0.3
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    xs = []
    for pdl in (1, 0):
        c.mesh.set_options(graph=graph, pdl=pdl)
        x = to_dev(np.zeros_like(f))
        r = c.mesh.cg_solve(b, x, tol=1e-10, maxit=500)
        xs.append((r[0], to_np(x)))
    assert xs[0][0] == xs[1][0]
    np.testing.assert_array_equal(xs[0][1], xs[1][1])


@pytest.mark.parametrize("kind", ["c1def", "singular", "walls", "cyl-c5", "lx4", "lx2"])
@pytest.mark.parametrize("layout", [0, 1])
def test_cg_layout_both_ways(kind, layout):
    # option cg_layout (x-planes-last element layout of the CG vectors,
    # DESIGN.md section 4) on and off, each against the oracle's PCG at the
    # north-star bar
    h1 = h2 = None
    h1c, h2c = 1.0, 0.0
    if kind == "c1def":
        c = Case("box", 7, nel=(4, 4, 4), deform=0.2)
        f = semgen.sin3_source(c.ml["coords"]).reshape(c.E, -1)
    elif kind == "singular":
        c = Case("box", 5, nel=(3, 4, 5), deform=0.2)
        f = c.field(91) + 0.7
    elif kind == "walls":
        c = Case("box", 5, nel=(3, 4, 3), periodic=(True, False, False), deform=0.2)
        f = c.field(71)
        h1 = semgen.positive_field(f.shape, 72)
        h2 = semgen.positive_field(f.shape, 73)
    elif kind == "cyl-c5":
        c = Case("cyl", 9, nc=2, nr=1, nz=3)
        h1c, h2c = math.sqrt(1.0 / 1e11), (11.0 / 6.0) / 1e-3
        f = semgen.cyl_source(c.ml["coords"], h1=h1c, h2=h2c).reshape(c.E, -1)
    elif kind == "lx4":
        c = Case("box", 3, nel=(3, 3, 4), periodic=(False, True, True), deform=0.1)
        f = c.field(74)
    else:  # lx = 2: no face or edge interiors, the planes are the whole element
        c = Case("box", 1, nel=(4, 3, 3), periodic=(True, True, False), deform=0.0)
        f = c.field(75)
    c.mesh.set_options(cg_layout=layout)
    x, it, rr, conv, xo, it_o, rr_o, conv_o = _solve_both(c, f, h1=h1, h2=h2, h1c=h1c, h2c=h2c, tol=1e-10)
    assert conv and conv_o and abs(it - it_o) <= 1, (it, it_o)
    assert rel_l2(x, xo) <= 1e-10
