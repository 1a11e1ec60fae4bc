"""GPU-vs-oracle parity of every step of the hot path, through the C ABI.

Tolerances (BASELINE.json north_star):
  geometry G, B            rel-L2 <= 1e-13
  Ax, Ax+dssum, rhs, dinv  rel-L2 <= 1e-12
  dssum / mask of a given field: bit-exact (same summation order)
  numbering: the library's topological ids induce exactly the oracle's
  partition of local nodes (bijection), unique counts equal.
"""
import numpy as np
import pytest

import oracle
import semgen
from gpu_common import Case, rel_l2, to_dev, to_np

pytestmark = pytest.mark.gpu

CASES = [
    ("box", 7, dict(nel=(4, 4, 4))),                                        # C1 shape
    ("box", 7, dict(nel=(4, 4, 4), deform=0.2)),                            # deformed C1
    ("box", 4, dict(nel=(3, 4, 5), periodic=(False, False, False))),        # walled, ragged
    ("box", 5, dict(nel=(3, 3, 4), periodic=(True, False, True), deform=0.2)),
    ("cyl", 9, dict(nc=2, nr=1, nz=3)),                                     # C5 shape, lx=10
]
IDS = ["c1", "c1def", "walled", "channel-def", "cyl-lx10"]


@pytest.fixture(scope="module", params=list(range(len(CASES))), ids=IDS)
def case(request):
    kind, N, kw = CASES[request.param]
    return Case(kind, N, **kw)


def test_gll_matches_oracle():
    from paper_2405_05640_b200 import sem
    for N in range(1, 12):
        xl, wl = sem.sem_gll(N)
        xo, wo = oracle.gll(N)
        np.testing.assert_allclose(xl, xo, atol=2e-15)
        np.testing.assert_allclose(wl, wo, rtol=2e-14)


def test_numbering_bijection(case):
    lib_ids = case.mesh.global_ids()
    info = case.mesh.info()
    assert info.n_unique == case.nuniq
    pairs = np.unique(np.stack([lib_ids.ravel(), case.ids.ravel()]), axis=1)
    assert pairs.shape[1] == case.nuniq
    assert len(np.unique(lib_ids)) == case.nuniq


def test_mult_mask(case):
    mult, mask = case.mesh.mult_mask()
    np.testing.assert_array_equal(to_np(mult), case.mult)
    np.testing.assert_array_equal(to_np(mask), case.mask)
    assert case.mesh.info().n_masked == int((case.mask == 0).sum())


def test_geometry(case):
    G, B = case.mesh.geom_get()
    assert rel_l2(to_np(G), case.Go) <= 1e-13
    assert rel_l2(to_np(B), case.Bo) <= 1e-13


@pytest.mark.parametrize("helm", ["poisson", "const", "arrays"])
def test_ax_local(case, helm):
    u = case.field(1)
    h1 = h2 = None
    h1c, h2c = 1.0, 0.0
    if helm == "const":
        h1c, h2c = 0.7, 3.0
    elif helm == "arrays":
        h1 = semgen.positive_field(u.shape, 2)
        h2 = semgen.positive_field(u.shape, 3)
    ref = oracle.ax(case.N, case.Go, case.Bo, u, h1, h2, h1c, h2c)
    w = to_dev(np.zeros_like(u))
    case.mesh.ax(to_dev(u), w, None if h1 is None else to_dev(h1), None if h2 is None else to_dev(h2),
                 h1c, h2c)
    assert rel_l2(to_np(w), ref) <= 1e-12


def test_gs_bit_exact(case):
    from paper_2405_05640_b200 import sem
    u = case.field(4)
    d = to_dev(u)
    case.mesh.gs_op(d, sem.SEM_GS_ADD)
    ref = oracle.dssum(case.ids, u.ravel(), case.nuniq).reshape(u.shape)
    np.testing.assert_array_equal(to_np(d), ref)
    case.mesh.gs_op(d, sem.SEM_GS_MASK)
    np.testing.assert_array_equal(to_np(d), ref * case.mask)


@pytest.mark.parametrize("helm", ["poisson", "arrays"])
def test_ax_dssum_fused(case, helm):
    from paper_2405_05640_b200 import sem
    u = case.field(5)
    h1 = h2 = None
    if helm == "arrays":
        h1 = semgen.positive_field(u.shape, 6)
        h2 = semgen.positive_field(u.shape, 7)
    ref = oracle.ax_dssum(case.N, case.Go, case.Bo, case.ids, u, mask=case.mask, h1=h1, h2=h2,
                          nuniq=case.nuniq)
    dh1 = None if h1 is None else to_dev(h1)
    dh2 = None if h2 is None else to_dev(h2)
    w = to_dev(np.zeros_like(u))
    du = to_dev(u)
    for _ in range(3):  # repeated launches: arrival counters must reset
        case.mesh.ax_dssum(du, w, dh1, dh2)
        assert rel_l2(to_np(w), ref) <= 1e-12
    # fused == unfused (ax, then gs ADD, then MASK) bit for bit
    w2 = to_dev(np.zeros_like(u))
    case.mesh.ax(du, w2, dh1, dh2)
    case.mesh.gs_op(w2, sem.SEM_GS_ADD)
    case.mesh.gs_op(w2, sem.SEM_GS_MASK)
    np.testing.assert_array_equal(to_np(w), to_np(w2))


def test_rhs_and_jacobi(case):
    f = case.field(8)
    b = to_dev(np.zeros_like(f))
    case.mesh.rhs(to_dev(f), b)
    ref = oracle.dssum(case.ids, (case.Bo * f).ravel(), case.nuniq).reshape(f.shape) * case.mask
    assert rel_l2(to_np(b), ref) <= 1e-12
    h1 = semgen.positive_field(f.shape, 9)
    h2 = semgen.positive_field(f.shape, 10)
    dinv = to_dev(np.zeros_like(f))
    case.mesh.jacobi(dinv, to_dev(h1), to_dev(h2))
    ref = oracle.jacobi(case.N, case.Go, case.Bo, case.ids, case.mask.ravel(), h1=h1, h2=h2,
                        nuniq=case.nuniq).reshape(f.shape)
    assert rel_l2(to_np(dinv), ref) <= 1e-12


@pytest.mark.parametrize("N", [1, 2, 3, 5, 6, 8, 10, 11])
def test_ax_dssum_all_orders(N):
    c = Case("box", N, nel=(3, 3, 3), periodic=(True, False, True), deform=0.1)
    u = c.field(11)
    ref = oracle.ax_dssum(N, c.Go, c.Bo, c.ids, u, mask=c.mask, h1c=1.3, h2c=0.4, nuniq=c.nuniq)
    w = to_dev(np.zeros_like(u))
    c.mesh.ax_dssum(to_dev(u), w, None, None, 1.3, 0.4)
    assert rel_l2(to_np(w), ref) <= 1e-12


def test_topology_errors():
    from paper_2405_05640_b200 import sem
    xi, _ = sem.sem_gll(3)
    m = semgen.box_mesh((2, 3, 3), xi, periodic=(True, True, True))  # 2 elements periodic
    with pytest.raises(sem.SemError) as ei:
        sem.Mesh(m["conn"].shape[0], 3, m["coords"], m["conn"], m["bc"])
    assert ei.value.status == sem.SEM_EINVAL
    m = semgen.box_mesh((1, 1, 1), xi, periodic=(False,) * 3)
    c = m["coords"].copy()
    c[0] = -c[0]
    mesh = sem.Mesh(1, 3, c, m["conn"], m["bc"])
    with pytest.raises(sem.SemError) as ei:
        mesh.geom_factors()
    assert ei.value.status == sem.SEM_EINVAL and "J <= 0" in str(ei.value)


def test_empty_mesh():
    from paper_2405_05640_b200 import sem
    import torch
    mesh = sem.Mesh(0, 4, np.zeros((3, 0, 125)), np.zeros((0, 8), dtype=np.int64), None)
    mesh.geom_factors()
    u = torch.zeros((0, 125), dtype=torch.float64, device="cuda")
    w = torch.zeros((0, 125), dtype=torch.float64, device="cuda")
    mesh.ax_dssum(u, w)
    torch.cuda.synchronize()


def test_ax_dssum_equals_separate_passes():
    """sem_ax_dssum (the operator and one gather-scatter pass, in its own
    schedule) against sem_ax + sem_gs_op(ADD) + sem_gs_op(MASK): bit for bit,
    repeated calls bit-identical, and the oracle's bar; the cylinder at
    lx = 10 (vertices with 6 copies, edges with 3) with walls and Helmholtz
    coefficients."""
    from paper_2405_05640_b200 import sem
    for kind in ("box", "cyl"):
        if kind == "box":
            c = Case("box", 5, nel=(5, 4, 3), periodic=(True, False, True), deform=0.2)
            h1c, h2c = 1.0, 0.0
        else:
            c = Case("cyl", 9, nc=2, nr=1, nz=4)
            h1c, h2c = 0.3, 2.0
        u = c.field(21)
        ref = oracle.ax_dssum(c.N, c.Go, c.Bo, c.ids, u, mask=c.mask, h1c=h1c, h2c=h2c, nuniq=c.nuniq)
        w = to_dev(np.zeros_like(u))
        c.mesh.ax_dssum(to_dev(u), w, h1c=h1c, h2c=h2c)
        w1 = to_np(w)
        c.mesh.ax_dssum(to_dev(u), w, h1c=h1c, h2c=h2c)
        np.testing.assert_array_equal(to_np(w), w1)
        assert rel_l2(w1, ref) <= 1e-12
        w2 = to_dev(u)
        c.mesh.ax(to_dev(u), w2, h1c=h1c, h2c=h2c)
        c.mesh.gs_op(w2, sem.SEM_GS_ADD)
        c.mesh.gs_op(w2, sem.SEM_GS_MASK)
        np.testing.assert_array_equal(w1, to_np(w2))


@pytest.mark.parametrize("deform", [0.0, 0.2])
def test_affine_variant(deform):
    # SURVEY 8(f) f3 (option affine; detection runs when it is set after
    # sem_geom_factors): on an undeformed box every element is affine and the
    # operator uses six metric constants per element; a deformed mesh keeps
    # the general path.  Same bars either way.
    c = Case("box", 7, nel=(4, 3, 5), periodic=(True, False, True), deform=deform,
             lengths=(2.0, 3.0, 1.5))
    c.mesh.set_options(affine=1)
    assert c.mesh.info().affine == (1 if deform == 0.0 else 0)
    u = c.field(31)
    ref = oracle.ax(c.N, c.Go, c.Bo, u, h1c=0.7, h2c=1.3)
    w = to_dev(np.zeros_like(u))
    c.mesh.ax(to_dev(u), w, h1c=0.7, h2c=1.3)
    assert rel_l2(to_np(w), ref) <= 1e-12
    ref = oracle.ax_dssum(c.N, c.Go, c.Bo, c.ids, u, mask=c.mask, nuniq=c.nuniq)
    c.mesh.ax_dssum(to_dev(u), w)
    assert rel_l2(to_np(w), ref) <= 1e-12
    f = c.field(32)
    b = to_dev(np.zeros_like(f))
    c.mesh.rhs(to_dev(f), b)
    x = to_dev(np.zeros_like(f))
    it, _, conv = c.mesh.cg_solve(b, x, tol=1e-10, maxit=500)
    bo = oracle.dssum(c.ids, (c.Bo * f).ravel(), c.nuniq) * c.mask.ravel()
    xo, it_o, _, _ = oracle.pcg(c.N, c.Go, c.Bo, c.ids, bo, mask=c.mask.ravel(), tol=1e-10, maxit=500,
                                nuniq=c.nuniq)
    assert conv and abs(it - it_o) <= 1
    assert rel_l2(to_np(x), xo.reshape(f.shape)) <= 1e-10
