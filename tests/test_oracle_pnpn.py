"""Pins of the oracle's time-step operators (O13-O17):
metric terms, collocation gradient, weak divergence, convection and one
first-order velocity-pressure splitting step (Karniadakis et
al. 1991; the TGV case PAPER.md:96).

* the weak divergence applied to the (unweighted) collocation gradient of phi
  IS the local stiffness A_e phi of O5 (G_ab = sum_m MJ_am dr_b/dx_m): an
  exact identity tying O13-O15 to the pinned operator;
* grad and wdiv are discrete adjoints: sum f.grad(p) = sum p wdiv(f);
* on an affine box the gradient of a linear field is exact, and sum_p MJ_am
  over an element = the element volume times dr_a/dx_m;
* the 2D Taylor-Green field u = (sin x cos y, -cos x sin y, 0) is an exact
  Navier-Stokes solution whose convection is a pressure gradient,
  (u.grad)u = -grad p_e with p_e = (cos 2x + cos 2y)/4: the oracle's
  convection equals -grad p_e to spectral accuracy, and one splitting step
  returns u/(1 + 2 nu dt) (the BDF1 decay of the viscous term, -Lap u = 2u)
  with p = p_e up to a constant, and a weakly divergence-free velocity.
"""
import numpy as np
import pytest

import oracle
import semgen
from helpers import rel_l2

TWO_PI = 2 * np.pi


def _mesh(nel, N, deform, periodic=(True, True, True)):
    xi, _ = oracle.gll(N)
    m = semgen.box_mesh(nel, xi, periodic=periodic, deform=deform)
    G, B = oracle.geom(N, m["coords"])
    MJ = oracle.metrics(N, m["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, periodic)
    return m, G, B, MJ, ids.reshape(G.shape[0], -1), nuniq


def test_wdiv_of_gradient_is_stiffness():
    N = 5
    m, G, B, MJ, ids, nuniq = _mesh((2, 3, 2), N, 0.2, periodic=(False,) * 3)
    phi = semgen.random_field(B.shape, 3)
    g = oracle.grad(N, MJ, phi)          # W J grad phi
    f = g / B[None]                       # the collocation gradient itself
    lhs = oracle.wdiv(N, MJ, f)
    ref = oracle.ax(N, G, B, phi)         # O5 with h1 = 1, h2 = 0
    assert rel_l2(lhs, ref) <= 1e-13


def test_grad_and_wdiv_are_adjoint():
    N = 4
    m, G, B, MJ, ids, nuniq = _mesh((3, 2, 2), N, 0.2)
    p = semgen.random_field(B.shape, 4)
    f = semgen.random_field((3,) + B.shape, 5)
    a = np.sum(f * oracle.grad(N, MJ, p))
    b = np.sum(p * oracle.wdiv(N, MJ, f))
    assert abs(a - b) <= 1e-12 * (abs(a) + np.sum(np.abs(f)))


def test_affine_gradient_exact_and_metric_sums():
    N = 3
    lengths = (2.0, 3.0, 5.0)
    xi, _ = oracle.gll(N)
    m = semgen.box_mesh((2, 2, 2), xi, periodic=(False,) * 3, lengths=lengths)
    G, B = oracle.geom(N, m["coords"])
    MJ = oracle.metrics(N, m["coords"])
    x, y, z = m["coords"]
    phi = 0.5 * x - 2.0 * y + 3.0 * z + 1.0
    g = oracle.grad(N, MJ, phi)
    for mm, c in enumerate((0.5, -2.0, 3.0)):
        assert np.allclose(g[mm], c * B, rtol=0, atol=1e-12)
    # sum over an element of W J dr_a/dx_m = volume * (2 / h_m) delta_am
    vol = np.prod([L / 2 for L in lengths])
    for a in range(3):
        for mm in range(3):
            s = MJ[0, a, mm].sum()
            ref = vol * (2.0 / (lengths[a] / 2)) if a == mm else 0.0
            assert abs(s - ref) <= 1e-12 * vol


def _tgv2d(coords):
    x, y, z = coords
    u = np.stack([np.sin(x) * np.cos(y), -np.cos(x) * np.sin(y), 0.0 * z])
    pe = (np.cos(2 * x) + np.cos(2 * y)) / 4.0
    return u, pe


@pytest.mark.parametrize("deform", [0.0, 0.15])
def test_tgv_convection_is_pressure_gradient(deform):
    # spectral convergence of W J (u.grad)u + W J grad p_e -> 0 with N
    errs = []
    for N in (5, 7, 9):
        m, G, B, MJ, ids, nuniq = _mesh((4, 4, 3), N, deform)
        u, pe = _tgv2d(m["coords"].reshape(3, *B.shape))
        c = oracle.convect(N, MJ, u.reshape(3, *B.shape))
        gp = oracle.grad(N, MJ, pe.reshape(B.shape))
        errs.append(rel_l2(c, -gp))
    assert errs[0] > 30 * errs[1] > 30 * 30 * errs[2] and errs[2] < 1e-6


def test_pnpn_step_tgv2d():
    N = 7
    nu, dt = 0.05, 0.01
    m, G, B, MJ, ids, nuniq = _mesh((4, 4, 3), N, 0.0)
    u, pe = _tgv2d(m["coords"].reshape(3, *B.shape))
    un, p, itp, itv = oracle.pnpn_step(N, G, B, MJ, ids, u, dt, nu, nuniq=nuniq)
    assert rel_l2(un, u / (1.0 + 2.0 * nu * dt)) <= 1e-6
    pm = p - np.sum(B * p) / B.sum()
    pem = pe.reshape(B.shape) - np.sum(B * pe.reshape(B.shape)) / B.sum()
    assert rel_l2(pm, pem) <= 1e-5
    # weakly divergence-free: the assembled (grad v, u) is ~0 against its size
    d = oracle.dssum(ids, oracle.wdiv(N, MJ, un).ravel(), nuniq)
    dref = oracle.dssum(ids, oracle.wdiv(N, MJ, np.stack([un[0], 0 * un[1], 0 * un[2]])).ravel(), nuniq)
    assert np.linalg.norm(d) <= 1e-5 * np.linalg.norm(dref)
    assert itp > 0 and all(k > 0 for k in itv)
