"""Pins of the oracle's geometry (O4), local operator (O5), dssum (O7) and
numbering (O6).

P5  affine element = textbook Kronecker sum (M x M x K + ...);
P6  sum B = volume; J > 0;
P7  Poisson A 1 = 0, symmetry u^T A v = v^T A u, PSD;
P8  assembled A = Q^T blockdiag(A_e) Q equals the textbook 3D Kronecker sum of
    assembled 1D GLL matrices on box meshes (periodic and walled), and
    Q (A u_g) = dssum(ax(Q u_g));
    deformed meshes: the energy u^T A u and the mass u^T B u converge
    spectrally to the exact integrals (the deformation maps the periodic box
    onto itself, so the exact values are those of the undeformed box).
"""
import math

import numpy as np
import pytest

import oracle
import semgen
from helpers import (assembled, bary_D, element_matrices, rel_l2, scatter_matrix,
                     scipy_gll, textbook_1d)


def _box(nel, N, periodic=(True, True, True), deform=0.0, lengths=(2 * math.pi,) * 3):
    xi, _ = oracle.gll(N)
    return semgen.box_mesh(nel, xi, lengths=lengths, periodic=periodic, deform=deform)


def test_affine_element_kronecker():
    # P5: hx x hy x hz box element, A_e = (hy hz/(2hx)) M(x)M(x)K + ... with
    # Kronecker order (k (x) j (x) i), M = diag(w), K = D^T W D
    N = 5
    hx, hy, hz = 0.7, 1.3, 0.4
    m = _box((1, 1, 1), N, periodic=(False,) * 3, lengths=(hx, hy, hz))
    G, B = oracle.geom(N, m["coords"])
    Ae = element_matrices(N, G, B)[0]
    xs, ws = scipy_gll(N)
    Dind = bary_D(xs)
    M = np.diag(ws)
    K = Dind.T @ M @ Dind
    ref = (hy * hz / (2 * hx)) * np.kron(M, np.kron(M, K)) \
        + (hx * hz / (2 * hy)) * np.kron(M, np.kron(K, M)) \
        + (hx * hy / (2 * hz)) * np.kron(K, np.kron(M, M))
    assert np.max(np.abs(Ae - ref)) < 1e-12 * np.max(np.abs(ref))
    # geometric factors of an affine box: G11 = w_i w_j w_k hy hz/(2 hx), G12 = 0
    W3 = np.einsum("k,j,i->kji", ws, ws, ws).ravel()
    np.testing.assert_allclose(G[0, 0], W3 * hy * hz / (2 * hx), rtol=1e-13)
    np.testing.assert_allclose(G[0, 3:], 0.0, atol=1e-15)
    np.testing.assert_allclose(B[0], W3 * hx * hy * hz / 8, rtol=1e-13)


@pytest.mark.parametrize("deform", [0.0, 0.2])
def test_volume_and_jacobian(deform):
    # P6: sum B = volume (exact for affine; spectral for the deformed torus map)
    N = 9 if deform else 4
    m = _box((3, 3, 3), N, deform=deform)
    G, B = oracle.geom(N, m["coords"])
    assert np.all(B > 0)
    vol = (2 * math.pi) ** 3
    assert abs(B.sum() - vol) / vol < (1e-14 if deform == 0 else 1e-6)


def test_cylinder_volume():
    # P6: sum B -> pi R^2 H = pi/4 spectrally on the O-grid cylinder
    errs = []
    for N in (2, 4, 6):
        xi, _ = oracle.gll(N)
        m = semgen.cylinder_mesh(xi, nc=2, nr=1, nz=2)
        G, B = oracle.geom(N, m["coords"])
        assert np.all(B > 0)
        errs.append(abs(B.sum() - math.pi / 4))
    assert errs[2] < 1e-6 and errs[2] < errs[1] < errs[0]


def test_negative_jacobian_rejected():
    N = 3
    m = _box((1, 1, 1), N, periodic=(False,) * 3)
    c = m["coords"].copy()
    c[0] = -c[0]  # mirror: J < 0
    with pytest.raises(oracle.OracleError):
        oracle.geom(N, c)


@pytest.mark.parametrize("deform", [0.0, 0.2])
def test_poisson_invariants(deform):
    # P7: A 1 = 0 per element; symmetric; PSD
    N = 4
    m = _box((3, 3, 3), N, deform=deform)
    G, B = oracle.geom(N, m["coords"])
    E = G.shape[0]
    n3 = (N + 1) ** 3
    w1 = oracle.ax(N, G, B, np.ones((E, n3)))
    assert np.max(np.abs(w1)) < 1e-12 * np.max(np.abs(G))
    rng = np.random.default_rng(7)
    u, v = rng.standard_normal((2, E, n3))
    Au, Av = oracle.ax(N, G, B, u), oracle.ax(N, G, B, v)
    assert abs(np.sum(v * Au) - np.sum(u * Av)) < 1e-12 * np.sum(np.abs(v * Au))
    Ae = element_matrices(N, G[:3], B[:3])
    for A in Ae:
        assert np.max(np.abs(A - A.T)) < 1e-12 * np.max(np.abs(A))
        assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > -1e-12 * np.max(np.abs(A))


@pytest.mark.parametrize("periodic", [(True, True, True), (False, False, False),
                                      (True, False, True)])
def test_assembled_equals_textbook_kronecker(periodic):
    # P8: brute-force global matrix Q^T blockdiag(A_e) Q on a small box equals
    # Kx (x) My (x) Mz + Mx (x) Ky (x) Mz + Mx (x) My (x) Kz of textbook 1D
    # assembled GLL matrices (independent nodes/weights/D from scipy/barycentric)
    N = 3
    nel = (3, 3, 3)
    L = (2.0, 3.0, 1.5)
    m = _box(nel, N, periodic=periodic, lengths=L)
    G, B = oracle.geom(N, m["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, periodic)
    Ae = element_matrices(N, G, B, h1c=1.0, h2c=0.0)
    A = assembled(N, Ae, ids, nuniq).toarray()
    xs, ws = scipy_gll(N)
    Dind = bary_D(xs)
    Ks, Ms = [], []
    for a in range(3):
        K1, M1 = textbook_1d(N, L[a] / nel[a], nel[a], periodic[a], xs, ws, Dind)
        Ks.append(K1)
        Ms.append(M1)
    # lattice id = I + nx (J + ny K)  ->  Kronecker order (z (x) y (x) x)
    ref = np.kron(Ms[2], np.kron(Ms[1], Ks[0])) + np.kron(Ms[2], np.kron(Ks[1], Ms[0])) \
        + np.kron(Ks[2], np.kron(Ms[1], Ms[0]))
    assert np.max(np.abs(A - ref)) < 1e-12 * np.max(np.abs(ref))
    # mass: h2 B assembled = Mz (x) My (x) Mx (diagonal)
    Bg = np.bincount(ids.ravel(), weights=B.ravel(), minlength=nuniq)
    np.testing.assert_allclose(Bg, np.diag(np.kron(Ms[2], np.kron(Ms[1], Ms[0]))), rtol=1e-13)


@pytest.mark.parametrize("deform", [0.0, 0.2])
def test_dssum_is_QQt(deform):
    # P8: dssum(ax(Q u_g)) = Q (A u_g) with A = Q^T blockdiag(A_e) Q
    N = 3
    nel = (3, 3, 3)
    m = _box(nel, N, deform=deform)
    G, B = oracle.geom(N, m["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, (True,) * 3)
    h1 = semgen.positive_field(ids.shape, 3)
    h2 = semgen.positive_field(ids.shape, 4)
    Ae = element_matrices(N, G, B, h1=h1, h2=h2)
    A = assembled(N, Ae, ids, nuniq)
    Q = scatter_matrix(ids, nuniq)
    ug = np.random.default_rng(1).standard_normal(nuniq)
    lhs = oracle.ax_dssum(N, G, B, ids, (Q @ ug).reshape(ids.shape), h1=h1, h2=h2)
    rhs = Q @ (A @ ug)
    assert rel_l2(lhs, rhs) < 1e-14
    # dssum itself: v_g = sum of copies, scattered back
    u = np.random.default_rng(2).standard_normal(ids.size)
    np.testing.assert_allclose(oracle.dssum(ids, u), Q @ (Q.T @ u), rtol=1e-14, atol=1e-14)


def test_deformed_energy_spectral():
    # P8 (deformed): u = sin x on the deformed periodic box.  u^T A u ->
    # int |grad u|^2 = int cos^2 x = 4 pi^3 and u^T B u -> int sin^2 x = 4 pi^3
    # (the deformation maps the 2pi-torus onto itself, so the exact integrals
    # are the undeformed ones); errors decay spectrally with N.
    errs = []
    for N in (3, 5, 7, 9):
        nel = (3, 3, 3)
        m = _box(nel, N, deform=0.2)
        G, B = oracle.geom(N, m["coords"])
        ids, nuniq = oracle.lattice_ids(nel, N, (True,) * 3)
        u = np.sin(m["coords"][0])
        Au = oracle.ax_dssum(N, G, B, ids, u)
        mlt = oracle.mult(ids, nuniq).reshape(u.shape)
        energy = np.sum(mlt * u * Au)
        mass = np.sum(B * u * u)
        errs.append((abs(energy - 4 * math.pi ** 3), abs(mass - 4 * math.pi ** 3)))
    e = np.array(errs)
    assert e[-1, 0] < 1e-5 * 4 * math.pi ** 3 and e[-1, 1] < 1e-5 * 4 * math.pi ** 3
    assert np.all(np.diff(np.log(e[:, 0])) < 0)
