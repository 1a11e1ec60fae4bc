"""Pins of the oracle's Jacobi diagonal (O9) and PCG (O10).

P11  dinv = 1/diag of the brute-force assembled matrix (non-affine, variable
     h1/h2, Dirichlet walls), 1 at masked nodes.
P12  PCG iterates = scipy.sparse.linalg.cg on the assembled unique-node system
     with M = diag^{-1} (mult-weighted local dots = Euclidean unique dots):
     same solution (1e-10) and iteration count (+-1).
P13  manufactured solutions (sin on C1, TGV pressure): error decays
     spectrally with N (BASELINE.json north_star: "spectral convergence of CG
     to a manufactured sin/cos solution").
P14  h1 = 0 => A = h2 B is diagonal => Jacobi is exact => 1 iteration.
Contract: b = 0 -> x = 0, iters = 0; maxit reached -> converged = False;
indefinite operator -> breakdown error.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
import semgen
from helpers import assembled, element_matrices, rel_l2, scatter_matrix


def _setup(nel, N, periodic, deform):
    xi, _ = oracle.gll(N)
    m = semgen.box_mesh(nel, xi, periodic=periodic, deform=deform)
    G, B = oracle.geom(N, m["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, periodic)
    mask = oracle.mask_from_bc(N, m["bc"], ids, nuniq)
    return m, G, B, ids, nuniq, mask


def test_jacobi_equals_assembled_diagonal():
    N = 4
    m, G, B, ids, nuniq, mask = _setup((3, 3, 3), N, (True, False, False), 0.2)
    h1 = semgen.positive_field(ids.shape, 11)
    h2 = semgen.positive_field(ids.shape, 12)
    dinv = oracle.jacobi(N, G, B, ids, mask, h1=h1, h2=h2, nuniq=nuniq)
    A = assembled(N, element_matrices(N, G, B, h1=h1, h2=h2), ids, nuniq)
    d = A.diagonal()[ids.ravel()]
    ref = np.where(mask == 0, 1.0, 1.0 / d)
    np.testing.assert_allclose(dinv, ref, rtol=1e-13)


def _scipy_pcg(A, b, dinv_g, tol, maxit):
    its = [0]

    def cb(xk):
        its[0] += 1
    M = sp.diags(dinv_g)
    x, info = spla.cg(A, b, rtol=tol, atol=0.0, maxiter=maxit, M=M, callback=cb)
    return x, its[0]


@pytest.mark.parametrize("case", ["c1_affine", "deformed_helmholtz_walls"])
def test_pcg_equals_scipy_cg(case):
    if case == "c1_affine":
        N, nel, periodic, deform = 7, (4, 4, 4), (True,) * 3, 0.0
    else:
        N, nel, periodic, deform = 4, (3, 3, 3), (True, False, False), 0.2
    m, G, B, ids, nuniq, mask = _setup(nel, N, periodic, deform)
    if case == "c1_affine":
        h1, h2, h1c, h2c = None, None, 1.0, 0.0
        Ae1 = element_matrices(N, G[:1], B[:1])
        Ae = np.broadcast_to(Ae1, (G.shape[0],) + Ae1.shape[1:])
        f = semgen.sin3_source(m["coords"])
    else:
        h1 = semgen.positive_field(ids.shape, 21)
        h2 = semgen.positive_field(ids.shape, 22)
        h1c, h2c = 1.0, 0.0
        Ae = element_matrices(N, G, B, h1=h1, h2=h2)
        f = semgen.random_field(ids.shape, 23)
    A = assembled(N, Ae, ids, nuniq)
    b = oracle.dssum(ids, (B * f).ravel(), nuniq) * mask
    tol = 1e-10
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, b, mask=mask, h1=h1, h2=h2, h1c=h1c, h2c=h2c,
                                    tol=tol, maxit=2000, nuniq=nuniq)
    assert conv and rr <= tol
    # the same system on unique nodes: restrict by picking one copy per node
    Q = scatter_matrix(ids, nuniq)
    first = np.zeros(nuniq, dtype=np.int64)
    first[ids.ravel()[::-1]] = np.arange(ids.size)[::-1]
    bg = b[first]
    keep = mask[first] != 0
    if np.all(keep):  # singular periodic Poisson: project the RHS
        bg = bg - bg.mean()
    Ak = A[keep][:, keep]
    dinv = oracle.jacobi(N, G, B, ids, mask, h1=h1, h2=h2, h1c=h1c, h2c=h2c, nuniq=nuniq)
    xg_k, its = _scipy_pcg(Ak, bg[keep], dinv[first][keep], tol, 2000)
    xg = np.zeros(nuniq)
    xg[keep] = xg_k
    if np.all(keep):
        xg -= xg.mean()
    assert abs(its - iters) <= 1, (its, iters)
    assert rel_l2(x.ravel(), Q @ xg) < 1e-9
    assert rel_l2(x.ravel(), Q @ xg) < 1e-10 or abs(its - iters) == 1


def _solve_manufactured(N, nel, exact, source, deform=0.0):
    m, G, B, ids, nuniq, mask = _setup(nel, N, (True,) * 3, deform)
    f = source(m["coords"])
    b = oracle.dssum(ids, (B * f).ravel(), nuniq)
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, b, tol=1e-12, maxit=3000, nuniq=nuniq)
    assert conv
    ue = exact(m["coords"]).ravel()
    # remove the volume mean from both (singular periodic Poisson, reading G15)
    vol = B.sum()
    x = x.ravel() - np.sum(B.ravel() * x.ravel()) / vol
    ue = ue - np.sum(B.ravel() * ue) / vol
    return np.max(np.abs(x - ue)), iters


@pytest.mark.parametrize("which", ["sin", "tgv"])
def test_manufactured_spectral_convergence(which):
    exact, source = {"sin": (semgen.sin3, semgen.sin3_source),
                     "tgv": (semgen.tgv_pressure, semgen.tgv_source)}[which]
    errs = [_solve_manufactured(N, (4, 4, 4), exact, source)[0] for N in (3, 5, 7)]
    # log-linear (spectral) decay: each +2 in N gains > 1.5 orders here
    assert errs[0] > 30 * errs[1] > 30 * 30 * errs[2] * 0.03
    assert errs[2] < 1e-5
    assert np.all(np.diff(np.log10(errs)) < -1.0)


def test_manufactured_deformed():
    e5, _ = _solve_manufactured(5, (4, 4, 4), semgen.sin3, semgen.sin3_source, deform=0.2)
    e7, _ = _solve_manufactured(7, (4, 4, 4), semgen.sin3, semgen.sin3_source, deform=0.2)
    assert e7 < e5 / 10 and e7 < 1e-3


def test_h1_zero_one_iteration():
    # P14
    N = 4
    m, G, B, ids, nuniq, mask = _setup((3, 3, 3), N, (True,) * 3, 0.2)
    b = oracle.dssum(ids, (B * semgen.random_field(ids.shape, 5)).ravel(), nuniq)
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, b, h1c=0.0, h2c=2.0, tol=1e-12, nuniq=nuniq)
    assert conv and iters == 1
    # exact solution of the diagonal system: x = b / (2 * dssum(B))
    Bg = oracle.dssum(ids, B.ravel(), nuniq)
    np.testing.assert_allclose(x.ravel(), b / (2.0 * Bg), rtol=1e-13)


def test_contract_edge_cases():
    N = 3
    m, G, B, ids, nuniq, mask = _setup((3, 3, 3), N, (False,) * 3, 0.0)
    z = np.zeros(ids.size)
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, z, mask=mask, tol=1e-10, nuniq=nuniq)
    assert iters == 0 and conv and np.all(x == 0)
    b = oracle.dssum(ids, (B * semgen.random_field(ids.shape, 9)).ravel(), nuniq) * mask
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, b, mask=mask, tol=1e-14, maxit=2, nuniq=nuniq)
    assert iters == 2 and not conv and rr > 0
    with pytest.raises(oracle.OracleError) as ei:
        oracle.pcg(N, G, B, ids, b, mask=mask, h1c=1.0, h2c=-1e4, tol=1e-10, nuniq=nuniq)
    assert ei.value.status == oracle.OR_EBREAKDOWN
    # tol = 0: fixed iteration count
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, b, mask=mask, tol=0.0, maxit=7, nuniq=nuniq)
    assert iters == 7 and not conv


def _unique_system(N, G, B, ids, nuniq, mask, h1=None, h2=None, h1c=1.0, h2c=0.0):
    """The assembled unique-node system (P8) and the restriction picking one
    copy per unique node."""
    if h1 is None and h2 is None:
        Ae = element_matrices(N, G, B, h1c=h1c, h2c=h2c)
    else:
        Ae = element_matrices(N, G, B, h1=h1, h2=h2)
    A = assembled(N, Ae, ids, nuniq)
    first = np.zeros(nuniq, dtype=np.int64)
    first[ids.ravel()[::-1]] = np.arange(ids.size)[::-1]
    return A, first


def test_singular_random_rhs_equals_scipy_exactly():
    """O10's singular branch (reading G15) pinned with a right-hand side whose
    weighted mean is NOT zero: b = dssum(B f), f ~ U(-1,1) + 0.7 on a deformed
    periodic Poisson box.  Reference: scipy's CG on the assembled unique-node
    system (P8), with b projected onto the mean-zero space of unique nodes and
    the solution projected the same way.

    The tolerance is chosen half-way (geometrically) between two consecutive
    scipy residuals, so the stopping iteration is not borderline and must be
    EXACTLY equal; the oracle's reported rel_res (its mult-weighted recursive
    residual over its mult-weighted ||b||) must equal scipy's true unique-node
    residual ||b - A x|| / ||b|| to 1e-12.  A dropped projection of b (CG on
    an inconsistent system), of x (a constant offset), or an unweighted
    stopping norm (different rel_res, different stop) each fail here."""
    N = 4
    m, G, B, ids, nuniq, mask = _setup((3, 3, 4), N, (True,) * 3, 0.2)
    f = semgen.random_field(ids.shape, 91) + 0.7
    b = oracle.dssum(ids, (B * f).ravel(), nuniq)
    A, first = _unique_system(N, G, B, ids, nuniq, mask)
    bg = b[first]
    assert abs(bg.mean()) > 0.01 * np.abs(bg).max()  # genuinely non-mean-zero
    bg = bg - bg.mean()
    dinv = oracle.jacobi(N, G, B, ids, mask, nuniq=nuniq)
    M = sp.diags(dinv[first])
    hist = []

    def cb(xk):
        hist.append(np.linalg.norm(bg - A @ xk) / np.linalg.norm(bg))
    spla.cg(A, bg, rtol=1e-13, atol=0.0, maxiter=5000, M=M, callback=cb)
    hist = np.array(hist)
    k = int(np.argmax(hist < 1e-8))  # first iterate (0-based) below 1e-8
    assert k > 5 and hist[k] < 1e-8 <= hist[k - 1]
    tol = math.sqrt(hist[k] * hist[k - 1])
    assert hist[k - 1] > 1.05 * tol and hist[k] < tol / 1.05  # not borderline
    its = [0]

    def cb2(xk):
        its[0] += 1
    xg, info = spla.cg(A, bg, rtol=tol, atol=0.0, maxiter=5000, M=M, callback=cb2)
    assert info == 0 and its[0] == k + 1
    rr_scipy = np.linalg.norm(bg - A @ xg) / np.linalg.norm(bg)
    xg = xg - xg.mean()
    x, iters, rr, conv = oracle.pcg(N, G, B, ids, b, tol=tol, maxit=5000, nuniq=nuniq)
    assert conv and iters == k + 1, (iters, k + 1)
    assert abs(rr - rr_scipy) <= 1e-12, (rr, rr_scipy)
    Q = scatter_matrix(ids, nuniq)
    assert rel_l2(x.ravel(), Q @ xg) <= 1e-10
    # the oracle's x is mean-zero on unique nodes
    mult = oracle.mult(ids, nuniq)
    assert abs(np.sum(mult * x.ravel())) <= 1e-12 * np.sum(mult * np.abs(x.ravel()))
