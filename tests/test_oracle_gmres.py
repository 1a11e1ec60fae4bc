"""Pins of the oracle's restarted GMRES (O12; "restarted GMRES
for the pressure solves"; Saad 2003, Alg. 9.5, right preconditioning).

The defining property of GMRES is that its k-th iterate (within a cycle)
minimises the residual over the Krylov space: with M = diag(dinv),
    x_k = x_c + M y,  y in K_k(A M, r_c),  ||r_c - A M y|| minimal,
where x_c, r_c are the cycle's start and the norm is the Euclidean norm on
unique nodes (= the mult-weighted local norm, reading G10).  The pins build
that least-squares problem on the ASSEMBLED unique-node system (P8) with an
orthonormal Krylov basis from numpy's Householder QR -- a different
algorithm from the oracle's modified Gram-Schmidt Arnoldi with Givens
rotations -- and compare iterates:
  * no restart, k = 1..8 (tol = 0 runs exactly maxit = k steps);
  * restart m = 3 over three cycles, each cycle brute-forced from the
    previous cycle's (brute-forced) result;
  * convergence to the direct solution (spsolve) on a walled Helmholtz
    system, and on the singular periodic Poisson system with a non-zero-mean
    right-hand side (projections of b and x, reading G15), where the
    solution must equal the mean-zero least-squares solution;
  * the true relative residual reported, the iteration count equal to the
    brute-force first k with ||r_k|| <= tol ||b|| (the residual estimate of
    the Givens recursion equals the true residual in exact arithmetic).
A dropped rotation, a wrong sign in g, left instead of right
preconditioning, or a missing restart update each fail one of these.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
import semgen
from helpers import assembled, element_matrices, rel_l2, scatter_matrix


def _system(nel, N, periodic, deform, helm):
    xi, _ = oracle.gll(N)
    m = semgen.box_mesh(nel, xi, periodic=periodic, deform=deform)
    G, B = oracle.geom(N, m["coords"])
    ids, nuniq = oracle.lattice_ids(nel, N, periodic)
    mask = oracle.mask_from_bc(N, m["bc"], ids, nuniq)
    h1c, h2c = (1.0, 0.7) if helm else (1.0, 0.0)
    Ae = element_matrices(N, G, B, h1c=h1c, h2c=h2c)
    A = assembled(N, Ae, ids, nuniq)
    first = np.zeros(nuniq, dtype=np.int64)
    first[ids.ravel()[::-1]] = np.arange(ids.size)[::-1]
    keep = mask[first] != 0
    dinv = oracle.jacobi(N, G, B, ids, mask, h1c=h1c, h2c=h2c, nuniq=nuniq)
    return dict(N=N, G=G, B=B, ids=ids, nuniq=nuniq, mask=mask, h1c=h1c, h2c=h2c, A=A, first=first, keep=keep,
                dinv=dinv, Q=scatter_matrix(ids, nuniq))


def _krylov_min(Ak, Mk, r, k):
    """argmin_{y in K_k(A M, r)} ||r - A M y||, returned as M y (numpy QR basis)."""
    AM = Ak @ sp.diags(Mk)
    Qb = (r / np.linalg.norm(r))[:, None]
    for _ in range(k - 1):
        v = AM @ Qb[:, -1]
        Qb, _ = np.linalg.qr(np.column_stack([Qb, v]))
    c, *_ = np.linalg.lstsq(AM @ Qb, r, rcond=None)
    return Mk * (Qb @ c)


def _restrict(s, xl):
    return xl.ravel()[s["first"]][s["keep"]]


def _rhs(s, seed, offset=0.0):
    f = semgen.random_field(s["ids"].shape, seed) + offset
    return oracle.dssum(s["ids"], (s["B"] * f).ravel(), s["nuniq"]) * s["mask"]


def _run(s, b, **kw):
    return oracle.gmres(s["N"], s["G"], s["B"], s["ids"], b, mask=s["mask"], h1c=s["h1c"], h2c=s["h2c"],
                        nuniq=s["nuniq"], dinv=s["dinv"], **kw)


@pytest.fixture(scope="module")
def walled():
    return _system((3, 3, 2), 4, (True, False, False), 0.2, helm=True)


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_iterate_minimises_residual_over_krylov_space(walled, k):
    s = walled
    b = _rhs(s, 41)
    x, it, rr, conv = _run(s, b, tol=0.0, maxit=k, restart=30)
    assert it == k and not conv
    Ak = s["A"][s["keep"]][:, s["keep"]]
    bk, Mk = _restrict(s, b), _restrict(s, s["dinv"])
    xk = _krylov_min(Ak, Mk, bk, k)
    assert rel_l2(_restrict(s, x), xk) <= 1e-10
    # reported residual = the true one
    assert abs(rr - np.linalg.norm(bk - Ak @ xk) / np.linalg.norm(bk)) <= 1e-12


def test_restarted_cycles(walled):
    s = walled
    b = _rhs(s, 42)
    x, it, rr, conv = _run(s, b, tol=0.0, maxit=9, restart=3)
    assert it == 9
    Ak = s["A"][s["keep"]][:, s["keep"]]
    bk, Mk = _restrict(s, b), _restrict(s, s["dinv"])
    xk = np.zeros_like(bk)
    for _ in range(3):
        xk = xk + _krylov_min(Ak, Mk, bk - Ak @ xk, 3)
    assert rel_l2(_restrict(s, x), xk) <= 1e-10
    # and restarts lose to the unrestarted method (minimal over a larger space)
    x30, _, rr30, _ = _run(s, b, tol=0.0, maxit=9, restart=30)
    assert rr30 < rr


def test_converges_to_direct_solution_and_stops_at_first_k(walled):
    s = walled
    b = _rhs(s, 43)
    tol = 1e-9
    x, it, rr, conv = _run(s, b, tol=tol, maxit=500, restart=200)
    assert conv and rr <= 2 * tol
    Ak = s["A"][s["keep"]][:, s["keep"]]
    bk, Mk = _restrict(s, b), _restrict(s, s["dinv"])
    xd = spla.spsolve(Ak.tocsc(), bk)
    assert rel_l2(_restrict(s, x), xd) <= 1e-7
    # the stopping iteration: the first k whose minimal residual is <= tol
    res = []
    for k in range(max(1, it - 2), it + 1):
        xk = _krylov_min(Ak, Mk, bk, k)
        res.append(np.linalg.norm(bk - Ak @ xk) / np.linalg.norm(bk))
    assert res[-1] <= tol * 1.01 and res[-2] > tol * 0.99


def test_singular_periodic_nonzero_mean_rhs():
    s = _system((3, 3, 3), 4, (True,) * 3, 0.2, helm=False)
    b = _rhs(s, 44, offset=0.7)
    x, it, rr, conv = _run(s, b, tol=1e-10, maxit=2000, restart=40)
    assert conv and rr <= 1e-9
    A = s["A"]
    bg = b[s["first"]]
    assert abs(bg.mean()) > 0.01 * np.abs(bg).max()
    bg = bg - bg.mean()
    # mean-zero least-squares solution of the singular system
    xg = spla.lsqr(A, bg, atol=1e-15, btol=1e-15, iter_lim=20000)[0]
    xg -= xg.mean()
    assert rel_l2(x.ravel(), s["Q"] @ xg) <= 1e-7
    mult = oracle.mult(s["ids"], s["nuniq"])
    assert abs(np.sum(mult * x.ravel())) <= 1e-12 * np.sum(mult * np.abs(x.ravel()))


def test_contract_edge_cases(walled):
    s = walled
    z = np.zeros(s["ids"].size)
    x, it, rr, conv = _run(s, z, tol=1e-10, maxit=10)
    assert it == 0 and conv and np.all(x == 0)
    b = _rhs(s, 45)
    x, it, rr, conv = _run(s, b, tol=1e-14, maxit=4, restart=2)
    assert it == 4 and not conv and rr > 0
