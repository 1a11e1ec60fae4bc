"""Pins of the oracle's hybrid-Schwarz multigrid preconditioner and FGMRES
(oracle/hsmg.py, "restarted GMRES for the
pressure solves with a hybrid-Schwarz multigrid preconditioner"; reading R16
in DESIGN.md).  Each piece is fixed by something other than itself:

  * Lagrange transfer matrices: exact on polynomials of the coarse degree,
    identity on equal nodes (mathematics of interpolation);
  * the extended 1-D operators = the principal submatrix, on one element's
    nodes, of the textbook assembled 1-D GLL stiffness/mass of a uniform
    3-element grid (helpers.textbook_1d) -- the "neighbour's share" reading;
  * the generalised eigenpairs: S^T B S = I, S^T A S = diag(mu);
  * the fast-diagonalisation local solve = a dense solve with the explicit
    Kronecker-sum matrix (brute force, np.kron);
  * on a uniform periodic box the separable local operator IS the principal
    submatrix of the assembled 3-D operator (built from oracle.ax on unit
    vectors, P8), Poisson and Helmholtz -- this pins the length scaling;
  * the averaged additive Schwarz smoother = the dense sum of principal-
    submatrix inverses over elements divided by the multiplicity;
  * prolongation: continuous in, continuous out, exact for a global
    polynomial of the coarse degree on an affine box;
  * restriction = adjoint of prolongation on unique nodes;
  * R A_f P = the exactly integrated coarse stiffness (textbook 1-D
    stiffness and Gauss-Legendre consistent mass, Kronecker-assembled);
  * the V-cycle: with an exact coarse solve its error propagation is the
    two-level product (I - P A_c^-1 R A)(I - S A) (dense matrices);
  * FGMRES with the Jacobi preconditioner = the C oracle's GMRES (two
    independent implementations, same iterations, x to 1e-12);
  * FGMRES + HSMG converges to the direct solution with far fewer iterations
    than Jacobi.
"""
import numpy as np
import pytest

import oracle
import semgen
from helpers import assembled, element_matrices, rel_l2, textbook_1d
from oracle import hsmg as H


def _box(nel, N, periodic, deform=0.0, lengths=None):
    xi, _ = oracle.gll(N)
    kw = {} if lengths is None else {"lengths": lengths}
    m = semgen.box_mesh(nel, xi, periodic=periodic, deform=deform, **kw)
    ids_fn = lambda Nl, c: oracle.lattice_ids(nel, Nl, periodic)  # noqa: E731
    return m, H.setup(N, m["coords"], m["bc"], ids_fn)


# ---- 1-D pieces ----------------------------------------------------------------

@pytest.mark.parametrize("nf,nc", [(7, 3), (9, 4), (4, 1), (3, 3)])
def test_lagrange_matrix_exact_on_coarse_polynomials(nf, nc):
    xc, _ = oracle.gll(nc)
    xf, _ = oracle.gll(nf)
    J = H.lagrange_matrix(xc, xf)
    for deg in range(nc + 1):
        assert np.allclose(J @ xc ** deg, xf ** deg, atol=1e-13, rtol=0)
    if nf == nc:
        assert np.allclose(J, np.eye(nf + 1), atol=1e-14)


@pytest.mark.parametrize("N", [1, 2, 3, 5, 8])
def test_extended_1d_operator_is_principal_submatrix(N):
    xi, w = oracle.gll(N)
    D = oracle.dmat(N, xi)
    K, M = textbook_1d(N, 2.0, 3, False, xi, w, D)  # three elements of length 2
    idx = np.arange(N, 2 * N + 1)  # the middle element's nodes
    Ae, Be, S, mu = H.fdm_1d(N)
    assert np.allclose(Ae, K[np.ix_(idx, idx)], atol=1e-12)
    assert np.allclose(Be, M[np.ix_(idx, idx)], atol=1e-14)
    assert np.allclose(S.T @ Be @ S, np.eye(N + 1), atol=1e-12)
    assert np.allclose(S.T @ Ae @ S, np.diag(mu), atol=1e-10 * max(1.0, mu.max()))
    assert mu.min() > 0  # Dirichlet one node outside: non-singular


@pytest.mark.parametrize("N", [1, 2, 4])
def test_fdm_solve_equals_dense_kronecker_solve(N):
    lx = N + 1
    rng = np.random.default_rng(7)
    L = rng.uniform(0.3, 2.0, (3, 3))
    r = rng.uniform(-1, 1, (3, lx ** 3))
    Ae, Be, _, _ = H.fdm_1d(N)
    for h1c, h2c in ((1.0, 0.0), (0.7, 2.5)):
        z = H.fdm_local_solve(N, L, r, h1c, h2c)
        for e in range(3):
            A1 = [(2.0 / L[e, d]) * Ae for d in range(3)]
            B1 = [(L[e, d] / 2.0) * Be for d in range(3)]
            # node i + lx j + lx^2 k: kron(z-factor, y-factor, x-factor)
            At = (h1c * (np.kron(B1[2], np.kron(B1[1], A1[0])) + np.kron(B1[2], np.kron(A1[1], B1[0]))
                         + np.kron(A1[2], np.kron(B1[1], B1[0])))
                  + h2c * np.kron(B1[2], np.kron(B1[1], B1[0])))
            assert rel_l2(z[e], np.linalg.solve(At, r[e])) <= 1e-12


@pytest.mark.parametrize("h2c", [0.0, 0.9])
def test_local_operator_is_principal_submatrix_of_assembled_3d(h2c):
    nel, N = (3, 3, 3), 2
    lengths = (1.5, 2.4, 3.3)  # elements 0.5 x 0.8 x 1.1
    m, levels = _box(nel, N, (True, True, True), lengths=lengths)
    lev = levels[0]
    assert np.allclose(lev["L"], [[0.5, 0.8, 1.1]] * 27, atol=1e-14)
    h1c = 1.3
    Ae = element_matrices(N, lev["G"], lev["B"], h1c=h1c, h2c=h2c)
    A = assembled(N, Ae, lev["ids"], lev["nuniq"]).toarray()
    ide = lev["ids"].reshape(27, -1)[13]  # an element; all its ids distinct
    assert len(set(ide)) == ide.size
    Asub = A[np.ix_(ide, ide)]
    n3 = ide.size
    # dense local operator from the FDM solve: columns of A~^-1
    Ainv = H.fdm_local_solve(N, lev["L"][13:14].repeat(n3, 0), np.eye(n3), h1c, h2c).T
    assert rel_l2(Ainv @ Asub, np.eye(n3)) <= 1e-11


def test_schwarz_is_averaged_sum_of_principal_submatrix_solves():
    """On a uniform periodic box: S = diag(1/m) sum_e R_e^T (A|_e)^-1 R_e with
    A|_e the principal submatrix of the assembled operator on element e's
    unique nodes (dense brute force)."""
    nel, N = (3, 3, 3), 2
    m, levels = _box(nel, N, (True, True, True), lengths=(1.5, 2.4, 3.3))
    lev = levels[0]
    h1c, h2c = 0.8, 0.3
    Ae = element_matrices(N, lev["G"], lev["B"], h1c=h1c, h2c=h2c)
    A = assembled(N, Ae, lev["ids"], lev["nuniq"]).toarray()
    nu = lev["nuniq"]
    ids = lev["ids"].reshape(27, -1)
    S = np.zeros((nu, nu))
    for e in range(27):
        g = ids[e]
        S[np.ix_(g, g)] += np.linalg.inv(A[np.ix_(g, g)])
    cnt = np.bincount(lev["ids"], minlength=nu)
    S = S / cnt[:, None]
    Sd, first, keep = _dense(lambda v: H.schwarz(lev, v, h1c, h2c), lev)
    assert keep.all()
    assert rel_l2(Sd, S) <= 1e-11


def test_element_lengths():
    m, levels = _box((3, 4, 3), 3, (True, False, True), lengths=(3.0, 2.0, 6.0))
    assert np.allclose(levels[0]["L"], [[1.0, 0.5, 2.0]], atol=1e-14)
    for lev in levels:  # same corners at every level
        assert np.allclose(lev["L"], levels[0]["L"], atol=1e-14)


# ---- transfers and level operators --------------------------------------------------

def test_level_orders():
    assert H.level_orders(7) == [7, 3, 1]
    assert H.level_orders(9) == [9, 4, 1]
    assert H.level_orders(3) == [3, 1]
    assert H.level_orders(2) == [2, 1]
    assert H.level_orders(1) == [1]


def test_prolongation_exact_and_continuous():
    m, levels = _box((3, 3, 3), 6, (False, False, False))
    f, c = levels[0], levels[1]  # orders 6 and 3
    X = c["coords"]
    u = (X[0] ** 3 - 2 * X[1] * X[2] ** 2 + X[0] * X[1]).reshape(-1)  # degree 3
    Pu = H.prolong(f, u)
    Xf = f["coords"]
    assert rel_l2(Pu, (Xf[0] ** 3 - 2 * Xf[1] * Xf[2] ** 2 + Xf[0] * Xf[1]).reshape(-1)) <= 1e-13
    # a continuous random coarse field stays continuous
    uc = oracle.dssum(c["ids"], semgen.random_field(c["ids"].size, 5), c["nuniq"]) * c["mult"]
    uf = H.prolong(f, uc)
    assert rel_l2(oracle.dssum(f["ids"], uf, f["nuniq"]) * f["mult"], uf) <= 1e-14


@pytest.mark.parametrize("periodic", [(True, True, True), (True, False, False)])
def test_restriction_is_adjoint_of_prolongation(periodic):
    m, levels = _box((3, 3, 3), 5, periodic, deform=0.15)
    for l in range(len(levels) - 1):
        f, c = levels[l], levels[l + 1]
        uc = oracle.dssum(c["ids"], semgen.random_field(c["ids"].size, 11 + l), c["nuniq"]) * c["mult"]
        if c["mask"] is not None:
            uc = uc * c["mask"]
        rf = oracle.dssum(f["ids"], semgen.random_field(f["ids"].size, 21 + l), f["nuniq"])
        if f["mask"] is not None:
            rf = rf * f["mask"]
        lhs = np.sum(f["mult"] * H.prolong(f, uc) * rf)  # unique-node dot
        rhs = np.sum(c["mult"] * uc * H.restrict(f, c, rf))
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


@pytest.mark.parametrize("N", [4, 6])
def test_galerkin_product_is_exact_coarse_stiffness(N):
    """R A_f P on a uniform periodic box = the EXACTLY integrated stiffness of
    the coarse space (the fine GLL rule integrates degree-2N_c products
    exactly), built from textbook 1-D matrices: the GLL stiffness (exact) and
    the consistent mass by Gauss-Legendre quadrature, assembled periodic and
    combined as kron(M, M, K) + kron(M, K, M) + kron(K, M, M)."""
    nel, lengths = (3, 3, 3), (3.0, 4.5, 6.0)
    m, levels = _box(nel, N, (True, True, True), lengths=lengths)
    f, c = levels[0], levels[1]
    Nc = c["N"]
    xc, wc = oracle.gll(Nc)
    Dc = oracle.dmat(Nc, xc)
    gx, gw = np.polynomial.legendre.leggauss(Nc + 2)
    Lg = H.lagrange_matrix(xc, gx)  # basis at Gauss points
    K1, M1 = [], []
    for d in range(3):
        h = lengths[d] / 3
        K, _ = textbook_1d(Nc, h, 3, True, xc, wc, Dc)
        Me = (h / 2) * Lg.T @ np.diag(gw) @ Lg
        M = np.zeros_like(K)
        n = 3 * Nc
        for e in range(3):
            idx = [(e * Nc + i) % n for i in range(Nc + 1)]
            M[np.ix_(idx, idx)] += Me
        K1.append(K)
        M1.append(M)
    Aex = (np.kron(M1[2], np.kron(M1[1], K1[0])) + np.kron(M1[2], np.kron(K1[1], M1[0]))
           + np.kron(K1[2], np.kron(M1[1], M1[0])))
    RAP, first, keep = _dense(lambda v: H.restrict(f, c, H.level_ax(f, H.prolong(f, v))), c)
    assert keep.all()
    assert rel_l2(RAP, Aex) <= 1e-12


# ---- the V-cycle ------------------------------------------------------------------------

def _dense(op, lev):
    """Matrix of a linear map on unique nodes (first copies), masked nodes dropped."""
    ids, nuniq, mult = lev["ids"], lev["nuniq"], lev["mult"]
    first = np.zeros(nuniq, dtype=np.int64)
    first[ids[::-1]] = np.arange(ids.size)[::-1]
    keep = np.ones(nuniq, bool) if lev["mask"] is None else lev["mask"][first] != 0
    cols = []
    for g in np.nonzero(keep)[0]:
        e = (ids == g).astype(np.float64)
        cols.append(op(e)[first][keep])
    return np.array(cols).T, first, keep


def test_vcycle_is_two_level_product_with_exact_coarse_solve():
    nel, N = (3, 3, 3), 3  # two levels: orders 3 and 1
    m, levels = _box(nel, N, (False, False, True), deform=0.1)
    f, c = levels
    h1c, h2c = 1.0, 0.0
    Af, first_f, keep_f = _dense(lambda v: H.level_ax(f, v, h1c, h2c), f)
    Sf, _, _ = _dense(lambda v: H.schwarz(f, v, h1c, h2c), f)
    Ac, first_c, keep_c = _dense(lambda v: H.level_ax(c, v, h1c, h2c), c)
    # P and R as matrices between kept unique nodes
    P = np.zeros((keep_f.sum(), keep_c.sum()))
    for j, g in enumerate(np.nonzero(keep_c)[0]):
        P[:, j] = H.prolong(f, (c["ids"] == g).astype(np.float64))[first_f][keep_f]
    R = np.zeros((keep_c.sum(), keep_f.sum()))
    for j, g in enumerate(np.nonzero(keep_f)[0]):
        R[:, j] = H.restrict(f, c, (f["ids"] == g).astype(np.float64))[first_c][keep_c]
    assert np.allclose(R, P.T, atol=1e-13)
    n = keep_f.sum()
    Eexp = (np.eye(n) - P @ np.linalg.solve(Ac, R @ Af)) @ (np.eye(n) - Sf @ Af)
    # M from the V-cycle (the coarse PCG converges on this small level)
    Mv, _, _ = _dense(lambda v: H.vcycle(levels, v, h1c, h2c, coarse_iters=500), f)
    # vcycle takes an assembled residual: its columns are M applied to e_g
    assert rel_l2(np.eye(n) - Mv @ Af, Eexp) <= 1e-9


# ---- FGMRES -------------------------------------------------------------------------------

@pytest.mark.parametrize("periodic,helm", [((True, True, True), False), ((True, False, False), True)])
def test_fgmres_jacobi_equals_c_gmres(periodic, helm):
    N, nel = 4, (3, 3, 3)
    m, levels = _box(nel, N, periodic, deform=0.15)
    lev = levels[0]
    h2c = 0.6 if helm else 0.0
    f = semgen.random_field(lev["ids"].size, 3) + 0.4  # non-mean-zero
    b = oracle.dssum(lev["ids"], (lev["B"].ravel() * f), lev["nuniq"])
    dinv = oracle.jacobi(N, lev["G"], lev["B"], lev["ids"], lev["mask"], h2c=h2c, nuniq=lev["nuniq"]).ravel()
    for tol, maxit, restart in ((1e-10, 1000, 15), (0.0, 23, 7)):
        x1, i1, r1, c1 = H.fgmres(levels, b, h2c=h2c, tol=tol, maxit=maxit, restart=restart,
                                  precond=lambda v: dinv * v)
        x2, i2, r2, c2 = oracle.gmres(N, lev["G"], lev["B"], lev["ids"], b.reshape(27, -1), mask=lev["mask"],
                                      h2c=h2c, tol=tol, maxit=maxit, restart=restart, nuniq=lev["nuniq"],
                                      dinv=dinv.reshape(27, -1))
        assert i1 == i2 and c1 == c2
        assert rel_l2(x1, x2) <= 1e-12
        assert abs(r1 - r2) <= 1e-12 + 1e-6 * r2


@pytest.mark.parametrize("N,nel,periodic,deform", [(4, (3, 3, 3), (True, True, True), 0.2),
                                                   (7, (3, 3, 4), (True, False, True), 0.1),
                                                   (5, (3, 4, 3), (False, False, False), 0.0)])
def test_fgmres_hsmg_converges_fast_to_direct_solution(N, nel, periodic, deform):
    m, levels = _box(nel, N, periodic, deform=deform)
    lev = levels[0]
    f = semgen.random_field(lev["ids"].size, 9) + 0.3
    b = oracle.dssum(lev["ids"], lev["B"].ravel() * f, lev["nuniq"])
    if lev["mask"] is not None:
        b = b * lev["mask"]
    x, it, rr, conv = H.fgmres(levels, b, tol=1e-10, maxit=500, restart=30)
    assert conv and rr <= 2e-10
    dinv = oracle.jacobi(N, lev["G"], lev["B"], lev["ids"], lev["mask"], nuniq=lev["nuniq"]).ravel()
    _, itj, _, _ = H.fgmres(levels, b, tol=1e-10, maxit=3000, restart=30, precond=lambda v: dinv * v)
    assert it * 4 <= itj, (it, itj)
    # direct solution of the assembled (projected when singular) system
    E = lev["ids"].size // (N + 1) ** 3
    A, first, keep = _dense(lambda v: H.level_ax(lev, v), lev)
    bk = b[first][keep]
    if lev["mask"] is None:  # singular: mean-zero least-squares solution
        bk = bk - bk.mean()
        xk = np.linalg.lstsq(A, bk, rcond=None)[0]
        xk = xk - xk.mean()
    else:
        xk = np.linalg.solve(A, bk)
    assert rel_l2(x[first][keep], xk) <= 1e-8
    assert E > 0
