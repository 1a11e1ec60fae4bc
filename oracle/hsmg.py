"""Oracle of the pressure preconditioner: hybrid-Schwarz multigrid (HSMG) and
flexible GMRES ("restarted GMRES for the
pressure solves with a hybrid-Schwarz multigrid preconditioner").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written from reading R16
(DESIGN.md), which fixes what the paper leaves open; every step below is
that reading written out, in its order and notation:

  levels     orders N_0 = N > N_1 = N // 2 (only if > 1) > N_{L-1} = 1; level
             coordinates = the fine element map evaluated at the level's GLL
             nodes; level operator A_l = mask . dssum . A_e at order N_l (R5)
  transfer   J_l [lx_l x lx_{l+1}], J[a, b] = lagrange_b^{(l+1)}(xi_a^{(l)});
             prolongation  P u = (J (x) J (x) J) u            (element-wise)
             restriction   R r = mask . dssum((J^T (x) J^T (x) J^T)(r / m))
  smoother   averaged additive Schwarz, one subdomain per element (its own
             nodes, overlapping its neighbours in the shared nodes), local
             operator = the separable ("fast diagonalisation") operator of
             the element's box: 1-D SEM stiffness/mass of length L_d with the
             diagonal end entries doubled (the neighbour's share: the
             principal submatrix of the assembled 1-D operator on the
             element's nodes), h1 (x) stiffness sum + h2 mass;
             S r = mask . (1/m) . dssum(A~_e^{-1} r_e)
  V-cycle    z_0 = S_0 r ; r_1 = R_0 (r - A_0 z_0) ; ... ; coarse: <= K steps of
             Jacobi-PCG (R10, tol 1e-12) on A_{L-1} ; z_l += P_l z_{l+1} upward
  Krylov     FGMRES(m) (Saad 1993): right-preconditioned with Z_j = M v_j
             stored, x = x_0 + Z y; otherwise the conventions of or_gmres
             (R14): MGS, Givens, |g_{j+1}| <= tol ||b||, true residual at the
             end of each cycle, singular projections of b and x.

Pins: tests/test_oracle_hsmg.py.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import oracle as O


# ---- 1-D pieces -------------------------------------------------------------

def lagrange_matrix(x_from, x_to):
    """J[a, b] = l_b(x_to[a]), l_b the Lagrange polynomial on nodes x_from
    (product formula)."""
    x_from = np.asarray(x_from, dtype=np.float64)
    x_to = np.asarray(x_to, dtype=np.float64)
    J = np.ones((x_to.size, x_from.size))
    for b in range(x_from.size):
        for q in range(x_from.size):
            if q != b:
                J[:, b] *= (x_to - x_from[q]) / (x_from[b] - x_from[q])
    return J


def fdm_1d(N: int):
    """R16: reference 1-D operators on [-1, 1] extended by the neighbours'
    share (end diagonal entries doubled), and their generalised eigenpairs:
    A_ext S = B_ext S diag(mu), S^T B_ext S = I.  Returns (A_ext, B_ext, S, mu)."""
    xi, w = O.gll(N)
    D = O.dmat(N, xi)
    A = D.T @ np.diag(w) @ D
    Bm = np.diag(w)
    Ae = A.copy()
    Be = Bm.copy()
    Ae[0, 0] += A[N, N]
    Ae[N, N] += A[0, 0]
    Be[0, 0] += w[N]
    Be[N, N] += w[0]
    mu, S = scipy.linalg.eigh(Ae, Be)
    return Ae, Be, S, mu


def element_lengths(N: int, coords):
    """R16: L[e, d] = mean over the 4 element edges along reference direction d
    of the straight distance between their end vertices."""
    lx = N + 1
    X = np.asarray(coords, dtype=np.float64).reshape(3, -1, lx, lx, lx)  # [c][e][k][j][i]
    E = X.shape[1]
    L = np.zeros((E, 3))
    ends = (0, N)
    for a in ends:
        for b in ends:
            L[:, 0] += np.linalg.norm(X[:, :, a, b, N] - X[:, :, a, b, 0], axis=0)
            L[:, 1] += np.linalg.norm(X[:, :, a, N, b] - X[:, :, a, 0, b], axis=0)
            L[:, 2] += np.linalg.norm(X[:, :, N, a, b] - X[:, :, 0, a, b], axis=0)
    return L / 4.0


def tensor3(Ax, Ay, Az, u, lx_in):
    """(Az (x) Ay (x) Ax) u per element, u [E][lx_in^3] with node i + lx j + lx^2 k."""
    E = u.size // lx_in ** 3
    U = np.asarray(u, dtype=np.float64).reshape(E, lx_in, lx_in, lx_in)  # [e][k][j][i]
    V = np.einsum("ai,ekji->ekja", Ax, U)
    V = np.einsum("bj,ekja->ekba", Ay, V)
    V = np.einsum("ck,ekba->ecba", Az, V)
    return V.reshape(E, -1)


# ---- the smoother -------------------------------------------------------------

def fdm_local_solve(N: int, L, r, h1c=1.0, h2c=0.0, fdm=None):
    """R16: z_e = A~_e^{-1} r_e for every element (no assembly), by fast
    diagonalisation: with S_d = sqrt(2/L_d) S and Lambda_d = (4/L_d^2) mu,
    A~_e^{-1} = (S_z (x) S_y (x) S_x) [h1 (Lx + Ly + Lz) + h2]^{-1} (...)^T."""
    _, _, S, mu = fdm if fdm is not None else fdm_1d(N)
    lx = N + 1
    E = L.shape[0]
    rh = tensor3(S.T, S.T, S.T, r, lx).reshape(E, lx, lx, lx)  # [e][k][j][i]
    lam = 4.0 * mu
    out = np.empty_like(rh)
    for e in range(E):
        Lx, Ly, Lz = L[e]
        den = (h1c * (lam[None, None, :] / Lx ** 2 + lam[None, :, None] / Ly ** 2 + lam[:, None, None] / Lz ** 2)
               + h2c)
        out[e] = rh[e] / den * (8.0 / (Lx * Ly * Lz))
    return tensor3(S, S, S, out.reshape(E, -1), lx)


def schwarz(lev, r, h1c=1.0, h2c=0.0):
    """R16: S r = mask . (1/m) . dssum(A~_e^{-1} r_e)."""
    z = fdm_local_solve(lev["N"], lev["L"], r, h1c, h2c, lev["fdm"]).ravel()
    z = O.dssum(lev["ids"], z, lev["nuniq"]) * lev["mult"]
    if lev["mask"] is not None:
        z = z * lev["mask"]
    return z


# ---- levels and transfers -------------------------------------------------------

def level_orders(N: int):
    """R16: N, N // 2 (if > 1), 1."""
    orders = [N]
    if N // 2 > 1:
        orders.append(N // 2)
    if N > 1:
        orders.append(1)
    return orders


def make_level(N: int, coords, ids, nuniq, bc):
    G, B = O.geom(N, coords)
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    mask = O.mask_from_bc(N, bc, ids, nuniq) if bc is not None else None
    if mask is not None and np.all(mask == 1.0):
        mask = None
    return {"N": N, "coords": np.asarray(coords, dtype=np.float64), "G": G, "B": B, "ids": ids,
            "nuniq": int(nuniq), "mult": O.mult(ids, nuniq), "mask": mask,
            "L": element_lengths(N, coords), "fdm": fdm_1d(N)}


def setup(N: int, coords, bc, ids_fn):
    """Levels of R16.  ids_fn(N_l, coords_l) -> (ids, nuniq) numbers the level
    (the oracle's own lattice or geometric numbering, O6)."""
    orders = level_orders(N)
    xf, _ = O.gll(N)
    E = np.asarray(coords).size // (3 * (N + 1) ** 3)
    levels = []
    for Nl in orders:
        xl, _ = O.gll(Nl)
        K = lagrange_matrix(xf, xl)  # fine map evaluated at the level's nodes
        cl = np.stack([tensor3(K, K, K, np.asarray(coords)[c].reshape(E, -1), N + 1) for c in range(3)])
        ids, nuniq = ids_fn(Nl, cl)
        levels.append(make_level(Nl, cl, ids, nuniq, bc))
    for l in range(len(levels) - 1):
        xa, _ = O.gll(levels[l]["N"])
        xb, _ = O.gll(levels[l + 1]["N"])
        levels[l]["J"] = lagrange_matrix(xb, xa)  # [lx_l][lx_{l+1}]
    return levels


def prolong(lev_f, u_c):
    J = lev_f["J"]
    return tensor3(J, J, J, u_c, J.shape[1]).ravel()


def restrict(lev_f, lev_c, r_f):
    J = lev_f["J"]
    t = tensor3(J.T, J.T, J.T, np.asarray(r_f).ravel() * lev_f["mult"], J.shape[0]).ravel()
    t = O.dssum(lev_c["ids"], t, lev_c["nuniq"])
    if lev_c["mask"] is not None:
        t = t * lev_c["mask"]
    return t


def level_ax(lev, u, h1c=1.0, h2c=0.0):
    return O.ax_dssum(lev["N"], lev["G"], lev["B"], lev["ids"], np.asarray(u).reshape(-1, (lev["N"] + 1) ** 3),
                      mask=lev["mask"], h1c=h1c, h2c=h2c, nuniq=lev["nuniq"]).ravel()


COARSE_TOL = 1e-12


def coarse_solve(lev, r, h1c=1.0, h2c=0.0, iters=20):
    """R16: at most K steps of the oracle's Jacobi-PCG (O10) from x = 0,
    stopping early at ||r|| <= 1e-12 ||b|| (small coarse problems converge in
    fewer than K steps; a tol = 0 run would then break down on r = 0)."""
    n3 = (lev["N"] + 1) ** 3
    x, _, _, _ = O.pcg(lev["N"], lev["G"], lev["B"], lev["ids"], np.asarray(r).reshape(-1, n3),
                       mask=lev["mask"], h1c=h1c, h2c=h2c, tol=COARSE_TOL, maxit=iters, nuniq=lev["nuniq"])
    return x.ravel()


def vcycle(levels, r, h1c=1.0, h2c=0.0, coarse_iters=5):
    """R16: one V(1,0) cycle z = M r (r assembled and masked)."""
    nl = len(levels)
    rs = [np.asarray(r, dtype=np.float64).ravel()]
    zs = []
    for l in range(nl - 1):
        z = schwarz(levels[l], rs[l], h1c, h2c)
        zs.append(z)
        res = rs[l] - level_ax(levels[l], z, h1c, h2c)
        rs.append(restrict(levels[l], levels[l + 1], res))
    zs.append(coarse_solve(levels[-1], rs[-1], h1c, h2c, coarse_iters))
    for l in range(nl - 2, -1, -1):
        zs[l] = zs[l] + prolong(levels[l], zs[l + 1])
    return zs[0]


# ---- flexible GMRES -------------------------------------------------------------

def fgmres(levels, b, h1c=1.0, h2c=0.0, tol=1e-12, maxit=1000, restart=30, precond=None, coarse_iters=5):
    """FGMRES(m) on A_0 x = b with z_j = precond(v_j) (default: the V-cycle);
    conventions of or_gmres (R14).  Returns (x, iters, rel_res, converged)."""
    lev = levels[0]
    mult, mask, nuniq = lev["mult"], lev["mask"], lev["nuniq"]
    M = precond if precond is not None else (lambda v: vcycle(levels, v, h1c, h2c, coarse_iters))
    b = np.asarray(b, dtype=np.float64).ravel().copy()
    if mask is not None:
        b = b * mask
    singular = mask is None and h2c == 0.0
    if singular:
        b = b - np.sum(mult * b) / nuniq
    n = b.size
    x = np.zeros(n)
    r = b.copy()
    dot = lambda a, c: float(np.sum(mult * a * c))
    bn = np.sqrt(dot(b, b))
    beta = bn
    if bn == 0.0:
        return x, 0, 0.0, True
    m = restart
    it, conv = 0, False
    while it < maxit:
        V = [r / beta]
        Z = []
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        k = 0
        for j in range(m):
            Z.append(M(V[j]))
            w = level_ax(lev, Z[j], h1c, h2c)
            for i in range(j + 1):
                H[i, j] = dot(w, V[i])
                w = w - H[i, j] * V[i]
            hn = np.sqrt(dot(w, w))
            H[j + 1, j] = hn
            V.append(w / hn if hn != 0.0 else w)
            for i in range(j):
                a, c = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * c
                H[i + 1, j] = -sn[i] * a + cs[i] * c
            d = np.sqrt(H[j, j] ** 2 + H[j + 1, j] ** 2)
            if not d > 0.0:
                raise O.OracleError(O.OR_EBREAKDOWN, "fgmres: breakdown")
            cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
            H[j, j], H[j + 1, j] = d, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            k = j + 1
            if tol > 0.0 and abs(g[j + 1]) <= tol * bn:
                conv = True
                break
            if hn == 0.0 or it >= maxit:
                break
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        for i in range(k):
            x = x + y[i] * Z[i]
        r = b - level_ax(lev, x, h1c, h2c)
        beta = np.sqrt(dot(r, r))
        if conv or beta == 0.0:
            break
    if singular:
        x = x - np.sum(mult * x) / nuniq
    return x, it, beta / bn, conv or beta == 0.0
