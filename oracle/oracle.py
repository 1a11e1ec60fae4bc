"""ctypes front-end of the C oracle plus the oracle's own node numbering.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Numbering (reading O6), independent of the CUDA library's
topological numbering built from vertex connectivity:
  * ``lattice_ids``: box meshes, element (ex,ey,ez) lexicographic with x
    fastest.  Local node (i,j,k) of element (ex,ey,ez) gets the
    lattice point (I,J,K) = (ex*N+i, ey*N+j, ez*N+k), taken modulo n_e*N on a
    periodic axis; unique count prod(n_e*N) periodic, prod(n_e*N+1) otherwise.
  * ``geometric_ids``: any conforming mesh: nodes whose coordinates coincide
    (optionally modulo a period per axis) within ``tol`` share an id.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_EINVAL, OR_ENOMEM, OR_EBREAKDOWN = 0, 1, 2, 5

__all__ = [
    "build", "lib", "gll", "dmat", "geom", "ax", "dssum", "mult", "mask_from_bc",
    "jacobi", "pcg", "gmres", "metrics", "grad", "wdiv", "convect", "pnpn_step", "lattice_ids", "geometric_ids", "OracleError", "ax_dssum",
    "OR_OK", "OR_EINVAL", "OR_ENOMEM", "OR_EBREAKDOWN",
]


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile sem_oracle.c into liboracle.so (plain gcc, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
               "-std=c11", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_gll.argtypes = [i32, P, P]
        L.or_dmat.argtypes = [i32, P, P]
        L.or_geom.argtypes = [i64, i32, P, P, P, P, P, P]
        L.or_ax.argtypes = [i64, i32, P, P, P, P, P, dbl, dbl, P, P]
        L.or_dssum.argtypes = [i64, P, i64, P]
        L.or_mult.argtypes = [i64, P, i64, P]
        L.or_mask.argtypes = [i64, i32, P, P, i64, P]
        L.or_jacobi.argtypes = [i64, i32, P, P, P, P, P, dbl, dbl, P, i64, P, P]
        L.or_pcg.argtypes = [i64, i32, P, P, P, P, P, dbl, dbl, P, i64, P, P, P, P, P,
                             dbl, i32, P, P, P]
        L.or_gmres.argtypes = [i64, i32, P, P, P, P, P, dbl, dbl, P, i64, P, P, P, P, P,
                               i32, dbl, i32, P, P, P]
        L.or_metrics.argtypes = [i64, i32, P, P, P, P]
        L.or_grad.argtypes = [i64, i32, P, P, P, P]
        L.or_wdiv.argtypes = [i64, i32, P, P, P, P]
        L.or_convect.argtypes = [i64, i32, P, P, P, P]
        for f in ("or_gll", "or_dmat", "or_geom", "or_ax", "or_dssum", "or_mult",
                  "or_mask", "or_jacobi", "or_pcg", "or_gmres", "or_metrics", "or_grad", "or_wdiv",
                  "or_convect"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _check(st, what):
    if st != OR_OK:
        raise OracleError(st, what)


def gll(N: int):
    """O1: GLL nodes (ascending) and weights for order N (lx = N+1)."""
    xi = np.zeros(N + 1)
    w = np.zeros(N + 1)
    _check(lib().or_gll(N, _p(xi), _p(w)), "gll")
    return xi, w


def dmat(N: int, xi=None):
    """O2: derivative matrix D[i, j] = l_j'(xi_i)."""
    if xi is None:
        xi, _ = gll(N)
    xi = _f64(xi)
    D = np.zeros((N + 1, N + 1))
    _check(lib().or_dmat(N, _p(xi), _p(D)), "dmat")
    return D


def geom(N: int, coords):
    """O4: G [E][6][lx^3] (G11,G22,G33,G12,G13,G23) and B [E][lx^3]."""
    coords = _f64(coords)
    lx = N + 1
    n3 = lx ** 3
    E = coords.size // (3 * n3)
    xi, w = gll(N)
    D = dmat(N, xi)
    G = np.zeros((E, 6, n3))
    B = np.zeros((E, n3))
    bad = ctypes.c_int64(-1)
    st = lib().or_geom(E, N, _p(w), _p(D), _p(coords), _p(G), _p(B), ctypes.byref(bad))
    if st != OR_OK:
        raise OracleError(st, f"geom (J<=0 in element {bad.value})")
    return G, B


def ax(N: int, G, B, u, h1=None, h2=None, h1c=1.0, h2c=0.0):
    """O5: unassembled local Ax, w [E][lx^3]."""
    G, B, u, h1, h2 = _f64(G), _f64(B), _f64(u), _f64(h1), _f64(h2)
    n3 = (N + 1) ** 3
    E = u.size // n3
    D = dmat(N)
    w = np.zeros((E, n3))
    _check(lib().or_ax(E, N, _p(D), _p(G), _p(B), _p(h1), _p(h2), float(h1c), float(h2c),
                       _p(u), _p(w)), "ax")
    return w


def dssum(ids, u, nuniq=None):
    """O7: gather-scatter ADD over global ids (sum in ascending local order)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    out = np.array(u, dtype=np.float64, copy=True, order="C")
    if nuniq is None:
        nuniq = int(ids.max()) + 1 if ids.size else 0
    _check(lib().or_dssum(ids.size, _p(ids), int(nuniq), _p(out)), "dssum")
    return out


def mult(ids, nuniq=None):
    """O7: mult_l = 1/m_{id(l)}."""
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    if nuniq is None:
        nuniq = int(ids.max()) + 1 if ids.size else 0
    m = np.zeros(ids.size)
    _check(lib().or_mult(ids.size, _p(ids), int(nuniq), _p(m)), "mult")
    return m


def mask_from_bc(N: int, bc, ids, nuniq=None):
    """O8: 0 where any copy of the node lies on a Dirichlet face, else 1."""
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    if nuniq is None:
        nuniq = int(ids.max()) + 1 if ids.size else 0
    n3 = (N + 1) ** 3
    E = ids.size // n3
    bcarr = None if bc is None else np.ascontiguousarray(bc, dtype=np.int8)
    m = np.zeros(ids.size)
    _check(lib().or_mask(E, N, _p(bcarr), _p(ids), int(nuniq), _p(m)), "mask")
    return m


def ax_dssum(N: int, G, B, ids, u, mask=None, h1=None, h2=None, h1c=1.0, h2c=0.0, nuniq=None):
    """mask * dssum(Ax(u)) in the local layout (the benchmarked operator)."""
    w = ax(N, G, B, u, h1, h2, h1c, h2c).ravel()
    w = dssum(ids, w, nuniq)
    if mask is not None:
        w = w * np.asarray(mask).ravel()
    return w.reshape(np.shape(u))


def jacobi(N: int, G, B, ids, mask=None, h1=None, h2=None, h1c=1.0, h2c=0.0, nuniq=None):
    """O9: dinv = 1/dssum(diag), 1 at masked nodes."""
    G, B, h1, h2, mask = _f64(G), _f64(B), _f64(h1), _f64(h2), _f64(mask)
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    if nuniq is None:
        nuniq = int(ids.max()) + 1
    n3 = (N + 1) ** 3
    E = ids.size // n3
    D = dmat(N)
    dinv = np.zeros(ids.size)
    _check(lib().or_jacobi(E, N, _p(D), _p(G), _p(B), _p(h1), _p(h2), float(h1c), float(h2c),
                           _p(ids), int(nuniq), _p(mask), _p(dinv)), "jacobi")
    return dinv


def pcg(N: int, G, B, ids, b, mask=None, h1=None, h2=None, h1c=1.0, h2c=0.0,
        tol=1e-12, maxit=1000, nuniq=None, dinv=None):
    """O10: Jacobi-PCG.  Returns (x, iters, rel_res, converged).

    Raises OracleError(OR_EBREAKDOWN) on breakdown (pAp <= 0 or NaN).
    """
    G, B, h1, h2, mask, b = _f64(G), _f64(B), _f64(h1), _f64(h2), _f64(mask), _f64(b)
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    if nuniq is None:
        nuniq = int(ids.max()) + 1
    n3 = (N + 1) ** 3
    E = ids.size // n3
    D = dmat(N)
    m = mult(ids, nuniq)
    if dinv is None:
        dinv = jacobi(N, G, B, ids, mask, h1, h2, h1c, h2c, nuniq)
    x = np.zeros(ids.size)
    iters, conv = ctypes.c_int(0), ctypes.c_int(0)
    rr = ctypes.c_double(0.0)
    st = lib().or_pcg(E, N, _p(D), _p(G), _p(B), _p(h1), _p(h2), float(h1c), float(h2c),
                      _p(ids), int(nuniq), _p(m), _p(mask), _p(dinv), _p(b), _p(x),
                      float(tol), int(maxit), ctypes.byref(iters), ctypes.byref(rr),
                      ctypes.byref(conv))
    _check(st, "pcg")
    return x.reshape(np.shape(b)), iters.value, rr.value, bool(conv.value)


def gmres(N: int, G, B, ids, b, mask=None, h1=None, h2=None, h1c=1.0, h2c=0.0,
          tol=1e-12, maxit=1000, restart=30, nuniq=None, dinv=None):
    """O12: restarted right-preconditioned GMRES(m).  Returns (x, iters,
    rel_res, converged); rel_res is the TRUE residual at the end.

    Raises OracleError(OR_EBREAKDOWN) on a zero Givens pivot.
    """
    G, B, h1, h2, mask, b = _f64(G), _f64(B), _f64(h1), _f64(h2), _f64(mask), _f64(b)
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    if nuniq is None:
        nuniq = int(ids.max()) + 1
    n3 = (N + 1) ** 3
    E = ids.size // n3
    D = dmat(N)
    m = mult(ids, nuniq)
    if dinv is None:
        dinv = jacobi(N, G, B, ids, mask, h1, h2, h1c, h2c, nuniq)
    x = np.zeros(ids.size)
    iters, conv = ctypes.c_int(0), ctypes.c_int(0)
    rr = ctypes.c_double(0.0)
    st = lib().or_gmres(E, N, _p(D), _p(G), _p(B), _p(h1), _p(h2), float(h1c), float(h2c),
                        _p(ids), int(nuniq), _p(m), _p(mask), _p(dinv), _p(b), _p(x),
                        int(restart), float(tol), int(maxit), ctypes.byref(iters), ctypes.byref(rr),
                        ctypes.byref(conv))
    _check(st, "gmres")
    return x.reshape(np.shape(b)), iters.value, rr.value, bool(conv.value)


def metrics(N: int, coords):
    """O13: mass-weighted metric terms MJ [E][3 (a)][3 (m)][n3] = W J dr_a/dx_m."""
    coords = _f64(coords)
    xi, w = gll(N)
    D = dmat(N)
    n3 = (N + 1) ** 3
    E = coords.size // (3 * n3)
    MJ = np.zeros((E, 3, 3, n3))
    _check(lib().or_metrics(E, N, _p(w), _p(D), _p(coords), _p(MJ)), "metrics")
    return MJ


def grad(N: int, MJ, u):
    """O14: mass-weighted collocation gradient [3][E][n3] of u [E][n3] (local)."""
    MJ, u = _f64(MJ), _f64(u)
    n3 = (N + 1) ** 3
    E = u.size // n3
    g = np.zeros((3, E, n3))
    _check(lib().or_grad(E, N, _p(dmat(N)), _p(MJ), _p(u), _p(g)), "grad")
    return g


def wdiv(N: int, MJ, f):
    """O15: weak divergence (grad v, f) [E][n3] of f [3][E][n3] (local)."""
    MJ, f = _f64(MJ), _f64(f)
    n3 = (N + 1) ** 3
    E = f.size // (3 * n3)
    d = np.zeros((E, n3))
    _check(lib().or_wdiv(E, N, _p(dmat(N)), _p(MJ), _p(f), _p(d)), "wdiv")
    return d


def convect(N: int, MJ, u):
    """O16: mass-weighted convection W J (u . grad) u_i, [3][E][n3] (local)."""
    MJ, u = _f64(MJ), _f64(u)
    n3 = (N + 1) ** 3
    E = u.size // (3 * n3)
    c = np.zeros((3, E, n3))
    _check(lib().or_convect(E, N, _p(dmat(N)), _p(MJ), _p(u), _p(c)), "convect")
    return c


def pnpn_step(N: int, G, B, MJ, ids, u, dt, nu, nuniq=None, tol=1e-12, maxit=5000, pressure_solve=None):
    """O17: one first-order velocity-pressure splitting step
    (BDF1 / EXT1; PAPER.md:72 cites Karniadakis et al. 1991 for the
    splitting) on a periodic mesh, written out in the scheme's order:
      1. convection  c_i = dssum(W J (u.grad) u_i)                      (O16)
      2. predictor   u~_i = (dssum(B u_i) - dt c_i) / dssum(B)
      3. pressure    A p = (1/dt) dssum(wdiv(u~)),  A = Poisson (O5),
                     singular -> mean-zero projections (O10)
      4. velocity    (nu A + B/dt) u_i = dssum(B u~_i)/dt - dssum(grad_i p)
                     (Helmholtz h1 = nu, h2 = 1/dt, O5/O10)
    u: [3][E][n3] continuous.  Returns (u_new [3][E][n3], p [E][n3], iterations
    of the pressure solve, of the three velocity solves).  pressure_solve(rp)
    -> (p, iterations) replaces the pressure PCG (e.g. the oracle's FGMRES
    with the multigrid preconditioner, oracle/hsmg.py)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    if nuniq is None:
        nuniq = int(ids.max()) + 1
    n3 = (N + 1) ** 3
    u = np.asarray(u, dtype=np.float64).reshape(3, -1, n3)
    E = u.shape[1]
    Bf = np.asarray(B, dtype=np.float64).ravel()
    Bg = dssum(ids, Bf, nuniq)
    c = convect(N, MJ, u)
    ut = np.empty_like(u)
    for i in range(3):
        ut[i] = ((dssum(ids, Bf * u[i].ravel(), nuniq) - dt * dssum(ids, c[i].ravel(), nuniq)) / Bg).reshape(E, n3)
    rp = dssum(ids, wdiv(N, MJ, ut).ravel(), nuniq) / dt
    if pressure_solve is None:
        p, itp, _, _ = pcg(N, G, B, ids, rp, h1c=1.0, h2c=0.0, tol=tol, maxit=maxit, nuniq=nuniq)
    else:
        p, itp = pressure_solve(rp)
    g = grad(N, MJ, p)
    un = np.empty_like(u)
    itv = []
    for i in range(3):
        rv = dssum(ids, Bf * ut[i].ravel(), nuniq) / dt - dssum(ids, g[i].ravel(), nuniq)
        xi_, it, _, _ = pcg(N, G, B, ids, rv, h1c=nu, h2c=1.0 / dt, tol=tol, maxit=maxit, nuniq=nuniq)
        un[i] = xi_.reshape(E, n3)
        itv.append(it)
    return un, np.asarray(p).reshape(E, n3), itp, itv


def lattice_ids(nel, N: int, periodic):
    """O6 (box meshes): lattice global ids, shape [E][lx^3]; returns (ids, nuniq)."""
    nx, ny, nz = nel
    lx = N + 1
    ex, ey, ez = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    # element index e = ex + nx*(ey + ny*ez)  (x fastest)
    ex = ex.transpose(2, 1, 0).ravel()
    ey = ey.transpose(2, 1, 0).ravel()
    ez = ez.transpose(2, 1, 0).ravel()
    k, j, i = np.meshgrid(np.arange(lx), np.arange(lx), np.arange(lx), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()  # node p = i + lx*j + lx^2*k
    I = ex[:, None] * N + i[None, :]
    J = ey[:, None] * N + j[None, :]
    K = ez[:, None] * N + k[None, :]
    dims = []
    for c, (n_e, per) in enumerate(zip(nel, periodic)):
        dims.append(n_e * N if per else n_e * N + 1)
    if periodic[0]:
        I = I % dims[0]
    if periodic[1]:
        J = J % dims[1]
    if periodic[2]:
        K = K % dims[2]
    ids = I + dims[0] * (J + dims[1] * K)
    return ids.astype(np.int64), int(dims[0] * dims[1] * dims[2])


def geometric_ids(coords, periods=(None, None, None), tol=1e-9):
    """O6 (general meshes): nodes with coincident coordinates share an id.

    coords: [3][E][n3] (or [3][nloc]).  ``periods``: per-axis period (or None);
    coordinates are wrapped into [0, period) first, with values within ``tol``
    of the period mapped to 0.  Ids are assigned in order of first appearance
    (ascending local index).  Returns (ids [nloc], nuniq).
    """
    X = np.array(coords, dtype=np.float64).reshape(3, -1)
    for a, per in enumerate(periods):
        if per is not None:
            v = np.mod(X[a], per)
            v[np.abs(v - per) < tol] = 0.0
            v[np.abs(v) < tol] = 0.0
            X[a] = v
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree
    n = X.shape[1]
    pairs = cKDTree(X.T).query_pairs(r=tol, output_type="ndarray")
    adj = coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(n, n))
    _, comp = connected_components(adj, directed=False)
    # renumber components by first appearance (ascending local index)
    _, first = np.unique(comp, return_index=True)
    rank = np.empty(first.size, dtype=np.int64)
    rank[np.argsort(first)] = np.arange(first.size)
    ids = rank[comp]
    return ids, int(first.size)
