"""Test-only helpers: brute-force assembly of the oracle's operator and
textbook reference matrices.  Uses only numpy/scipy and the oracle."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

import oracle


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def element_matrices(N, G, B, h1=None, h2=None, h1c=1.0, h2c=0.0):
    """A_e [E][n3][n3] by applying oracle.ax (O5) to unit vectors (P8)."""
    n3 = (N + 1) ** 3
    E = G.shape[0]
    A = np.zeros((E, n3, n3))
    eye = np.eye(n3)
    for e in range(E):
        Ge = np.broadcast_to(G[e], (n3, 6, n3))
        Be = np.broadcast_to(B[e], (n3, n3))
        h1e = None if h1 is None else np.broadcast_to(np.reshape(h1, (E, n3))[e], (n3, n3))
        h2e = None if h2 is None else np.broadcast_to(np.reshape(h2, (E, n3))[e], (n3, n3))
        W = oracle.ax(N, Ge, Be, eye, h1e, h2e, h1c, h2c)  # row c = A_e e_c
        A[e] = W.T
    return A


def scatter_matrix(ids, nuniq):
    """Q: local <- unique (Q[l, g] = 1 iff id(l) = g)."""
    ids = np.asarray(ids).ravel()
    n = ids.size
    return sp.csr_matrix((np.ones(n), (np.arange(n), ids)), shape=(n, nuniq))


def assembled(N, Ae, ids, nuniq):
    """A = Q^T blockdiag(A_e) Q (sparse)."""
    Q = scatter_matrix(ids, nuniq)
    Ab = sp.block_diag([sp.csr_matrix(a) for a in Ae], format="csr")
    return (Q.T @ Ab @ Q).tocsr()


def textbook_1d(N, h, n_el, periodic, xi, w, D):
    """Assembled 1D GLL stiffness K and (diagonal) mass M on a uniform grid:
    element K_e = (2/h) D^T W D, M_e = (h/2) W (Deville-Fischer-Mund 2002)."""
    W = np.diag(w)
    Ke = (2.0 / h) * D.T @ W @ D
    Me = (h / 2.0) * W
    n = n_el * N if periodic else n_el * N + 1
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    for e in range(n_el):
        idx = [(e * N + i) % n if periodic else e * N + i for i in range(N + 1)]
        K[np.ix_(idx, idx)] += Ke
        M[np.ix_(idx, idx)] += Me
    return K, M


def scipy_gll(N):
    """Independent GLL rule: interior nodes = roots of P_{N-1}^{(1,1)}
    (scipy.special.roots_jacobi, Golub-Welsch), w = 2/(N(N+1) P_N(x)^2)."""
    from scipy.special import eval_legendre, roots_jacobi
    if N == 1:
        x = np.array([-1.0, 1.0])
    else:
        r, _ = roots_jacobi(N - 1, 1.0, 1.0)
        x = np.concatenate([[-1.0], np.sort(r), [1.0]])
    w = 2.0 / (N * (N + 1) * eval_legendre(N, x) ** 2)
    return x, w


def bary_D(x):
    """Independent collocation derivative matrix by barycentric weights:
    D_ij = (lam_j/lam_i)/(x_i - x_j), D_ii = -sum_{j!=i} D_ij."""
    x = np.asarray(x, dtype=np.float64)
    n = x.size
    lam = np.array([1.0 / np.prod([x[j] - x[k] for k in range(n) if k != j]) for j in range(n)])
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = lam[j] / lam[i] / (x[i] - x[j])
        D[i, i] = -np.sum(D[i, :])
    return D
