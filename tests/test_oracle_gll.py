"""Pins of the oracle's GLL rule (O1) and derivative matrix (O2).

P1 closed forms, P2 quadrature exactness (BASELINE.json north_star: "GLL
quadrature exactness for polynomials up to degree 2N-1"), P3 derivative
exactness, P4 the N=2 1D stiffness worked example (tests/golden/k1d_n2.txt).
"""
import os

import numpy as np
import pytest

import oracle
from helpers import bary_D, scipy_gll

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_gll_closed_forms():
    # P1: N=1 -> {-1,1}, w={1,1}; N=2 -> {-1,0,1}, w={1/3,4/3,1/3};
    #     N=3 -> {-1,-1/sqrt5,1/sqrt5,1}, w={1/6,5/6,5/6,1/6}
    xi, w = oracle.gll(1)
    np.testing.assert_allclose(xi, [-1, 1], atol=0)
    np.testing.assert_allclose(w, [1, 1], rtol=1e-15)
    xi, w = oracle.gll(2)
    np.testing.assert_allclose(xi, [-1, 0, 1], atol=1e-16)
    np.testing.assert_allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-15)
    xi, w = oracle.gll(3)
    s = 1 / np.sqrt(5)
    np.testing.assert_allclose(xi, [-1, -s, s, 1], rtol=1e-15)
    np.testing.assert_allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], rtol=1e-15)


@pytest.mark.parametrize("N", range(1, 16))
def test_gll_matches_golub_welsch(N):
    xi, w = oracle.gll(N)
    xs, ws = scipy_gll(N)
    np.testing.assert_allclose(xi, xs, atol=5e-15)
    np.testing.assert_allclose(w, ws, rtol=1e-13)
    assert abs(w.sum() - 2.0) < 1e-14
    np.testing.assert_array_equal(xi, -xi[::-1])  # exact symmetry after symmetrisation
    assert np.all(np.diff(xi) > 0)


@pytest.mark.parametrize("N", [3, 5, 7, 9, 11])
def test_gll_exactness(N):
    # P2: exact for x^k, k <= 2N-1; not exact at k = 2N
    xi, w = oracle.gll(N)
    for k in range(0, 2 * N):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, xi ** k) - exact) < 1e-14, k
    exact = 2.0 / (2 * N + 1)
    assert abs(np.dot(w, xi ** (2 * N)) - exact) > 1e-10  # >> roundoff


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 7, 9, 11])
def test_dmat(N):
    # P3: D xi^N = N xi^(N-1); D 1 = 0; D_00 = -N(N+1)/4; interior diagonal 0;
    # equals the barycentric differentiation matrix (independent construction)
    xi, _ = oracle.gll(N)
    D = oracle.dmat(N)
    np.testing.assert_allclose(D @ np.ones(N + 1), 0, atol=1e-12 * N * N)
    np.testing.assert_allclose(D @ xi ** N, N * xi ** (N - 1), atol=1e-12 * N * N)
    rng = np.random.default_rng(N)
    c = rng.standard_normal(N + 1)
    p = np.polynomial.Polynomial(c)
    np.testing.assert_allclose(D @ p(xi), p.deriv()(xi), atol=1e-12 * N * N * np.abs(c).sum())
    assert D[0, 0] == -N * (N + 1) / 4 and D[N, N] == N * (N + 1) / 4
    for i in range(1, N):
        assert D[i, i] == 0.0
    np.testing.assert_allclose(D, bary_D(xi), atol=2e-13 * N * N)


def test_k1d_worked_example():
    # P4: N=2, K = D^T W D = (1/6)[[7,-8,1],[-8,16,-8],[1,-8,7]]
    xi, w = oracle.gll(2)
    D = oracle.dmat(2)
    K = D.T @ np.diag(w) @ D
    gold = np.loadtxt(os.path.join(GOLDEN, "k1d_n2.txt"))
    np.testing.assert_allclose(K, gold / 6.0, atol=1e-15)
