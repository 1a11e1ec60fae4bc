// GLL rule and collocation derivative matrix (host, once per mesh).
//
// "basis functions of order N, collocated on the
// Gauss-Lobatto-Legendre points".  Reading R1/R2: the interior
// GLL nodes are the zeros of L_N' = c P^(1,1)_{N-1}; we obtain them by
// Golub-Welsch -- the eigenvalues of the symmetric Jacobi matrix of the
// (1-x)(1+x) weight, off-diagonal b_k = sqrt(k(k+2)/((2k+1)(2k+3))) -- with a
// cyclic Jacobi eigen-solver, then weights w_i = 2/(N(N+1) L_N(xi_i)^2).  The
// derivative matrix uses barycentric weights: D_il = (lam_l/lam_i)/(xi_i-xi_l),
// D_ii = -sum_{l != i} D_il (negative-sum trick).  This is deliberately a
// different construction from the oracle's Newton/Legendre-ratio one.
#include <math.h>

#include <algorithm>
#include <vector>

#include "internal.h"

namespace sem {

static void jacobi_eigenvalues(std::vector<double>& A, int n, std::vector<double>& ev) {
  // cyclic Jacobi rotations on a dense symmetric n x n matrix (n <= 16)
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A[p * n + q] * A[p * n + q];
    if (off < 1e-40) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = A[p * n + q];
        if (fabs(apq) < 1e-300) continue;
        double app = A[p * n + p], aqq = A[q * n + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
      }
  }
  ev.resize(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
  std::sort(ev.begin(), ev.end());
}

static double legendre_N(int N, double x) {
  double p0 = 1.0, p1 = x;
  if (N == 0) return 1.0;
  for (int k = 1; k < N; ++k) {
    double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

bool gll_golub_welsch(int N, double* xi, double* w) {
  if (N < 1 || N > 15) return false;
  const int n = N - 1;  // interior nodes
  std::vector<double> ev;
  if (n > 0) {
    std::vector<double> A(n * n, 0.0);
    for (int k = 1; k < n; ++k) {
      double b = sqrt((double)k * (k + 2) / ((2.0 * k + 1) * (2.0 * k + 3)));
      A[(k - 1) * n + k] = b;
      A[k * n + (k - 1)] = b;
    }
    jacobi_eigenvalues(A, n, ev);
  }
  xi[0] = -1.0;
  xi[N] = 1.0;
  for (int i = 1; i < N; ++i) xi[i] = ev[i - 1];
  // enforce exact antisymmetry of the node set
  std::vector<double> t(N + 1);
  for (int i = 0; i <= N; ++i) t[i] = 0.5 * (xi[i] - xi[N - i]);
  for (int i = 0; i <= N; ++i) xi[i] = t[i];
  for (int i = 0; i <= N; ++i) {
    double L = legendre_N(N, xi[i]);
    w[i] = 2.0 / ((double)N * (N + 1) * L * L);
  }
  return true;
}

void deriv_matrix(int N, const double* xi, double* D) {
  const int lx = N + 1;
  std::vector<double> lam(lx);
  for (int j = 0; j < lx; ++j) {
    double p = 1.0;
    for (int k = 0; k < lx; ++k)
      if (k != j) p *= (xi[j] - xi[k]);
    lam[j] = 1.0 / p;
  }
  for (int i = 0; i < lx; ++i) {
    double diag = 0.0;
    for (int l = 0; l < lx; ++l) {
      if (l == i) continue;
      double v = lam[l] / lam[i] / (xi[i] - xi[l]);
      D[i * lx + l] = v;
      diag -= v;
    }
    D[i * lx + i] = diag;
  }
}

}  // namespace sem
