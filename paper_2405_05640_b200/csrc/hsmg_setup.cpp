// Host set-up of the hybrid-Schwarz multigrid preconditioner (SURVEY 8(f)
// f2; reading R16): level orders, the fast-diagonalisation
// factors of the extended 1-D operators, the Lagrange transfer matrices, the
// level coordinates and the element lengths.  Once per mesh.
#include <math.h>

#include <algorithm>
#include <vector>

#include "hsmg.h"

namespace sem {

bool gll_golub_welsch(int N, double* xi, double* w);
void deriv_matrix(int N, const double* xi, double* D);

int hsmg_level_orders(int N, int* orders) {
  int n = 0;
  orders[n++] = N;
  if (N / 2 > 1) orders[n++] = N / 2;
  if (N > 1) orders[n++] = 1;
  return n;
}

// cyclic Jacobi on a dense symmetric n x n matrix A (destroyed): eigenvalues
// ev and eigenvectors V (column c of V[l*n + c])
static void jacobi_eig(std::vector<double>& A, int n, std::vector<double>& ev, std::vector<double>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < n; ++p) {
      diag += A[p * n + p] * A[p * n + p];
      for (int q = p + 1; q < n; ++q) off += A[p * n + q] * A[p * n + q];
    }
    if (off <= 1e-32 * diag) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (fabs(apq) < 1e-300) continue;
        const double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- A R
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // A <- R^T A
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {  // V <- V R
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  ev.resize(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
}

// R16: A_ext = D^T W D with the end diagonal entries doubled (the neighbour's
// share), B_ext = W with the end weights doubled; A_ext S = B_ext S diag(mu),
// S^T B_ext S = I via C = B^-1/2 A B^-1/2 = Q diag(mu) Q^T, S = B^-1/2 Q.
bool hsmg_fdm_1d(int N, double* S, double* lam) {
  const int lx = N + 1;
  std::vector<double> xi(lx), w(lx), D((size_t)lx * lx);
  if (!gll_golub_welsch(N, xi.data(), w.data())) return false;
  deriv_matrix(N, xi.data(), D.data());
  std::vector<double> A((size_t)lx * lx, 0.0), Bd(w);
  for (int p = 0; p < lx; ++p)
    for (int q = 0; q < lx; ++q) {
      double s = 0.0;
      for (int k = 0; k < lx; ++k) s += D[k * lx + p] * w[k] * D[k * lx + q];
      A[p * lx + q] = s;
    }
  const double a00 = A[0], ann = A[N * lx + N];
  A[0] += ann;
  A[N * lx + N] += a00;
  Bd[0] += w[N];
  Bd[N] += w[0];
  std::vector<double> C((size_t)lx * lx), ev, Q;
  for (int p = 0; p < lx; ++p)
    for (int q = 0; q < lx; ++q) C[p * lx + q] = A[p * lx + q] / sqrt(Bd[p] * Bd[q]);
  jacobi_eig(C, lx, ev, Q);
  for (int l = 0; l < lx; ++l)
    for (int c = 0; c < lx; ++c) S[l * lx + c] = Q[l * lx + c] / sqrt(Bd[l]);
  for (int c = 0; c < lx; ++c) lam[c] = 4.0 * ev[c];
  return true;
}

void hsmg_lagrange(int nfrom, const double* xfrom, int nto, const double* xto, double* J) {
  for (int a = 0; a < nto; ++a)
    for (int b = 0; b < nfrom; ++b) {
      double p = 1.0;
      for (int q = 0; q < nfrom; ++q)
        if (q != b) p *= (xto[a] - xfrom[q]) / (xfrom[b] - xfrom[q]);
      J[a * nfrom + b] = p;
    }
}

// cc = (K (x) K (x) K) cf per element and coordinate; K [lxc][lxf]
void hsmg_interp_coords(int64_t E, int lxf, int lxc, const double* K, const double* cf, double* cc) {
  const int64_t nf = (int64_t)lxf * lxf * lxf, nc = (int64_t)lxc * lxc * lxc;
  std::vector<double> t1((size_t)lxf * lxf * lxc), t2((size_t)lxf * lxc * lxc);
  for (int c = 0; c < 3; ++c)
    for (int64_t e = 0; e < E; ++e) {
      const double* u = cf + ((int64_t)c * E + e) * nf;
      double* o = cc + ((int64_t)c * E + e) * nc;
      for (int k = 0; k < lxf; ++k)
        for (int j = 0; j < lxf; ++j)
          for (int a = 0; a < lxc; ++a) {
            double s = 0.0;
            for (int i = 0; i < lxf; ++i) s += K[a * lxf + i] * u[i + lxf * (j + lxf * k)];
            t1[a + lxc * (j + lxf * k)] = s;
          }
      for (int k = 0; k < lxf; ++k)
        for (int b = 0; b < lxc; ++b)
          for (int a = 0; a < lxc; ++a) {
            double s = 0.0;
            for (int j = 0; j < lxf; ++j) s += K[b * lxf + j] * t1[a + lxc * (j + lxf * k)];
            t2[a + lxc * (b + lxc * k)] = s;
          }
      for (int g = 0; g < lxc; ++g)
        for (int b = 0; b < lxc; ++b)
          for (int a = 0; a < lxc; ++a) {
            double s = 0.0;
            for (int k = 0; k < lxf; ++k) s += K[g * lxf + k] * t2[a + lxc * (b + lxc * k)];
            o[a + lxc * (b + lxc * g)] = s;
          }
    }
}

// L[e][d] = mean over the 4 edges along reference direction d of the
// straight distance between their end vertices
void hsmg_element_lengths(int64_t E, int lx, const double* coords, double* L) {
  const int N = lx - 1;
  const int64_t n3 = (int64_t)lx * lx * lx;
  auto X = [&](int c, int64_t e, int i, int j, int k) { return coords[((int64_t)c * E + e) * n3 + i + lx * (j + lx * k)]; };
  auto dist = [&](int64_t e, int i0, int j0, int k0, int i1, int j1, int k1) {
    double s = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double d = X(c, e, i1, j1, k1) - X(c, e, i0, j0, k0);
      s += d * d;
    }
    return sqrt(s);
  };
  for (int64_t e = 0; e < E; ++e) {
    double lx_ = 0.0, ly = 0.0, lz = 0.0;
    for (int a : {0, N})
      for (int b : {0, N}) {
        lx_ += dist(e, 0, b, a, N, b, a);
        ly += dist(e, b, 0, a, b, N, a);
        lz += dist(e, b, a, 0, b, a, N);
      }
    L[e * 3 + 0] = lx_ / 4.0;
    L[e * 3 + 1] = ly / 4.0;
    L[e * 3 + 2] = lz / 4.0;
  }
}

}  // namespace sem
