/*
 * oracle/sem_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * SEM hot path of arXiv 2405.05640 (Karp et al.): matrix-free local operator
 * Ax, direct-stiffness summation (dssum / gather-scatter), Dirichlet mask,
 * Jacobi diagonal and Jacobi-preconditioned CG.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA library in
 * paper_2405_05640_b200/ and must never be called from the product path.
 *
 * Where the paper fixes the method (PAPER.md section "Neko", lines 71-74):
 *   - "the computational domain is split into E non-overlapping hexahedral
 *      elements" with "high-order polynomial basis functions of order N,
 *      collocated on the Gauss-Lobatto-Legendre points";
 *   - operators are applied "element-by-element or matrix-free" and the only
 *     coupling is the "unit-depth" "gather-scatter phase";
 *   - "preconditioned Krylov subspace methods are used to solve linear
 *      systems on the form Ax=b", with "CG together with a
 *      block-Jacobi preconditioner" for the Helmholtz (velocity) solves
 *      (PAPER.md:72).
 * The paper never writes the operator; every formula below is the standard
 * SEM definition of Deville, Fischer & Mund (2002), which the paper cites for
 * the method.  The precise readings (O1..O10) are
 * listed in DESIGN.md section "Readings" and in SURVEY.md section 8(c).
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction) so that every
 * operation is the IEEE operation written here.  OpenMP is used only as a
 * `parallel for` over independent elements; no reordering of any sum.
 *
 * Layout (reading O3): local node l = i + lx*j + lx^2*k + lx^3*e, i <-> r,
 * j <-> s, k <-> t.  Coordinates SoA [3][E][lx^3].  Geometric factors
 * [E][6][lx^3] in the order G11, G22, G33, G12, G13, G23.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOMEM 2
#define OR_EBREAKDOWN 5

/* ------------------------------------------------------------------------ */
/* O1: Legendre polynomial L_N(x) and its derivative by the three-term
 * recurrence (k+1) L_{k+1} = (2k+1) x L_k - k L_{k-1},
 * L'_{k+1} = L'_{k-1} + (2k+1) L_k.                                          */
static void legendre(int N, double x, double* L, double* dL) {
  double Lm1 = 1.0, L0 = x;     /* L_0, L_1 */
  double dLm1 = 0.0, dL0 = 1.0; /* L_0', L_1' */
  if (N == 0) { *L = 1.0; *dL = 0.0; return; }
  for (int k = 1; k < N; ++k) {
    double Lp1 = ((2.0 * k + 1.0) * x * L0 - k * Lm1) / (k + 1.0);
    double dLp1 = dLm1 + (2.0 * k + 1.0) * L0;
    Lm1 = L0; L0 = Lp1;
    dLm1 = dL0; dL0 = dLp1;
  }
  *L = L0; *dL = dL0;
}

/* O1: GLL nodes xi_0..xi_N (ascending) and weights.
 * xi_0 = -1, xi_N = +1, interior xi_i = roots of L_N', found by Newton on
 * L_N' from the Chebyshev-Gauss-Lobatto guess -cos(pi i / N) until
 * |dx| < 1e-15; L_N'' from the Legendre ODE
 * (1-x^2) L'' - 2x L' + N(N+1) L = 0.  Then symmetrise
 * xi_i <- (xi_i - xi_{N-i})/2.  Weights w_i = 2 / (N(N+1) L_N(xi_i)^2).     */
int or_gll(int N, double* xi, double* w) {
  if (N < 1) return OR_EINVAL;
  const double pi = 3.14159265358979323846;
  xi[0] = -1.0; xi[N] = 1.0;
  for (int i = 1; i < N; ++i) {
    double x = -cos(pi * i / N);
    for (int it = 0; it < 100; ++it) {
      double L, dL;
      legendre(N, x, &L, &dL);
      double d2L = (2.0 * x * dL - N * (N + 1.0) * L) / (1.0 - x * x);
      double dx = dL / d2L;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    xi[i] = x;
  }
  double* tmp = (double*)malloc(sizeof(double) * (N + 1));
  if (!tmp) return OR_ENOMEM;
  for (int i = 0; i <= N; ++i) tmp[i] = 0.5 * (xi[i] - xi[N - i]);
  for (int i = 0; i <= N; ++i) xi[i] = tmp[i];
  free(tmp);
  for (int i = 0; i <= N; ++i) {
    double L, dL;
    legendre(N, xi[i], &L, &dL);
    w[i] = 2.0 / (N * (N + 1.0) * L * L);
  }
  return OR_OK;
}

/* O2: GLL collocation derivative matrix, D[i*lx + j] = l_j'(xi_i):
 * D_ij = L_N(xi_i) / (L_N(xi_j) (xi_i - xi_j)), i != j;
 * D_00 = -N(N+1)/4, D_NN = +N(N+1)/4, other D_ii = 0.                       */
int or_dmat(int N, const double* xi, double* D) {
  if (N < 1) return OR_EINVAL;
  int lx = N + 1;
  for (int i = 0; i < lx; ++i) {
    for (int j = 0; j < lx; ++j) {
      double Li, Lj, d;
      legendre(N, xi[i], &Li, &d);
      legendre(N, xi[j], &Lj, &d);
      if (i != j) D[i * lx + j] = Li / (Lj * (xi[i] - xi[j]));
      else D[i * lx + j] = 0.0;
    }
  }
  D[0] = -N * (N + 1.0) / 4.0;
  D[N * lx + N] = N * (N + 1.0) / 4.0;
  return OR_OK;
}

#define IDX(i, j, k) ((i) + lx * ((j) + lx * (k)))

/* O4: geometric factors.  Per node: X[m][a] = dx_m/dr_a by D along r, s, t;
 * J = det X (error if <= 0); R = X^{-1}, R[a][m] = dr_a/dx_m;
 * G_ab = w_i w_j w_k J sum_m R[a][m] R[b][m]  (ab = 11,22,33,12,13,23);
 * B = w_i w_j w_k J.
 * Returns OR_EINVAL and the first offending element in *bad_elem if J <= 0. */
int or_geom(int64_t E, int N, const double* w, const double* D,
            const double* coords, double* G, double* B, int64_t* bad_elem) {
  if (N < 1 || E < 0) return OR_EINVAL;
  const int lx = N + 1, n3 = lx * lx * lx;
  int64_t bad = -1;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    const double* xm[3];
    for (int m = 0; m < 3; ++m) xm[m] = coords + (size_t)m * E * n3 + (size_t)e * n3;
    for (int k = 0; k < lx; ++k)
      for (int j = 0; j < lx; ++j)
        for (int i = 0; i < lx; ++i) {
          double X[3][3];
          for (int m = 0; m < 3; ++m) {
            double dr = 0.0, ds = 0.0, dt = 0.0;
            for (int l = 0; l < lx; ++l) {
              dr += D[i * lx + l] * xm[m][IDX(l, j, k)];
              ds += D[j * lx + l] * xm[m][IDX(i, l, k)];
              dt += D[k * lx + l] * xm[m][IDX(i, j, l)];
            }
            X[m][0] = dr; X[m][1] = ds; X[m][2] = dt;
          }
          double J = X[0][0] * (X[1][1] * X[2][2] - X[1][2] * X[2][1])
                   - X[0][1] * (X[1][0] * X[2][2] - X[1][2] * X[2][0])
                   + X[0][2] * (X[1][0] * X[2][1] - X[1][1] * X[2][0]);
          if (!(J > 0.0)) {
#pragma omp critical
            { if (bad < 0 || e < bad) bad = e; }
          }
          /* R = X^{-1} = adj(X) / J, adj(X)[a][m] = cofactor C[m][a]. */
          double R[3][3];
          R[0][0] = (X[1][1] * X[2][2] - X[1][2] * X[2][1]) / J;
          R[0][1] = (X[0][2] * X[2][1] - X[0][1] * X[2][2]) / J;
          R[0][2] = (X[0][1] * X[1][2] - X[0][2] * X[1][1]) / J;
          R[1][0] = (X[1][2] * X[2][0] - X[1][0] * X[2][2]) / J;
          R[1][1] = (X[0][0] * X[2][2] - X[0][2] * X[2][0]) / J;
          R[1][2] = (X[0][2] * X[1][0] - X[0][0] * X[1][2]) / J;
          R[2][0] = (X[1][0] * X[2][1] - X[1][1] * X[2][0]) / J;
          R[2][1] = (X[0][1] * X[2][0] - X[0][0] * X[2][1]) / J;
          R[2][2] = (X[0][0] * X[1][1] - X[0][1] * X[1][0]) / J;
          const double W = w[i] * w[j] * w[k];
          const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
          for (int c = 0; c < 6; ++c) {
            const int a = ab[c][0], b = ab[c][1];
            double s = 0.0;
            for (int m = 0; m < 3; ++m) s += R[a][m] * R[b][m];
            G[((size_t)e * 6 + c) * n3 + IDX(i, j, k)] = W * J * s;
          }
          B[(size_t)e * n3 + IDX(i, j, k)] = W * J;
        }
  }
  if (bad_elem) *bad_elem = bad;
  return bad >= 0 ? OR_EINVAL : OR_OK;
}

/* O5: local (unassembled) Helmholtz operator, element by element.
 *   ur(i,j,k) = sum_l D(i,l) u(l,j,k);  us = sum_l D(j,l) u(i,l,k);
 *   ut = sum_l D(k,l) u(i,j,l);
 *   q_a = h1 * sum_b G_ab u_b;
 *   w(i,j,k) = sum_l D(l,i) q_r(l,j,k) + sum_l D(l,j) q_s(i,l,k)
 *            + sum_l D(l,k) q_t(i,j,l) + h2 * B * u.
 * h1, h2: per-node arrays [E][lx^3] or NULL (then constants h1c, h2c).
 * B may be NULL when h2 is identically zero.                                */
int or_ax(int64_t E, int N, const double* D, const double* G, const double* B,
          const double* h1, const double* h2, double h1c, double h2c,
          const double* u, double* w) {
  if (N < 1 || E < 0) return OR_EINVAL;
  const int lx = N + 1, n3 = lx * lx * lx;
  int status = OR_OK;
#pragma omp parallel
  {
    double* qr = (double*)malloc(sizeof(double) * n3);
    double* qs = (double*)malloc(sizeof(double) * n3);
    double* qt = (double*)malloc(sizeof(double) * n3);
    if (!qr || !qs || !qt) {
#pragma omp critical
      status = OR_ENOMEM;
    } else {
#pragma omp for schedule(static)
      for (int64_t e = 0; e < E; ++e) {
        const double* ue = u + (size_t)e * n3;
        const double* Ge = G + (size_t)e * 6 * n3;
        for (int k = 0; k < lx; ++k)
          for (int j = 0; j < lx; ++j)
            for (int i = 0; i < lx; ++i) {
              double ur = 0.0, us = 0.0, ut = 0.0;
              for (int l = 0; l < lx; ++l) {
                ur += D[i * lx + l] * ue[IDX(l, j, k)];
                us += D[j * lx + l] * ue[IDX(i, l, k)];
                ut += D[k * lx + l] * ue[IDX(i, j, l)];
              }
              const int p = IDX(i, j, k);
              const double g11 = Ge[0 * n3 + p], g22 = Ge[1 * n3 + p], g33 = Ge[2 * n3 + p];
              const double g12 = Ge[3 * n3 + p], g13 = Ge[4 * n3 + p], g23 = Ge[5 * n3 + p];
              const double hh = h1 ? h1[(size_t)e * n3 + p] : h1c;
              qr[p] = hh * (g11 * ur + g12 * us + g13 * ut);
              qs[p] = hh * (g12 * ur + g22 * us + g23 * ut);
              qt[p] = hh * (g13 * ur + g23 * us + g33 * ut);
            }
        for (int k = 0; k < lx; ++k)
          for (int j = 0; j < lx; ++j)
            for (int i = 0; i < lx; ++i) {
              double s = 0.0;
              for (int l = 0; l < lx; ++l) s += D[l * lx + i] * qr[IDX(l, j, k)];
              for (int l = 0; l < lx; ++l) s += D[l * lx + j] * qs[IDX(i, l, k)];
              for (int l = 0; l < lx; ++l) s += D[l * lx + k] * qt[IDX(i, j, l)];
              const int p = IDX(i, j, k);
              const double hm = h2 ? h2[(size_t)e * n3 + p] : h2c;
              if (hm != 0.0) s += hm * B[(size_t)e * n3 + p] * ue[p];
              w[(size_t)e * n3 + p] = s;
            }
      }
    }
    free(qr); free(qs); free(qt);
  }
  return status;
}

/* O7: dssum (gather-scatter ADD): v_g = sum_{l: id(l)=g} u_l summed in
 * ascending l, then u_l <- v_{id(l)}.                                       */
int or_dssum(int64_t nloc, const int64_t* ids, int64_t nuniq, double* u) {
  double* v = (double*)calloc((size_t)(nuniq > 0 ? nuniq : 1), sizeof(double));
  if (!v) return OR_ENOMEM;
  for (int64_t l = 0; l < nloc; ++l) {
    if (ids[l] < 0 || ids[l] >= nuniq) { free(v); return OR_EINVAL; }
    v[ids[l]] += u[l];
  }
  for (int64_t l = 0; l < nloc; ++l) u[l] = v[ids[l]];
  free(v);
  return OR_OK;
}

/* O7: multiplicity m_g = number of copies; mult_l = 1 / m_{id(l)}.          */
int or_mult(int64_t nloc, const int64_t* ids, int64_t nuniq, double* mult) {
  int64_t* m = (int64_t*)calloc((size_t)(nuniq > 0 ? nuniq : 1), sizeof(int64_t));
  if (!m) return OR_ENOMEM;
  for (int64_t l = 0; l < nloc; ++l) m[ids[l]] += 1;
  for (int64_t l = 0; l < nloc; ++l) mult[l] = 1.0 / (double)m[ids[l]];
  free(m);
  return OR_OK;
}

/* O8: mask.  A local node is masked (mask=0) if ANY copy of its global node
 * lies on a face flagged Dirichlet in bc[E][6] (faces r-,r+,s-,s+,t-,t+);
 * otherwise mask=1.                                                          */
int or_mask(int64_t E, int N, const int8_t* bc, const int64_t* ids, int64_t nuniq,
            double* mask) {
  const int lx = N + 1, n3 = lx * lx * lx;
  char* dir = (char*)calloc((size_t)(nuniq > 0 ? nuniq : 1), 1);
  if (!dir) return OR_ENOMEM;
  for (int64_t e = 0; e < E; ++e)
    for (int k = 0; k < lx; ++k)
      for (int j = 0; j < lx; ++j)
        for (int i = 0; i < lx; ++i) {
          const int on[6] = {i == 0, i == N, j == 0, j == N, k == 0, k == N};
          int d = 0;
          for (int f = 0; f < 6; ++f)
            if (bc && bc[e * 6 + f] == 1 && on[f]) d = 1;
          if (d) dir[ids[(size_t)e * n3 + IDX(i, j, k)]] = 1;
        }
  const int64_t nloc = E * n3;
  for (int64_t l = 0; l < nloc; ++l) mask[l] = dir[ids[l]] ? 0.0 : 1.0;
  free(dir);
  return OR_OK;
}

/* O9: exact local diagonal of the Helmholtz operator,
 * d(i,j,k) = h1 [ sum_l D(l,i)^2 G11(l,j,k) + sum_l D(l,j)^2 G22(i,l,k)
 *               + sum_l D(l,k)^2 G33(i,j,l) + 2 D(i,i) D(j,j) G12(i,j,k)
 *               + 2 D(i,i) D(k,k) G13(i,j,k) + 2 D(j,j) D(k,k) G23(i,j,k) ]
 *          + h2 B(i,j,k),
 * with h1 taken at the quadrature node of each term; then d <- dssum(d);
 * dinv = 1/d, and dinv = 1 at masked nodes.  mask may be NULL (no mask).   */
int or_jacobi(int64_t E, int N, const double* D, const double* G, const double* B,
              const double* h1, const double* h2, double h1c, double h2c,
              const int64_t* ids, int64_t nuniq, const double* mask, double* dinv) {
  const int lx = N + 1, n3 = lx * lx * lx;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    const double* Ge = G + (size_t)e * 6 * n3;
    for (int k = 0; k < lx; ++k)
      for (int j = 0; j < lx; ++j)
        for (int i = 0; i < lx; ++i) {
          double s = 0.0;
#define H1AT(p) (h1 ? h1[(size_t)e * n3 + (p)] : h1c)
          for (int l = 0; l < lx; ++l) {
            const int p = IDX(l, j, k);
            s += D[l * lx + i] * D[l * lx + i] * H1AT(p) * Ge[0 * n3 + p];
          }
          for (int l = 0; l < lx; ++l) {
            const int p = IDX(i, l, k);
            s += D[l * lx + j] * D[l * lx + j] * H1AT(p) * Ge[1 * n3 + p];
          }
          for (int l = 0; l < lx; ++l) {
            const int p = IDX(i, j, l);
            s += D[l * lx + k] * D[l * lx + k] * H1AT(p) * Ge[2 * n3 + p];
          }
          const int p = IDX(i, j, k);
          s += 2.0 * D[i * lx + i] * D[j * lx + j] * H1AT(p) * Ge[3 * n3 + p];
          s += 2.0 * D[i * lx + i] * D[k * lx + k] * H1AT(p) * Ge[4 * n3 + p];
          s += 2.0 * D[j * lx + j] * D[k * lx + k] * H1AT(p) * Ge[5 * n3 + p];
#undef H1AT
          const double hm = h2 ? h2[(size_t)e * n3 + p] : h2c;
          if (hm != 0.0) s += hm * B[(size_t)e * n3 + p];
          dinv[(size_t)e * n3 + p] = s;
        }
  }
  const int64_t nloc = E * n3;
  int st = or_dssum(nloc, ids, nuniq, dinv);
  if (st) return st;
  for (int64_t l = 0; l < nloc; ++l) {
    if (mask && mask[l] == 0.0) dinv[l] = 1.0;
    else dinv[l] = 1.0 / dinv[l];
  }
  return OR_OK;
}

/* mult-weighted inner product <a,b> = sum_l mult_l a_l b_l (reading G10),
 * summed in ascending l.                                                    */
static double wdot(int64_t n, const double* mult, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t l = 0; l < n; ++l) s += mult[l] * a[l] * b[l];
  return s;
}

/* O10: Jacobi-preconditioned CG, in exactly this order:
 *   singular := (no masked node) and (h2 == 0 everywhere)
 *   b <- mask b;  if singular: b <- b - (sum mult b)/n_unique
 *   x <- 0; r <- b; bn <- sqrt(<r,r>); if bn == 0: iters=0, converged
 *   for k = 1..maxit:
 *     z <- dinv r; rtz <- <r,z>; beta <- (k==1 ? 0 : rtz/rtz_prev); rtz_prev <- rtz
 *     p <- z + beta p
 *     w <- mask dssum(Ax(p))
 *     pAp <- <w,p>; if not(pAp > 0): BREAKDOWN
 *     alpha <- rtz/pAp; x <- x + alpha p; r <- r - alpha w
 *     rn <- sqrt(<r,r>); if tol > 0 and rn <= tol bn: iters=k, converged; stop
 *   if singular: x <- x - (sum mult x)/n_unique
 * b is not modified (a copy is masked/projected).  mask may be NULL.
 * On exit *iters = iterations done, *rel_res = rn/bn, *converged = 0/1.     */
int or_pcg(int64_t E, int N, const double* D, const double* G, const double* B,
           const double* h1, const double* h2, double h1c, double h2c,
           const int64_t* ids, int64_t nuniq, const double* mult, const double* mask,
           const double* dinv, const double* b_in, double* x, double tol, int maxit,
           int* iters, double* rel_res, int* converged) {
  const int lx = N + 1, n3 = lx * lx * lx;
  const int64_t n = E * n3;
  int status = OR_OK;
  double *r = 0, *z = 0, *p = 0, *w = 0;
  r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  z = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  p = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!r || !z || !p || !w) { status = OR_ENOMEM; goto done; }

  int any_masked = 0;
  if (mask)
    for (int64_t l = 0; l < n; ++l) if (mask[l] == 0.0) { any_masked = 1; break; }
  int h2zero = 1;
  if (h2) { for (int64_t l = 0; l < n; ++l) if (h2[l] != 0.0) { h2zero = 0; break; } }
  else if (h2c != 0.0) h2zero = 0;
  const int singular = !any_masked && h2zero;

  for (int64_t l = 0; l < n; ++l) r[l] = mask ? mask[l] * b_in[l] : b_in[l];
  if (singular) {
    double s = 0.0;
    for (int64_t l = 0; l < n; ++l) s += mult[l] * r[l];
    const double mean = s / (double)nuniq;
    for (int64_t l = 0; l < n; ++l) r[l] -= mean;
  }
  for (int64_t l = 0; l < n; ++l) x[l] = 0.0;
  const double bn = sqrt(wdot(n, mult, r, r));
  *iters = 0; *rel_res = 0.0; *converged = 1;
  if (bn == 0.0) goto done;
  *converged = 0;

  double rtz_prev = 0.0, rn = bn;
  int k;
  for (k = 1; k <= maxit; ++k) {
    for (int64_t l = 0; l < n; ++l) z[l] = dinv[l] * r[l];
    const double rtz = wdot(n, mult, r, z);
    const double beta = (k == 1) ? 0.0 : rtz / rtz_prev;
    rtz_prev = rtz;
    for (int64_t l = 0; l < n; ++l) p[l] = z[l] + beta * p[l];
    status = or_ax(E, N, D, G, B, h1, h2, h1c, h2c, p, w);
    if (status) goto done;
    status = or_dssum(n, ids, nuniq, w);
    if (status) goto done;
    if (mask) for (int64_t l = 0; l < n; ++l) w[l] *= mask[l];
    const double pAp = wdot(n, mult, w, p);
    if (!(pAp > 0.0)) { status = OR_EBREAKDOWN; *iters = k; goto done; }
    const double alpha = rtz / pAp;
    for (int64_t l = 0; l < n; ++l) x[l] += alpha * p[l];
    for (int64_t l = 0; l < n; ++l) r[l] -= alpha * w[l];
    rn = sqrt(wdot(n, mult, r, r));
    *iters = k;
    if (tol > 0.0 && rn <= tol * bn) { *converged = 1; break; }
  }
  *rel_res = rn / bn;
  if (singular) {
    double s = 0.0;
    for (int64_t l = 0; l < n; ++l) s += mult[l] * x[l];
    const double mean = s / (double)nuniq;
    for (int64_t l = 0; l < n; ++l) x[l] -= mean;
  }
done:
  free(r); free(z); free(p); free(w);
  return status;
}

/* ------------------------------------------------------------------------ */
/* O12: restarted GMRES for the pressure system --
 * "we use restarted GMRES for the pressure solves with a hybrid-Schwarz
 * multigrid preconditioner".  The paper gives no algorithm;
 * this is GMRES(m) with RIGHT preconditioning exactly as in Saad, "Iterative
 * Methods for Sparse Linear Systems" (2nd ed., 2003), Algorithm 9.5, with the
 * Arnoldi process by modified Gram-Schmidt (Algorithm 6.2) and the
 * least-squares problem solved by Givens rotations (section 6.5.3).  The
 * preconditioner is M = diag(dinv) (point Jacobi; the hybrid-Schwarz
 * multigrid is the next step, reading R14).  Same conventions as
 * or_pcg (reading R10): A = mask . dssum . A_e, inner products mult-weighted,
 * x0 = 0, singular systems projected (b before, x after), relative stopping
 * rule on the residual estimate |g_{j+1}| <= tol ||b||, tol = 0 runs exactly
 * maxit iterations.
 *   b <- mask b ; if singular: b <- b - (sum mult b)/n_unique
 *   x <- 0 ; bn <- ||b|| ; r <- b ; beta <- bn ; if bn == 0: return
 *   iters <- 0
 *   while iters < maxit:                                  (one cycle)
 *     v_0 <- r / beta ; g <- (beta, 0, ..., 0)
 *     for j = 0 .. m-1:
 *       w <- mask dssum(A_e (dinv v_j))                    (w = A M v_j)
 *       for i = 0 .. j: h_ij <- <w, v_i> ; w <- w - h_ij v_i      (MGS)
 *       h_{j+1,j} <- ||w|| ; v_{j+1} <- w / h_{j+1,j} (if h_{j+1,j} != 0)
 *       for i < j: [h_ij, h_{i+1,j}] <- [c_i h_ij + s_i h_{i+1,j},
 *                                         -s_i h_ij + c_i h_{i+1,j}]
 *       d <- sqrt(h_jj^2 + h_{j+1,j}^2) ; c_j <- h_jj/d ; s_j <- h_{j+1,j}/d
 *       h_jj <- d ; g_{j+1} <- -s_j g_j ; g_j <- c_j g_j
 *       iters += 1
 *       stop the cycle if tol > 0 and |g_{j+1}| <= tol bn (converged),
 *         or h_{j+1,j} == 0 (happy breakdown: exact), or iters == maxit
 *     y <- H(0:k, 0:k)^{-1} g(0:k) (back substitution, k = cycle length)
 *     x <- x + dinv (sum_i y_i v_i)                        (x += M V y)
 *     r <- b - mask dssum(A_e x) ; beta <- ||r||
 *     if converged: break
 *   if singular: x <- x - (sum mult x)/n_unique
 * On exit *iters = Arnoldi steps done, *rel_res = ||r|| / bn of the TRUE
 * residual at the end, *converged = the estimate's test.  A zero pivot
 * (d == 0) is a breakdown (OR_EBREAKDOWN).                                 */
int or_gmres(int64_t E, int N, const double* D, const double* G, const double* B,
             const double* h1, const double* h2, double h1c, double h2c,
             const int64_t* ids, int64_t nuniq, const double* mult, const double* mask,
             const double* dinv, const double* b_in, double* x, int m, double tol, int maxit,
             int* iters, double* rel_res, int* converged) {
  const int lx = N + 1, n3 = lx * lx * lx;
  const int64_t n = E * n3;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  int status = OR_OK;
  if (m < 1) return OR_EINVAL;
  double *b = malloc(sizeof(double) * nn), *r = malloc(sizeof(double) * nn),
         *w = malloc(sizeof(double) * nn), *z = malloc(sizeof(double) * nn);
  double* V = malloc(sizeof(double) * nn * (size_t)(m + 1));
  double* H = calloc((size_t)(m + 1) * (size_t)m, sizeof(double)); /* H[i*m + j] */
  double *cs = calloc((size_t)m, sizeof(double)), *sn = calloc((size_t)m, sizeof(double));
  double *g = calloc((size_t)(m + 1), sizeof(double)), *y = calloc((size_t)m, sizeof(double));
  if (!b || !r || !w || !z || !V || !H || !cs || !sn || !g || !y) { status = OR_ENOMEM; goto done; }

  int any_masked = 0;
  if (mask)
    for (int64_t l = 0; l < n; ++l) if (mask[l] == 0.0) { any_masked = 1; break; }
  int h2zero = 1;
  if (h2) { for (int64_t l = 0; l < n; ++l) if (h2[l] != 0.0) { h2zero = 0; break; } }
  else if (h2c != 0.0) h2zero = 0;
  const int singular = !any_masked && h2zero;

  for (int64_t l = 0; l < n; ++l) b[l] = mask ? mask[l] * b_in[l] : b_in[l];
  if (singular) {
    double s = 0.0;
    for (int64_t l = 0; l < n; ++l) s += mult[l] * b[l];
    const double mean = s / (double)nuniq;
    for (int64_t l = 0; l < n; ++l) b[l] -= mean;
  }
  for (int64_t l = 0; l < n; ++l) { x[l] = 0.0; r[l] = b[l]; }
  const double bn = sqrt(wdot(n, mult, b, b));
  double beta = bn;
  *iters = 0; *rel_res = 0.0; *converged = 1;
  if (bn == 0.0) goto done;
  *converged = 0;

  int it = 0, conv = 0;
  while (it < maxit) {
    for (int64_t l = 0; l < n; ++l) V[l] = r[l] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    int k = 0;  /* Arnoldi steps in this cycle */
    for (int j = 0; j < m; ++j) {
      double* vj = V + (size_t)j * nn;
      for (int64_t l = 0; l < n; ++l) z[l] = dinv[l] * vj[l];
      status = or_ax(E, N, D, G, B, h1, h2, h1c, h2c, z, w);
      if (status) goto done;
      status = or_dssum(n, ids, nuniq, w);
      if (status) goto done;
      if (mask) for (int64_t l = 0; l < n; ++l) w[l] *= mask[l];
      for (int i = 0; i <= j; ++i) {
        const double* vi = V + (size_t)i * nn;
        const double hij = wdot(n, mult, w, vi);
        H[i * m + j] = hij;
        for (int64_t l = 0; l < n; ++l) w[l] -= hij * vi[l];
      }
      const double hn = sqrt(wdot(n, mult, w, w));
      H[(j + 1) * m + j] = hn;
      if (hn != 0.0) {
        double* vn = V + (size_t)(j + 1) * nn;
        for (int64_t l = 0; l < n; ++l) vn[l] = w[l] / hn;
      }
      for (int i = 0; i < j; ++i) {
        const double a = H[i * m + j], c = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * c;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
      }
      const double hjj = H[j * m + j], hj1 = H[(j + 1) * m + j];
      const double d = sqrt(hjj * hjj + hj1 * hj1);
      if (!(d > 0.0)) { status = OR_EBREAKDOWN; *iters = it + 1; goto done; }
      cs[j] = hjj / d;
      sn[j] = hj1 / d;
      H[j * m + j] = d;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++it;
      k = j + 1;
      if (tol > 0.0 && fabs(g[j + 1]) <= tol * bn) { conv = 1; break; }
      if (hn == 0.0 || it >= maxit) break;
    }
    /* y = H(0:k,0:k)^-1 g(0:k), back substitution */
    for (int i = k - 1; i >= 0; --i) {
      double s = g[i];
      for (int q = i + 1; q < k; ++q) s -= H[i * m + q] * y[q];
      y[i] = s / H[i * m + i];
    }
    /* x += M V y */
    for (int64_t l = 0; l < n; ++l) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += y[i] * V[(size_t)i * nn + l];
      x[l] += dinv[l] * s;
    }
    /* true residual r = b - A x */
    status = or_ax(E, N, D, G, B, h1, h2, h1c, h2c, x, w);
    if (status) goto done;
    status = or_dssum(n, ids, nuniq, w);
    if (status) goto done;
    for (int64_t l = 0; l < n; ++l) r[l] = b[l] - (mask ? mask[l] * w[l] : w[l]);
    beta = sqrt(wdot(n, mult, r, r));
    if (conv || beta == 0.0) break;
  }
  *iters = it;
  *rel_res = beta / bn;
  *converged = conv || beta == 0.0;
  if (singular) {
    double s = 0.0;
    for (int64_t l = 0; l < n; ++l) s += mult[l] * x[l];
    const double mean = s / (double)nuniq;
    for (int64_t l = 0; l < n; ++l) x[l] -= mean;
  }
done:
  free(b); free(r); free(w); free(z); free(V); free(H); free(cs); free(sn); free(g); free(y);
  return status;
}

/* ------------------------------------------------------------------------ */
/* the operators of one PnPn time step ("the
 * exact splitting of the velocity and pressure follows ... Karniadakis
 * (1991)"; PAPER.md:96 the TGV case, "time per time step").
 * The paper writes none of them; these are the standard SEM collocation /
 * weak forms (Deville, Fischer & Mund 2002) in the notation of O4/O5, with
 * MJ_am = w_i w_j w_k J (dr_a/dx_m) the mass-weighted metric terms (so that
 * G_ab = sum_m MJ_am (dr_b/dx_m)).                                          */

/* O13: MJ[(e*9 + 3a + m)*n3 + p] = W J R[a][m] (R = X^{-1}, as in or_geom). */
int or_metrics(int64_t E, int N, const double* w, const double* D, const double* coords, double* MJ) {
  if (N < 1 || E < 0) return OR_EINVAL;
  const int lx = N + 1, n3 = lx * lx * lx;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    const double* xm[3];
    for (int m = 0; m < 3; ++m) xm[m] = coords + (size_t)m * E * n3 + (size_t)e * n3;
    for (int k = 0; k < lx; ++k)
      for (int j = 0; j < lx; ++j)
        for (int i = 0; i < lx; ++i) {
          double X[3][3];
          for (int m = 0; m < 3; ++m) {
            double dr = 0.0, ds = 0.0, dt = 0.0;
            for (int l = 0; l < lx; ++l) {
              dr += D[i * lx + l] * xm[m][IDX(l, j, k)];
              ds += D[j * lx + l] * xm[m][IDX(i, l, k)];
              dt += D[k * lx + l] * xm[m][IDX(i, j, l)];
            }
            X[m][0] = dr; X[m][1] = ds; X[m][2] = dt;
          }
          const double J = X[0][0] * (X[1][1] * X[2][2] - X[1][2] * X[2][1])
                         - X[0][1] * (X[1][0] * X[2][2] - X[1][2] * X[2][0])
                         + X[0][2] * (X[1][0] * X[2][1] - X[1][1] * X[2][0]);
          double R[3][3];
          R[0][0] = (X[1][1] * X[2][2] - X[1][2] * X[2][1]) / J;
          R[0][1] = (X[0][2] * X[2][1] - X[0][1] * X[2][2]) / J;
          R[0][2] = (X[0][1] * X[1][2] - X[0][2] * X[1][1]) / J;
          R[1][0] = (X[1][2] * X[2][0] - X[1][0] * X[2][2]) / J;
          R[1][1] = (X[0][0] * X[2][2] - X[0][2] * X[2][0]) / J;
          R[1][2] = (X[0][2] * X[1][0] - X[0][0] * X[1][2]) / J;
          R[2][0] = (X[1][0] * X[2][1] - X[1][1] * X[2][0]) / J;
          R[2][1] = (X[0][1] * X[2][0] - X[0][0] * X[2][1]) / J;
          R[2][2] = (X[0][0] * X[1][1] - X[0][1] * X[1][0]) / J;
          const double WJ = w[i] * w[j] * w[k] * J;
          for (int a = 0; a < 3; ++a)
            for (int m = 0; m < 3; ++m) MJ[((size_t)e * 9 + 3 * a + m) * n3 + IDX(i, j, k)] = WJ * R[a][m];
        }
  }
  return OR_OK;
}

/* reference derivatives of one element field: d[a][p] = (D_a u)(p) */
static void ref_grad(int lx, const double* D, const double* ue, double* dr, double* ds, double* dt) {
  for (int k = 0; k < lx; ++k)
    for (int j = 0; j < lx; ++j)
      for (int i = 0; i < lx; ++i) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int l = 0; l < lx; ++l) {
          a += D[i * lx + l] * ue[IDX(l, j, k)];
          b += D[j * lx + l] * ue[IDX(i, l, k)];
          c += D[k * lx + l] * ue[IDX(i, j, l)];
        }
        dr[IDX(i, j, k)] = a; ds[IDX(i, j, k)] = b; dt[IDX(i, j, k)] = c;
      }
}

/* O14: mass-weighted collocation gradient, local:
 *   g_m(p) = sum_a MJ_am(p) (D_a u)(p),  g: [3][E][n3]  (= (v, du/dx_m) by GLL quadrature) */
int or_grad(int64_t E, int N, const double* D, const double* MJ, const double* u, double* g) {
  if (N < 1 || E < 0) return OR_EINVAL;
  const int lx = N + 1, n3 = lx * lx * lx;
  int status = OR_OK;
#pragma omp parallel
  {
    double* d = (double*)malloc(sizeof(double) * 3 * (size_t)n3);
    if (!d) {
#pragma omp atomic write
      status = OR_ENOMEM;
    }
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
      if (!d) continue;
      ref_grad(lx, D, u + (size_t)e * n3, d, d + n3, d + 2 * n3);
      for (int m = 0; m < 3; ++m)
        for (int p = 0; p < n3; ++p) {
          double s = 0.0;
          for (int a = 0; a < 3; ++a) s += MJ[((size_t)e * 9 + 3 * a + m) * n3 + p] * d[(size_t)a * n3 + p];
          g[(size_t)m * E * n3 + (size_t)e * n3 + p] = s;
        }
    }
    free(d);
  }
  return status;
}

/* O15: weak divergence, local: (grad v, f) by GLL quadrature,
 *   dv(p) = sum_a sum_l D(l, i_a(p)) q_a(l along a),  q_a = sum_m MJ_am f_m,
 * i.e. dv = D_r^T q_r + D_s^T q_s + D_t^T q_t  (f: [3][E][n3]). */
int or_wdiv(int64_t E, int N, const double* D, const double* MJ, const double* f, double* dv) {
  if (N < 1 || E < 0) return OR_EINVAL;
  const int lx = N + 1, n3 = lx * lx * lx;
  int status = OR_OK;
#pragma omp parallel
  {
    double* q = (double*)malloc(sizeof(double) * 3 * (size_t)n3);
    if (!q) {
#pragma omp atomic write
      status = OR_ENOMEM;
    }
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
      if (!q) continue;
      for (int a = 0; a < 3; ++a)
        for (int p = 0; p < n3; ++p) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m)
            s += MJ[((size_t)e * 9 + 3 * a + m) * n3 + p] * f[(size_t)m * E * n3 + (size_t)e * n3 + p];
          q[(size_t)a * n3 + p] = s;
        }
      for (int k = 0; k < lx; ++k)
        for (int j = 0; j < lx; ++j)
          for (int i = 0; i < lx; ++i) {
            double s = 0.0;
            for (int l = 0; l < lx; ++l) s += D[l * lx + i] * q[IDX(l, j, k)];
            for (int l = 0; l < lx; ++l) s += D[l * lx + j] * q[n3 + IDX(i, l, k)];
            for (int l = 0; l < lx; ++l) s += D[l * lx + k] * q[2 * n3 + IDX(i, j, l)];
            dv[(size_t)e * n3 + IDX(i, j, k)] = s;
          }
    }
    free(q);
  }
  return status;
}

/* O16: mass-weighted convection, local: c_i = sum_m u_m (g of u_i)_m
 *   = W J (u . grad) u_i at every node  (u, c: [3][E][n3]). */
int or_convect(int64_t E, int N, const double* D, const double* MJ, const double* u, double* c) {
  if (N < 1 || E < 0) return OR_EINVAL;
  const int lx = N + 1, n3 = lx * lx * lx;
  const size_t nl = (size_t)E * n3;
  int status = OR_OK;
#pragma omp parallel
  {
    double* d = (double*)malloc(sizeof(double) * 3 * (size_t)n3);
    if (!d) {
#pragma omp atomic write
      status = OR_ENOMEM;
    }
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
      if (!d) continue;
      for (int ci = 0; ci < 3; ++ci) {
        ref_grad(lx, D, u + ci * nl + (size_t)e * n3, d, d + n3, d + 2 * n3);
        for (int p = 0; p < n3; ++p) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m) {
            double gm = 0.0;
            for (int a = 0; a < 3; ++a) gm += MJ[((size_t)e * 9 + 3 * a + m) * n3 + p] * d[(size_t)a * n3 + p];
            s += u[m * nl + (size_t)e * n3 + p] * gm;
          }
          c[ci * nl + (size_t)e * n3 + p] = s;
        }
      }
    }
    free(d);
  }
  return status;
}
