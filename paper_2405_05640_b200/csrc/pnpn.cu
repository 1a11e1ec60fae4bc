// Operators of one velocity-pressure splitting time step (
// PAPER.md:72 "the exact splitting of the velocity and pressure follows ...
// Karniadakis (1991)"; "time per time step").  Readings R15 in
// DESIGN.md; the same forms as the oracle's O13-O16:
//   k_metrics  MJ_am = W J dr_a/dx_m, [E][9][n3] (once per mesh, on demand)
//   k_grad     g_m = sum_a MJ_am (D_a p)               (W J grad p, local)
//   k_wdiv     dv  = sum_a D_a^T (sum_m MJ_am f_m)     ((grad v, f), local)
//   k_convect  c_i = sum_m u_m sum_a MJ_am (D_a u_i)   (W J (u.grad)u_i, local)
// One CTA of lx^2 threads per element, thread (i,j) owning column (i,j,:)
// like the operator; the element's fields are staged in shared memory for
// the r/s contractions.  All three are bound by HBM (MJ is 72 B per node).
#include <stdint.h>

#include "device_common.cuh"

namespace sem {

__constant__ double c_Dn[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];
__constant__ double c_wn[kMaxN + 2][kMaxN + 1];

cudaError_t upload_basis_pnpn(int N, const double* D, const double* w) {
  const int lx = N + 1;
  cudaError_t e = cudaMemcpyToSymbol(c_Dn, D, sizeof(double) * lx * lx,
                                     sizeof(double) * lx * (kMaxN + 1) * (kMaxN + 1));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_wn, w, sizeof(double) * lx, sizeof(double) * lx * (kMaxN + 1));
}

template <int LX>
__global__ void __launch_bounds__(LX* LX) k_metrics(const double* __restrict__ coords, int64_t E,
                                                      double* __restrict__ MJ) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sx[3][N3];
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  for (int q = tid; q < N3; q += NT)
#pragma unroll
    for (int c = 0; c < 3; ++c) sx[c][q] = coords[(size_t)c * E * N3 + (size_t)e * N3 + q];
  __syncthreads();
  for (int k = 0; k < LX; ++k) {
    double X[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        dr += c_Dn[LX][i * LX + l] * sx[c][l + LX * (j + LX * k)];
        ds += c_Dn[LX][j * LX + l] * sx[c][i + LX * (l + LX * k)];
        dt += c_Dn[LX][k * LX + l] * sx[c][i + LX * (j + LX * l)];
      }
      X[c][0] = dr;
      X[c][1] = ds;
      X[c][2] = dt;
    }
    const double C00 = X[1][1] * X[2][2] - X[1][2] * X[2][1];
    const double C01 = X[1][2] * X[2][0] - X[1][0] * X[2][2];
    const double C02 = X[1][0] * X[2][1] - X[1][1] * X[2][0];
    const double J = X[0][0] * C00 + X[0][1] * C01 + X[0][2] * C02;
    const double WJ = c_wn[LX][i] * c_wn[LX][j] * c_wn[LX][k];
    // W J R[a][m] = W adj(X)[a][m]
    double A[3][3];
    A[0][0] = C00;
    A[1][0] = C01;
    A[2][0] = C02;
    A[0][1] = X[0][2] * X[2][1] - X[0][1] * X[2][2];
    A[1][1] = X[0][0] * X[2][2] - X[0][2] * X[2][0];
    A[2][1] = X[0][1] * X[2][0] - X[0][0] * X[2][1];
    A[0][2] = X[0][1] * X[1][2] - X[0][2] * X[1][1];
    A[1][2] = X[0][2] * X[1][0] - X[0][0] * X[1][2];
    A[2][2] = X[0][0] * X[1][1] - X[0][1] * X[1][0];
    (void)J;
    const int p = tid + NT * k;
    double* Me = MJ + (size_t)e * 9 * N3;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int m = 0; m < 3; ++m) Me[(3 * a + m) * N3 + p] = WJ * A[a][m];
  }
}

// reference derivatives of the tile s at column (i,j), plane k
template <int LX>
__device__ __forceinline__ void ref_d(const double* s, int i, int j, int k, double& dr, double& ds, double& dt) {
  constexpr int NT = LX * LX;
  dr = ds = dt = 0.0;
#pragma unroll
  for (int l = 0; l < LX; ++l) {
    dr = fma(c_Dn[LX][i * LX + l], s[l + LX * j + NT * k], dr);
    ds = fma(c_Dn[LX][j * LX + l], s[i + LX * l + NT * k], ds);
    dt = fma(c_Dn[LX][k * LX + l], s[i + LX * j + NT * l], dt);
  }
}

// g_m = sum_a MJ_am D_a p; g: [3][E][n3]
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_grad(const double* __restrict__ p, const double* __restrict__ MJ,
                                                   int64_t E, double* __restrict__ g) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sp[N3];
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  for (int q = tid; q < N3; q += NT) sp[q] = p[(size_t)e * N3 + q];
  __syncthreads();
  const double* Me = MJ + (size_t)e * 9 * N3;
  for (int k = 0; k < LX; ++k) {
    const int q = tid + NT * k;
    double d[3];
    ref_d<LX>(sp, i, j, k, d[0], d[1], d[2]);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) s = fma(Me[(3 * a + m) * N3 + q], d[a], s);
      g[(size_t)m * E * N3 + (size_t)e * N3 + q] = s;
    }
  }
}

// dv = sum_a D_a^T q_a, q_a = sum_m MJ_am f_m; f: [3][E][n3]
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_wdiv(const double* __restrict__ f, const double* __restrict__ MJ,
                                                   int64_t E, double* __restrict__ dv) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sq[3][N3];
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  const double* Me = MJ + (size_t)e * 9 * N3;
  for (int q = tid; q < N3; q += NT) {
    double fm[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) fm[m] = f[(size_t)m * E * N3 + (size_t)e * N3 + q];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) s = fma(Me[(3 * a + m) * N3 + q], fm[m], s);
      sq[a][q] = s;
    }
  }
  __syncthreads();
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      s = fma(c_Dn[LX][l * LX + i], sq[0][l + LX * j + NT * k], s);
      s = fma(c_Dn[LX][l * LX + j], sq[1][i + LX * l + NT * k], s);
      s = fma(c_Dn[LX][l * LX + k], sq[2][i + LX * j + NT * l], s);
    }
    dv[(size_t)e * N3 + tid + NT * k] = s;
  }
}

// c_i = sum_m u_m sum_a MJ_am D_a u_i; u, c: [3][E][n3]
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_convect(const double* __restrict__ u, const double* __restrict__ MJ,
                                                      int64_t E, double* __restrict__ c) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double su[3][N3];
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  for (int q = tid; q < N3; q += NT)
#pragma unroll
    for (int m = 0; m < 3; ++m) su[m][q] = u[(size_t)m * E * N3 + (size_t)e * N3 + q];
  __syncthreads();
  const double* Me = MJ + (size_t)e * 9 * N3;
  for (int k = 0; k < LX; ++k) {
    const int q = tid + NT * k;
    double M[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int m = 0; m < 3; ++m) M[a][m] = Me[(3 * a + m) * N3 + q];
    const double um[3] = {su[0][q], su[1][q], su[2][q]};
#pragma unroll
    for (int ci = 0; ci < 3; ++ci) {
      double d[3];
      ref_d<LX>(su[ci], i, j, k, d[0], d[1], d[2]);
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        double gm = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) gm = fma(M[a][m], d[a], gm);
        s = fma(um[m], gm, s);
      }
      c[(size_t)ci * E * N3 + (size_t)e * N3 + q] = s;
    }
  }
}

// elementwise pieces of the step
__global__ void k_pn_axpy(const double* __restrict__ a, double sa, const double* __restrict__ b, double sb,
                          double* __restrict__ out, int64_t n) {  // out = sa a + sb b
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = sa * a[q] + sb * b[q];
}
__global__ void k_pn_mul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                         int64_t n) {  // out = a b
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = a[q] * b[q];
}
__global__ void k_pn_div(double* __restrict__ a, const double* __restrict__ b, int64_t n) {  // a /= b
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    a[q] = a[q] / b[q];
}

static unsigned pn_grid(const sem_mesh* m, int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > (int64_t)m->nsm * 16) b = (int64_t)m->nsm * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_metrics(const sem_mesh* m, double* MJ, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_metrics<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(m->coords, m->E, MJ)));
  return cudaGetLastError();
}
cudaError_t launch_grad(const sem_mesh* m, const double* p, const double* MJ, double* g, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_grad<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(p, MJ, m->E, g)));
  return cudaGetLastError();
}
cudaError_t launch_wdiv(const sem_mesh* m, const double* f, const double* MJ, double* dv, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_wdiv<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(f, MJ, m->E, dv)));
  return cudaGetLastError();
}
cudaError_t launch_convect(const sem_mesh* m, const double* u, const double* MJ, double* c, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_convect<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(u, MJ, m->E, c)));
  return cudaGetLastError();
}
cudaError_t launch_pn_axpy(const sem_mesh* m, const double* a, double sa, const double* b, double sb, double* out,
                           int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  k_pn_axpy<<<pn_grid(m, n), 256, 0, s>>>(a, sa, b, sb, out, n);
  return cudaGetLastError();
}
cudaError_t launch_pn_mul(const sem_mesh* m, const double* a, const double* b, double* out, int64_t n,
                          cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  k_pn_mul<<<pn_grid(m, n), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}
cudaError_t launch_pn_div(const sem_mesh* m, double* a, const double* b, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  k_pn_div<<<pn_grid(m, n), 256, 0, s>>>(a, b, n);
  return cudaGetLastError();
}

}  // namespace sem
