// Restarted GMRES(m) with right (Jacobi) preconditioning for the pressure
// system -- "we use restarted GMRES for the pressure solves";
// SURVEY.md 8(f) row f2, reading R14.  Same algorithm as the
// oracle's or_gmres (Saad 2003, Alg. 9.5; Givens rotations, section 6.5.3)
// except that the Arnoldi step orthogonalises by classical Gram-Schmidt with
// one re-orthogonalisation (CGS2: equal to modified Gram-Schmidt in exact
// arithmetic, and two fused vector passes instead of j+1 dependent ones):
//   w  = mask dssum(A_e z_j),  z_j = dinv v_j           (operator, fused gs)
//   h  = V^T w                                          k_gm_dots
//   w1 = w - V h ; h2 = V^T w1 ; nn = <w1, w1>          k_gm_update
//   H(:, j) = h + h2 ; sigma = sqrt(nn - |h2|^2) ; Givens ; stopping test
//                                                       k_gm_givens
//   v_{j+1} = (w1 - V h2) / sigma ; z_{j+1} = dinv v_{j+1}   k_gm_next
// and per cycle: y = H^-1 g (k_gm_solve), x += dinv (V y) (k_gm_xupd), the
// true residual r = b - mask dssum(A_e x) and v_0 = r / |r| (k_gm_resid,
// k_gm_start).  Inner products are mult-weighted (reading R10); every
// reduction is deterministic (per-block partials, the last block sums them
// in block order).  All scalars stay on the device; the host only reads
// them once per cycle.
#include <stdint.h>

#include <algorithm>

#include "device_common.cuh"
#include "gmres.h"

namespace sem {

constexpr int kGmThreads = 256;

static unsigned gm_blocks(const sem_mesh* m) {
  return (unsigned)std::min<int64_t>((int64_t)m->nsm * 4, kGmMaxBlocks);
}

// h[k] = sum_l mult_l w_l V_k,l for k < nvec (NV >= nvec)
template <int NV>
__global__ void __launch_bounds__(kGmThreads) k_gm_dots(const double* __restrict__ w, const double* __restrict__ V,
                                                        int64_t ld, int nvec, const double* __restrict__ mult,
                                                        int64_t n, double* part, unsigned* ticket, double* out,
                                                        const GmScalars* gs) {
  __shared__ double s_red[32 * NV];
  __shared__ int s_flag;
  if (gs->cycle_stop) return;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double wq = mult[q] * w[q];
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (k < nvec) acc[k] += wq * V[k * ld + q];
  }
  grid_sum_last_block<NV>(acc, part, ticket, out, s_red, &s_flag);
}

// w <- w - sum_k c_k V_k ; then h2[k] = <w, V_k> (k < nvec) and nn = <w, w>
// into out[0..nvec) and out[NV]
template <int NV>
__global__ void __launch_bounds__(kGmThreads) k_gm_update(double* __restrict__ w, const double* __restrict__ V,
                                                          int64_t ld, int nvec, const double* __restrict__ c,
                                                          const double* __restrict__ mult, int64_t n, double* part,
                                                          unsigned* ticket, double* out, const GmScalars* gs) {
  __shared__ double s_red[32 * (NV + 1)];
  __shared__ double s_c[NV];
  __shared__ int s_flag;
  if (gs->cycle_stop) return;
  if (threadIdx.x < NV) s_c[threadIdx.x] = threadIdx.x < nvec ? c[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[NV + 1];
#pragma unroll
  for (int k = 0; k <= NV; ++k) acc[k] = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double v[NV];
    double wq = w[q];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      v[k] = (k < nvec) ? V[k * ld + q] : 0.0;
      wq -= s_c[k] * v[k];
    }
    w[q] = wq;
    const double mw = mult[q] * wq;
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += mw * v[k];
    acc[NV] += mw * wq;
  }
  grid_sum_last_block<NV + 1>(acc, part, ticket, out, s_red, &s_flag);
}

// v_{j+1} = (w - sum_k c_k V_k) / sigma ; z = dinv v_{j+1}
template <int NV>
__global__ void __launch_bounds__(kGmThreads) k_gm_next(const double* __restrict__ w, const double* V, int64_t ld,
                                                        int nvec, const double* __restrict__ c,
                                                        const double* __restrict__ dinv, int64_t n, double* vout,
                                                        double* __restrict__ z, const GmScalars* gs) {
  __shared__ double s_c[NV];
  if (gs->cycle_stop || !(gs->sigma > 0.0)) return;
  if (threadIdx.x < NV) s_c[threadIdx.x] = threadIdx.x < nvec ? c[threadIdx.x] : 0.0;
  __syncthreads();
  const double is = 1.0 / gs->sigma;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double wq = w[q];
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (k < nvec) wq -= s_c[k] * V[k * ld + q];
    const double vq = wq * is;
    vout[q] = vq;
    if (z) z[q] = dinv[q] * vq;
  }
}

// Arnoldi column j from the reductions, Givens rotations, stopping test
__global__ void k_gm_givens(GmScalars* gs) {
  if (gs->cycle_stop) return;
  const int M = gs->restart, j = gs->j;
  double h2n = 0.0;
  for (int i = 0; i <= j; ++i) {
    gs->H[i * M + j] = gs->h[i] + gs->h2[i];
    h2n += gs->h2[i] * gs->h2[i];
  }
  const double s2 = gs->nn - h2n;
  const double sigma = s2 > 0.0 ? sqrt(s2) : 0.0;
  gs->sigma = sigma;
  gs->H[(j + 1) * M + j] = sigma;
  for (int i = 0; i < j; ++i) {
    const double a = gs->H[i * M + j], c = gs->H[(i + 1) * M + j];
    gs->H[i * M + j] = gs->cs[i] * a + gs->sn[i] * c;
    gs->H[(i + 1) * M + j] = -gs->sn[i] * a + gs->cs[i] * c;
  }
  const double hjj = gs->H[j * M + j], hj1 = gs->H[(j + 1) * M + j];
  const double d = sqrt(hjj * hjj + hj1 * hj1);
  if (!(d > 0.0)) {
    gs->breakdown = 1;
    gs->done = 1;
    gs->cycle_stop = 1;
    return;
  }
  gs->cs[j] = hjj / d;
  gs->sn[j] = hj1 / d;
  gs->H[j * M + j] = d;
  gs->H[(j + 1) * M + j] = 0.0;
  gs->g[j + 1] = -gs->sn[j] * gs->g[j];
  gs->g[j] = gs->cs[j] * gs->g[j];
  gs->it += 1;
  gs->k = j + 1;
  gs->j = j + 1;
  if (gs->tol > 0.0 && fabs(gs->g[j + 1]) <= gs->tol * gs->bn) {
    gs->converged = 1;
    gs->done = 1;
  }
  if (gs->it >= gs->maxit) gs->done = 1;
  if (gs->done || !(sigma > 0.0) || gs->j >= M) gs->cycle_stop = 1;
}

// y = H(0:k, 0:k)^-1 g(0:k)
__global__ void k_gm_solve(GmScalars* gs) {
  const int M = gs->restart, k = gs->k;
  for (int i = k - 1; i >= 0; --i) {
    double s = gs->g[i];
    for (int q = i + 1; q < k; ++q) s -= gs->H[i * M + q] * gs->y[q];
    gs->y[i] = s / gs->H[i * M + i];
  }
}

// x += dinv (sum_{k0 <= i < k0 + NV, i < k} y_i V_i); flexible: x += sum y_i Z_i
// (V = Z, dinv = NULL)
template <int NV>
__global__ void __launch_bounds__(kGmThreads) k_gm_xupd(double* __restrict__ x, const double* __restrict__ V,
                                                        int64_t ld, int k0, const double* __restrict__ dinv,
                                                        int64_t n, const GmScalars* gs) {
  __shared__ double s_y[NV];
  const int k = gs->k;
  if (k <= k0) return;
  if (threadIdx.x < NV) s_y[threadIdx.x] = (k0 + (int)threadIdx.x < k) ? gs->y[k0 + threadIdx.x] : 0.0;
  __syncthreads();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (k0 + i < k) s += s_y[i] * V[(k0 + i) * ld + q];
    x[q] += dinv ? dinv[q] * s : s;
  }
}

// v_0 <- b - w (w = mask dssum A x); out = <v_0, v_0>
__global__ void __launch_bounds__(kGmThreads) k_gm_resid(const double* __restrict__ b, const double* __restrict__ w,
                                                         double* __restrict__ v0, const double* __restrict__ mult,
                                                         int64_t n, double* part, unsigned* ticket, double* out) {
  __shared__ double s_red[32];
  __shared__ int s_flag;
  double acc[1] = {0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double r = b[q] - w[q];
    v0[q] = r;
    acc[0] += mult[q] * r * r;
  }
  grid_sum_last_block<1>(acc, part, ticket, out, s_red, &s_flag);
}

// a new cycle: beta = sqrt(out), v_0 /= beta, z = dinv v_0, g = (beta, 0..)
__global__ void __launch_bounds__(kGmThreads) k_gm_start(double* __restrict__ v0, const double* __restrict__ dinv,
                                                         double* __restrict__ z, int64_t n, const GmScalars* gs,
                                                         int first) {
  const double beta = sqrt(gs->nn);
  if (gs->done || !(beta > 0.0)) return;
  const double ib = 1.0 / beta;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double v = v0[q] * ib;
    v0[q] = v;
    if (z) z[q] = dinv[q] * v;
  }
  (void)first;
}

// host-side scalar bookkeeping of a new cycle (one thread): after every block
// of k_gm_start has read nn
__global__ void k_gm_cycle(GmScalars* gs, int first) {
  const double beta = sqrt(gs->nn);
  if (first) gs->bn = beta;
  gs->beta = beta;
  if (first && !(beta > 0.0)) {
    gs->done = 1;
    gs->converged = 1;
  }
  if (!first && (gs->converged || !(beta > 0.0))) gs->done = 1;
  if (gs->it >= gs->maxit) gs->done = 1;
  for (int i = 0; i <= gs->restart; ++i) gs->g[i] = 0.0;
  gs->g[0] = beta;
  gs->j = 0;
  gs->k = 0;
  gs->cycle_stop = gs->done;
}

// ---- launchers ----------------------------------------------------------
#define GM_NV_DISPATCH(nvec, CALL)                     \
  do {                                                 \
    if ((nvec) <= 8) {                                 \
      constexpr int NV = 8;                            \
      CALL;                                            \
    } else if ((nvec) <= 16) {                         \
      constexpr int NV = 16;                           \
      CALL;                                            \
    } else {                                           \
      constexpr int NV = 32;                           \
      CALL;                                            \
    }                                                  \
  } while (0)

cudaError_t gm_launch_dots(sem_mesh* m, GmState* G, int nvec, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  GM_NV_DISPATCH(nvec, (k_gm_dots<NV><<<gm_blocks(m), kGmThreads, 0, s>>>(
                           m->w, G->V, m->nloc, nvec, m->mult, m->nloc, G->part, G->ticket, G->gs->h, G->gs)));
  return cudaGetLastError();
}

cudaError_t gm_launch_update(sem_mesh* m, GmState* G, int nvec, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  // the reduction writes [h2 (NV), nn]: copy nn into place after (k_gm_givens reads gs->nn)
  GM_NV_DISPATCH(nvec, (k_gm_update<NV><<<gm_blocks(m), kGmThreads, 0, s>>>(
                           m->w, G->V, m->nloc, nvec, G->gs->h, m->mult, m->nloc, G->part, G->ticket,
                           G->red, G->gs)));
  return cudaGetLastError();
}

__global__ void k_gm_unpack(GmScalars* gs, const double* red, int nvec, int NV) {
  if (gs->cycle_stop) return;
  for (int k = 0; k < nvec; ++k) gs->h2[k] = red[k];
  gs->nn = red[NV];
}

cudaError_t gm_launch_unpack(sem_mesh* m, GmState* G, int nvec, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  const int NV = nvec <= 8 ? 8 : (nvec <= 16 ? 16 : 32);
  k_gm_unpack<<<1, 1, 0, s>>>(G->gs, G->red, nvec, NV);
  return cudaGetLastError();
}

cudaError_t gm_launch_givens(sem_mesh* m, GmState* G, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_gm_givens<<<1, 1, 0, s>>>(G->gs);
  return cudaGetLastError();
}

cudaError_t gm_launch_next(sem_mesh* m, GmState* G, int j, bool flex, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  const int nvec = j + 1;
  GM_NV_DISPATCH(nvec, (k_gm_next<NV><<<gm_blocks(m), kGmThreads, 0, s>>>(
                           m->w, G->V, m->nloc, nvec, G->gs->h2, m->dinv, m->nloc, G->V + (int64_t)(j + 1) * m->nloc,
                           flex ? nullptr : G->z, G->gs)));
  return cudaGetLastError();
}

cudaError_t gm_launch_cycle_end(sem_mesh* m, GmState* G, double* x, bool flex, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_gm_solve<<<1, 1, 0, s>>>(G->gs);
  for (int k0 = 0; k0 < G->restart; k0 += 16) {
    SEM_COUNT_LAUNCH(m);
    k_gm_xupd<16><<<gm_blocks(m), kGmThreads, 0, s>>>(x, flex ? G->Z : G->V, m->nloc, k0,
                                                     flex ? nullptr : m->dinv, m->nloc, G->gs);
  }
  return cudaGetLastError();
}

cudaError_t gm_launch_resid(sem_mesh* m, GmState* G, const double* b, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_gm_resid<<<gm_blocks(m), kGmThreads, 0, s>>>(b, m->w, G->V, m->mult, m->nloc, G->part, G->ticket, &G->gs->nn);
  return cudaGetLastError();
}

cudaError_t gm_launch_start(sem_mesh* m, GmState* G, int first, bool flex, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_gm_start<<<gm_blocks(m), kGmThreads, 0, s>>>(G->V, m->dinv, flex ? nullptr : G->z, m->nloc, G->gs, first);
  SEM_COUNT_LAUNCH(m);
  k_gm_cycle<<<1, 1, 0, s>>>(G->gs, first);
  return cudaGetLastError();
}

}  // namespace sem
