// Kernels of the hybrid-Schwarz multigrid preconditioner (SURVEY 8(f) f2,
// PAPER.md:72; reading R16, the oracle's oracle/hsmg.py in the same order):
//   k_fdm       z_e = A~_e^-1 r_e, the fast-diagonalisation local solve of
//               the element's separable box operator (no assembly):
//               (S (x) S (x) S) [h1 (lam_i/Lx^2 + lam_j/Ly^2 + lam_k/Lz^2)
//               + h2]^-1 8/(Lx Ly Lz) (S (x) S (x) S)^T r_e
//   k_restrict  rc_e = (J^T (x) J^T (x) J^T)((r - w) / m)   (before dssum)
//   k_prolong   zf_e += (J (x) J (x) J) zc_e
//   k_scale     z *= 1/m (the averaging of the additive Schwarz sum)
// One CTA of lx^2 threads per element, thread (i, j) owning the column
// (i, j, :); the r and s contractions go through shared memory, t in
// registers (the operator's mapping, csrc/ax_kernel.cuh).
#include <stdint.h>

#include <algorithm>

#include "device_common.cuh"
#include "hsmg.h"

namespace sem {

#define HIDX(i, j, k) ((i) + LX * ((j) + LX * (k)))

template <int LX>
__global__ void __launch_bounds__(LX* LX) k_fdm(const double* __restrict__ r, double* __restrict__ z,
                                                const double* __restrict__ Lel, const double* __restrict__ fdm,
                                                double h1c, double h2c, const int* skip) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sS[LX * LX], sLam[LX];
  __shared__ double a[N3], b[N3];
  if (skip && *skip) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  sS[tid] = fdm[tid];
  if (tid < LX) sLam[tid] = fdm[NT + tid];
  const double* re = r + e * N3;
#pragma unroll
  for (int k = 0; k < LX; ++k) a[tid + NT * k] = re[tid + NT * k];
  const double Lx = Lel[3 * e], Ly = Lel[3 * e + 1], Lz = Lel[3 * e + 2];
  __syncthreads();
  // forward r: b[i(mode), j, k] = sum_l S[l][i] a[l, j, k]
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) s += sS[l * LX + i] * a[HIDX(l, j, k)];
    b[HIDX(i, j, k)] = s;
  }
  __syncthreads();
  // forward s: a[i, j(mode), k] = sum_l S[l][j] b[i, l, k]
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) s += sS[l * LX + j] * b[HIDX(i, l, k)];
    a[HIDX(i, j, k)] = s;
  }
  __syncthreads();
  // forward t, the diagonal scaling, backward t: the column in registers
  double col[LX], u[LX];
#pragma unroll
  for (int l = 0; l < LX; ++l) col[l] = a[HIDX(i, j, l)];
  const double cx = sLam[i] / (Lx * Lx), cy = sLam[j] / (Ly * Ly), vol = 8.0 / (Lx * Ly * Lz);
  const double iz2 = 1.0 / (Lz * Lz);
#pragma unroll
  for (int c = 0; c < LX; ++c) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) s += sS[l * LX + c] * col[l];
    u[c] = s / (h1c * (cx + cy + sLam[c] * iz2) + h2c) * vol;
  }
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < LX; ++c) s += sS[k * LX + c] * u[c];
    b[HIDX(i, j, k)] = s;
  }
  __syncthreads();
  // backward s: a[i, j, k] = sum_c S[j][c] b[i, c, k]
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < LX; ++c) s += sS[j * LX + c] * b[HIDX(i, c, k)];
    a[HIDX(i, j, k)] = s;
  }
  __syncthreads();
  // backward r: z[i, j, k] = sum_c S[i][c] a[c, j, k]
  double* ze = z + e * N3;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < LX; ++c) s += sS[i * LX + c] * a[HIDX(c, j, k)];
    ze[HIDX(i, j, k)] = s;
  }
}

// rc_e = (J^T (x) J^T (x) J^T)((r - w) mult); fine order LX, coarse lxc <= LX
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_restrict(const double* __restrict__ r, const double* __restrict__ w,
                                                     const double* __restrict__ mult, const double* __restrict__ J,
                                                     int lxc, double* __restrict__ rc, const int* skip) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sJ[LX * LX];
  __shared__ double a[N3], b[N3];
  if (skip && *skip) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  if (tid < LX * lxc) sJ[tid] = J[tid];  // J[a * lxc + b], a < LX (fine), b < lxc
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int64_t q = e * N3 + tid + NT * k;
    a[tid + NT * k] = (w ? r[q] - w[q] : r[q]) * mult[q];
  }
  __syncthreads();
  // r: b[ic, j, k] = sum_l J[l][ic] a[l, j, k]   (ic < lxc)
  if (i < lxc) {
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) s += sJ[l * lxc + i] * a[HIDX(l, j, k)];
      b[HIDX(i, j, k)] = s;
    }
  }
  __syncthreads();
  // s: a[ic, jc, k] = sum_l J[l][jc] b[ic, l, k]
  if (i < lxc && j < lxc) {
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) s += sJ[l * lxc + j] * b[HIDX(i, l, k)];
      a[HIDX(i, j, k)] = s;
    }
    // t: rc[ic, jc, kc] = sum_l J[l][kc] a[ic, jc, l]
    double col[LX];
#pragma unroll
    for (int l = 0; l < LX; ++l) col[l] = a[HIDX(i, j, l)];
    double* o = rc + e * (int64_t)lxc * lxc * lxc;
    for (int kc = 0; kc < lxc; ++kc) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) s += sJ[l * lxc + kc] * col[l];
      o[i + lxc * (j + lxc * kc)] = s;
    }
  }
}

// zf_e += (J (x) J (x) J) zc_e
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_prolong(const double* __restrict__ zc, const double* __restrict__ J,
                                                    int lxc, double* __restrict__ zf, const int* skip) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sJ[LX * LX];
  __shared__ double a[N3], b[N3];
  if (skip && *skip) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  const int nc3 = lxc * lxc * lxc;
  if (tid < LX * lxc) sJ[tid] = J[tid];
  const double* ze = zc + e * (int64_t)nc3;
  for (int q = tid; q < nc3; q += NT) a[q] = ze[q];  // packed [kc][jc][ic] with stride lxc
  __syncthreads();
  // r: b[i, jc, kc] = sum_c J[i][c] a[c, jc, kc]   (packed coarse strides)
  for (int q = j; q < lxc * lxc; q += LX) {  // q = jc + lxc kc
    double s = 0.0;
    for (int c = 0; c < lxc; ++c) s += sJ[i * lxc + c] * a[c + lxc * q];
    b[i + LX * q] = s;  // b[i][q] with row stride LX
  }
  __syncthreads();
  // s: a[i, j, kc] = sum_c J[j][c] b[i, c, kc]
  for (int kc = 0; kc < lxc; ++kc) {
    double s = 0.0;
    for (int c = 0; c < lxc; ++c) s += sJ[j * lxc + c] * b[i + LX * (c + lxc * kc)];
    a[HIDX(i, j, kc)] = s;
  }
  // t (registers): zf[i, j, k] += sum_c J[k][c] a[i, j, c]   (own column: no barrier)
  double col[LX];
  for (int c = 0; c < lxc; ++c) col[c] = a[HIDX(i, j, c)];
  double* zo = zf + e * N3;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
    for (int c = 0; c < lxc; ++c) s += sJ[k * lxc + c] * col[c];
    zo[HIDX(i, j, k)] += s;
  }
}

__global__ void k_scale_mult(double* __restrict__ z, const double* __restrict__ mult, int64_t n, const int* skip) {
  if (skip && *skip) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    z[q] *= mult[q];
}

#undef HIDX

cudaError_t launch_fdm(const sem_mesh* m, const double* r, double* z, const double* L, const double* fdm, double h1c,
                       double h2c, const int* skip, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_fdm<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(r, z, L, fdm, h1c, h2c, skip)));
  return cudaGetLastError();
}

cudaError_t launch_restrict(const sem_mesh* mf, int lxc, const double* r, const double* w, const double* J,
                            double* rc, const int* skip, cudaStream_t s) {
  if (mf->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(mf);
  SEM_LX_DISPATCH(mf->lx,
                  (k_restrict<LX><<<(unsigned)mf->E, dim3(LX, LX), 0, s>>>(r, w, mf->mult, J, lxc, rc, skip)));
  return cudaGetLastError();
}

cudaError_t launch_prolong_add(const sem_mesh* mf, int lxc, const double* zc, const double* J, double* zf,
                               const int* skip, cudaStream_t s) {
  if (mf->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(mf);
  SEM_LX_DISPATCH(mf->lx, (k_prolong<LX><<<(unsigned)mf->E, dim3(LX, LX), 0, s>>>(zc, J, lxc, zf, skip)));
  return cudaGetLastError();
}

cudaError_t launch_scale_mult(const sem_mesh* m, double* z, const int* skip, cudaStream_t s) {
  if (m->nloc == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  const unsigned blocks = (unsigned)std::min<int64_t>((int64_t)m->nsm * 8, (m->nloc + 255) / 256);
  k_scale_mult<<<blocks, 256, 0, s>>>(z, m->mult, m->nloc, skip);
  return cudaGetLastError();
}

}  // namespace sem
