// Kernels of the hybrid-Schwarz multigrid preconditioner (SURVEY 8(f) f2,
// PAPER.md:72; reading R16, the oracle's oracle/hsmg.py in the same order):
//   k_fdm       z_e = A~_e^-1 r_e, the fast-diagonalisation local solve of
//               the element's separable box operator (no assembly):
//               (S (x) S (x) S) [h1 (lam_i/Lx^2 + lam_j/Ly^2 + lam_k/Lz^2)
//               + h2]^-1 8/(Lx Ly Lz) (S (x) S (x) S)^T r_e
//   k_restrict  rc_e = (J^T (x) J^T (x) J^T)((r - w) / m)   (before dssum)
//   k_prolong   zf_e += (J (x) J (x) J) zc_e
// One CTA of lx^2 threads per element, thread (i, j) owning the column
// (i, j, :); the r and s contractions go through shared memory, t in
// registers (the operator's mapping, csrc/ax_kernel.cuh).
#include <stdint.h>

#include <algorithm>

#include "device_common.cuh"
#include "hsmg.h"

#ifndef SEM_FDM_DMMA
#define SEM_FDM_DMMA 1  // lx = 8 local solves on the fp64 tensor cores (0: CUDA cores, for A/B)
#endif

namespace sem {

#define HIDX(i, j, k) ((i) + LX * ((j) + LX * (k)))

// elements per CTA of the per-element kernels: one at lx >= 5, several at
// the coarse orders (a 16- or 4-thread CTA per element leaves the SM's block
// slots full and the kernel latency-bound)
__host__ __device__ constexpr int hsmg_epb(int lx) { return lx <= 4 ? 64 / (lx * lx) : 1; }
static unsigned hsmg_grid(int64_t E, int epb) { return (unsigned)((E + epb - 1) / epb); }

template <int LX, int EPB>
__global__ void __launch_bounds__(LX * LX * EPB) k_fdm(const double* __restrict__ r, double* __restrict__ z,
                                                const double* __restrict__ Lel, const double* __restrict__ fdm,
                                                double h1c, double h2c, const int* skip, int64_t E) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sS[LX * LX], sLam[LX];
  __shared__ double a_[EPB][N3], b_[EPB][N3];
  double* a = a_[threadIdx.z];
  double* b = b_[threadIdx.z];
  if (skip && *skip) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e0 = (int64_t)blockIdx.x * EPB + threadIdx.z;
  const bool live = e0 < E;
  const int64_t e = live ? e0 : E - 1;  // a spare slot recomputes the last element, stores nothing
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
    if (live) ze[HIDX(i, j, k)] = s;
  }
}

// lx = 8: the same local solve on the fp64 tensor cores (DMMA, mma.sync
// m8n8k4.f64; tcgen05 has no fp64 kind).  Each of the six contractions of an
// element is the GEMM Out(8 x 64) = M(8 x 8) . T(8 x 64) with M = S^T
// (forward) or S (backward) and T the element tile viewed with the
// contracted direction as rows: 8 N-tiles x 2 K-steps = 16 DMMAs, split over
// the element's two warps (4 N-tiles each).  M's fragments are per-lane
// constants (4 doubles); T's come from shared memory; the diagonal scaling
// rides on the store of the forward t-contraction and the backward
// r-contraction stores straight to global memory.  Three elements per CTA.
// Fragment layouts (PTX ISA, m8n8k4 .f64): A row = lane/4, col = lane%4;
// B row = lane%4, col = lane/4; C/D row = lane/4, cols = 2 (lane%4) + {0,1}.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// shared-memory slot of node (i, j, k): rows padded to 12, planes to 104
// doubles (bank-conflict search over the 96 fragment accesses and the tile
// load: 288 wavefronts against 448 unpadded, 224 the minimum)
constexpr int kF8Y = 12, kF8Z = 104, kF8Tile = 8 * kF8Z;
__device__ __forceinline__ int fdm8_slot(int i, int j, int k) { return i + kF8Y * j + kF8Z * k; }

// slot (shared) or node index (global) of (contracted index l, column col)
// for contraction direction DIR
template <int DIR, bool GLOBAL = false>
__device__ __forceinline__ int fdm8_addr(int l, int col) {
  int i, j, k;
  if (DIR == 0) {
    i = l, j = col & 7, k = col >> 3;  // col = j + 8 k
  } else if (DIR == 1) {
    i = col & 7, j = l, k = col >> 3;  // col = i + 8 k
  } else {
    i = col & 7, j = col >> 3, k = l;  // col = i + 8 j
  }
  return GLOBAL ? i + 8 * j + 64 * k : fdm8_slot(i, j, k);
}

template <int DIR, int MODE>  // MODE 0: store to shared, 1: scaled store to shared, 2: store to global
__device__ __forceinline__ void fdm8_contract(const double* in, double* out, double a0, double a1, int lane, int nt0,
                                              const double* lam, double cx, double cy, double cz, double h1c,
                                              double h2c, double vol) {
  const int bl = lane & 3, bc = lane >> 2;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int nt = nt0 + t;
    const int colb = nt * 8 + bc;
    double d0 = 0.0, d1 = 0.0;
    dmma884(d0, d1, a0, in[fdm8_addr<DIR>(bl, colb)]);
    dmma884(d0, d1, a1, in[fdm8_addr<DIR>(bl + 4, colb)]);
    const int c = bc, col0 = nt * 8 + 2 * bl;
    if (MODE == 1) {  // DIR 2 forward: node (i, j, c) with col = i + 8 j
      const int i0 = col0 & 7, j0 = col0 >> 3;
      const double base = h1c * (lam[j0] * cy + lam[c] * cz) + h2c;
      d0 *= vol / (base + h1c * lam[i0] * cx);
      d1 *= vol / (base + h1c * lam[i0 + 1] * cx);
    }
    if (MODE == 2) {
      out[fdm8_addr<DIR, true>(c, col0)] = d0;
      out[fdm8_addr<DIR, true>(c, col0 + 1)] = d1;
    } else {
      out[fdm8_addr<DIR>(c, col0)] = d0;
      out[fdm8_addr<DIR>(c, col0 + 1)] = d1;
    }
  }
}

constexpr int kF8Elems = 3;  // elements per CTA (two warps each)
__global__ void __launch_bounds__(64 * kF8Elems, 5) k_fdm8_dmma(const double* __restrict__ r, double* __restrict__ z,
                                                            const double* __restrict__ Lel,
                                                            const double* __restrict__ fdm, double h1c, double h2c,
                                                            int64_t E, const int* skip) {
  constexpr int N3 = 512;
  __shared__ __align__(16) double buf[kF8Elems][2][kF8Tile];
  __shared__ double sLam[8];
  if (skip && *skip) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int le = warp >> 1, nt0 = (warp & 1) * 4;  // local element, its N-tile half
  const int64_t e = (int64_t)blockIdx.x * kF8Elems + le;
  const bool live = e < E;
  if (tid < 8) sLam[tid] = fdm[64 + tid];
  // M fragments: forward S^T (a0 = S[lane%4][lane/4], a1 = S[lane%4 + 4][lane/4]),
  // backward S (a0 = S[lane/4][lane%4], a1 = S[lane/4][lane%4 + 4])
  const int ar = lane >> 2, ac = lane & 3;
  const double f0 = fdm[ac * 8 + ar], f1 = fdm[(ac + 4) * 8 + ar];
  const double b0 = fdm[ar * 8 + ac], b1 = fdm[ar * 8 + ac + 4];
  double* A = buf[le][0];
  double* B = buf[le][1];
  const int et = tid & 63;  // thread within the element's 64
  if (live) {
    const double* re = r + e * N3;
#pragma unroll
    for (int q = 0; q < 8; ++q) A[fdm8_slot(et & 7, et >> 3, q)] = re[et + 64 * q];
  }
  double cx = 0.0, cy = 0.0, cz = 0.0, vol = 0.0;
  if (live) {
    const double Lx = Lel[3 * e], Ly = Lel[3 * e + 1], Lz = Lel[3 * e + 2];
    cx = 1.0 / (Lx * Lx);
    cy = 1.0 / (Ly * Ly);
    cz = 1.0 / (Lz * Lz);
    vol = 8.0 / (Lx * Ly * Lz);
  }
  __syncthreads();
  fdm8_contract<0, 0>(A, B, f0, f1, lane, nt0, sLam, cx, cy, cz, h1c, h2c, vol);
  __syncthreads();
  fdm8_contract<1, 0>(B, A, f0, f1, lane, nt0, sLam, cx, cy, cz, h1c, h2c, vol);
  __syncthreads();
  fdm8_contract<2, 1>(A, B, f0, f1, lane, nt0, sLam, cx, cy, cz, h1c, h2c, vol);
  __syncthreads();
  fdm8_contract<2, 0>(B, A, b0, b1, lane, nt0, sLam, cx, cy, cz, h1c, h2c, vol);
  __syncthreads();
  fdm8_contract<1, 0>(A, B, b0, b1, lane, nt0, sLam, cx, cy, cz, h1c, h2c, vol);
  __syncthreads();
  if (live) fdm8_contract<0, 2>(B, z + e * N3, b0, b1, lane, nt0, sLam, cx, cy, cz, h1c, h2c, vol);
}

// rc_e = (J^T (x) J^T (x) J^T)(r mult - mask w); fine order LX, coarse
// lxc <= LX.  w is the UNASSEMBLED A_e z: the coarse dssum that follows
// assembles it, since dssum(J^T y) = P^T Q^T y for any local y (the local
// interpolation of a continuous coarse field is continuous), so the
// restricted residual equals R(r - mask dssum(A_e z)) of reading R16
// without a fine-level gather-scatter pass
template <int LX, int EPB>
__global__ void __launch_bounds__(LX * LX * EPB) k_restrict(const double* __restrict__ r, const double* __restrict__ w,
                                                     const double* __restrict__ mult, const double* __restrict__ J,
                                                     const double* __restrict__ mask, int lxc,
                                                     double* __restrict__ rc, const int* skip, int64_t E) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sJ[LX * LX];
  __shared__ double a_[EPB][N3], b_[EPB][N3];
  double* a = a_[threadIdx.z];
  double* b = b_[threadIdx.z];
  if (skip && *skip) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e0 = (int64_t)blockIdx.x * EPB + threadIdx.z;
  const bool live = e0 < E;
  const int64_t e = live ? e0 : E - 1;  // a spare slot recomputes the last element, stores nothing
  if (tid < LX * lxc) sJ[tid] = J[tid];  // J[a * lxc + b], a < LX (fine), b < lxc
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int64_t q = e * N3 + tid + NT * k;
    a[tid + NT * k] = w ? r[q] * mult[q] - mask[q] * w[q] : r[q] * mult[q];
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
      if (live) o[i + lxc * (j + lxc * kc)] = s;
    }
  }
}

// zf_e += (J (x) J (x) J) zc_e
template <int LX, int EPB>
__global__ void __launch_bounds__(LX * LX * EPB) k_prolong(const double* __restrict__ zc, const double* __restrict__ J,
                                                    int lxc, double* __restrict__ zf, const int* skip, int64_t E) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX;
  __shared__ double sJ[LX * LX];
  __shared__ double a_[EPB][N3], b_[EPB][N3];
  double* a = a_[threadIdx.z];
  double* b = b_[threadIdx.z];
  if (skip && *skip) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e0 = (int64_t)blockIdx.x * EPB + threadIdx.z;
  const bool live = e0 < E;
  const int64_t e = live ? e0 : E - 1;  // a spare slot recomputes the last element, stores nothing
  const int nc3 = lxc * lxc * lxc;
  if (tid < LX * lxc) sJ[tid] = J[tid];
  const double* ze = zc + e * (int64_t)nc3;
  for (int q = tid; q < nc3; q += NT) a[q] = ze[q];  // packed [kc][jc][ic] with stride lxc
  // the fine column this thread updates, requested now so its latency hides
  // behind the three contractions
  double* zo = zf + e * N3;
  double zcol[LX];
#pragma unroll
  for (int k = 0; k < LX; ++k) zcol[k] = zo[HIDX(i, j, k)];
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
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double s = 0.0;
    for (int c = 0; c < lxc; ++c) s += sJ[k * lxc + c] * col[c];
    if (live) zo[HIDX(i, j, k)] = zcol[k] + s;
  }
}


#undef HIDX

cudaError_t launch_fdm(const sem_mesh* m, const double* r, double* z, const double* L, const double* fdm, double h1c,
                       double h2c, const int* skip, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  if (SEM_FDM_DMMA && m->lx == 8) {
    k_fdm8_dmma<<<(unsigned)((m->E + kF8Elems - 1) / kF8Elems), 64 * kF8Elems, 0, s>>>(r, z, L, fdm, h1c, h2c, m->E,
                                                                                   skip);
    return cudaGetLastError();
  }
  SEM_LX_DISPATCH(m->lx, (k_fdm<LX, hsmg_epb(LX)><<<hsmg_grid(m->E, hsmg_epb(LX)), dim3(LX, LX, hsmg_epb(LX)), 0, s>>>(
                             r, z, L, fdm, h1c, h2c, skip, m->E)));
  return cudaGetLastError();
}

cudaError_t launch_restrict(const sem_mesh* mf, int lxc, const double* r, const double* w, const double* J,
                            double* rc, const int* skip, cudaStream_t s) {
  if (mf->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(mf);
  SEM_LX_DISPATCH(mf->lx,
                  (k_restrict<LX, hsmg_epb(LX)><<<hsmg_grid(mf->E, hsmg_epb(LX)), dim3(LX, LX, hsmg_epb(LX)), 0, s>>>(
                      r, w, mf->mult, J, mf->mask, lxc, rc, skip, mf->E)));
  return cudaGetLastError();
}

cudaError_t launch_prolong_add(const sem_mesh* mf, int lxc, const double* zc, const double* J, double* zf,
                               const int* skip, cudaStream_t s) {
  if (mf->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(mf);
  SEM_LX_DISPATCH(mf->lx, (k_prolong<LX, hsmg_epb(LX)><<<hsmg_grid(mf->E, hsmg_epb(LX)), dim3(LX, LX, hsmg_epb(LX)), 0, s>>>(
                              zc, J, lxc, zf, skip, mf->E)));
  return cudaGetLastError();
}


}  // namespace sem
