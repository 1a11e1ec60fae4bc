// Affine-element operator on the fp64 tensor cores (reading
// R5 with G_ab = C_ab w_i w_j w_k, option affine_dmma).
//
// The affine operator reads 16 B per node (u in, w out) and is bound by the
// shared-memory traffic of its six lx-point contractions on the CUDA cores
// (ncu: L1tex 94-96 %, profiles/r06_affine.md).  Here, at lx = 8, every
// contraction is a product of the 8x8 derivative matrix with an 8 x 64
// slice of the element tile, issued as mma.sync m8n8k4 f64 (DMMA): the A
// fragments (D, or D^T backwards) stay in registers, each B fragment is one
// shared load per thread per MMA (eight FMAs per shared load instead of
// one).  Two warps per element, each owning four of the eight 8-column
// tiles of every contraction; two elements per CTA.
//
//   forward   u_r = D_r u, u_s = D_s u (tiles T1, T2), u_t = D_t u, then
//             q_a = h W sum_b C_ab u_b pointwise (W = w_i w_j w_k) into
//             T1, T2 and the u tile
//   backward  w = D_r^T q_r + D_s^T q_s + D_t^T q_t (+ h2 B u)
//
// The column ownership makes most phases warp-local: a warp's DIR 0/1
// columns are the planes k < 4 (or >= 4) and its DIR 2 columns the rows
// j < 4 (or >= 4), so only four CTA barriers are needed (after the load,
// before the t-direction forward, before the backward, before its last
// direction).  Padded shared layout (rows of 12, planes of 100 doubles; cf. the
// multigrid smoother, hsmg.cu).
#include <stdint.h>

#include "ax.cuh"

namespace sem {

namespace {
constexpr int kDY = 12, kDZ = 100, kDTile = 8 * kDZ;
constexpr int kDElems = 2;  // elements per CTA (two warps each)

__device__ __forceinline__ int dslot(int i, int j, int k) { return i + kDY * j + kDZ * k; }

// slot (or natural node index) of (index l along DIR, column col)
template <int DIR, bool NAT = false>
__device__ __forceinline__ int daddr(int l, int col) {
  int i, j, k;
  if (DIR == 0) {
    i = l, j = col & 7, k = col >> 3;  // col = j + 8 k
  } else if (DIR == 1) {
    i = col & 7, j = l, k = col >> 3;  // col = i + 8 k
  } else {
    i = col & 7, j = col >> 3, k = l;  // col = i + 8 j
  }
  return NAT ? i + 8 * j + 64 * k : dslot(i, j, k);
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// the warp's four 8-column tiles of one contraction: out(m, col) =
// sum_l A(m, l) in(l, col); thread result (m = lane/4, cols 2 (lane%4) + 0/1)
template <int DIR>
__device__ __forceinline__ void dcontract(const double* in, double a0, double a1, int lane, int nt0, double (&d)[4][2]) {
  const int bl = lane & 3, bc = lane >> 2;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int colb = (nt0 + t) * 8 + bc;
    d[t][0] = d[t][1] = 0.0;
    dmma884(d[t][0], d[t][1], a0, in[daddr<DIR>(bl, colb)]);
    dmma884(d[t][0], d[t][1], a1, in[daddr<DIR>(bl + 4, colb)]);
  }
}
}  // namespace

__constant__ double c_Dd[64];  // D (lx = 8), D_il at [i * 8 + l]
__constant__ double c_Wd[8];   // GLL weights (lx = 8)

cudaError_t ax_dmma_upload_basis(const double* D, const double* w) {
  cudaError_t e = cudaMemcpyToSymbol(c_Dd, D, sizeof(double) * 64);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_Wd, w, sizeof(double) * 8);
}

template <int HM, bool CG>
__global__ void __launch_bounds__(64 * kDElems) k_ax8_aff_dmma(const AxKP P) {
  __shared__ __align__(16) double buf[kDElems][3][kDTile];
  __shared__ double sW[8];
  __shared__ double s_red[kDElems][2];
  if ((P.skip && *P.skip) || (CG && P.sc->done)) return;  // uniform over the launch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 8) sW[tid] = c_Wd[tid];
  const int le = warp >> 1, half = warp & 1, nt0 = half * 4;
  const int64_t q = (int64_t)blockIdx.x * kDElems + le;
  const int64_t count = P.npos;
  const bool live = q < count;
  const int64_t e = live ? (P.elist ? (int64_t)P.elist[P.elem0 + q] : P.elem0 + q) : 0;
  double* U = buf[le][0];
  double* T1 = buf[le][1];
  double* T2 = buf[le][2];
  const int et = tid & 63;
  if (live) {
    if constexpr (CG) {  // p <- dinv r + beta p (and the deferred x += alpha p_old)
      const double beta = P.sc->beta, xa = P.sc->xalpha;
      const size_t eo = (size_t)e * 512;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const size_t g = eo + et + 64 * p;
        const double pv = P.p[g];
        if (P.x) P.x[g] += xa * pv;
        const double pn = __ldg(P.dinv + g) * __ldg(P.r + g) + beta * pv;
        P.p[g] = pn;
        U[dslot(et & 7, et >> 3, p)] = pn;
      }
    } else {
      const double* ue = P.u + e * 512;
#pragma unroll
      for (int p = 0; p < 8; ++p) U[dslot(et & 7, et >> 3, p)] = __ldg(ue + et + 64 * p);
    }
  }
  // A fragments: forward D (A(m, l) = D_ml), backward D^T (A(m, l) = D_lm)
  const int ar = lane >> 2, ac = lane & 3;
  const double f0 = c_Dd[ar * 8 + ac], f1 = c_Dd[ar * 8 + ac + 4];
  const double b0 = c_Dd[ac * 8 + ar], b1 = c_Dd[(ac + 4) * 8 + ar];
  double C[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) C[c] = live ? __ldg(P.gaff + e * 6 + c) : 0.0;
  __syncthreads();
  double d[4][2];
  const int bl = lane & 3, m = lane >> 2;
  // forward r and s: the warp's planes k in [4 half, 4 half + 4)
  dcontract<0>(U, f0, f1, lane, nt0, d);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int col0 = (nt0 + t) * 8 + 2 * bl;
    T1[daddr<0>(m, col0)] = d[t][0];
    T1[daddr<0>(m, col0 + 1)] = d[t][1];
  }
  dcontract<1>(U, f0, f1, lane, nt0, d);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int col0 = (nt0 + t) * 8 + 2 * bl;
    T2[daddr<1>(m, col0)] = d[t][0];
    T2[daddr<1>(m, col0 + 1)] = d[t][1];
  }
  __syncthreads();
  // forward t (the warp's rows j in [4 half, 4 half + 4)), then q pointwise
  dcontract<2>(U, f0, f1, lane, nt0, d);
  __syncwarp();  // the warp's reads of U (its own columns) are done; each lane
                 // then reads and writes only its own nodes
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = (nt0 + t) * 8 + 2 * bl + h;
      const int i = col & 7, j = col >> 3, k = m;
      const int sl = dslot(i, j, k);
      const double ur = T1[sl], us = T2[sl], ut = d[t][h];
      const double W = sW[i] * sW[j] * sW[k];
      T1[sl] = W * (C[0] * ur + C[3] * us + C[4] * ut);
      T2[sl] = W * (C[3] * ur + C[1] * us + C[5] * ut);
      U[sl] = W * (C[4] * ur + C[5] * us + C[2] * ut);
    }
  __syncthreads();
  // backward r then s, accumulated in place in T1 (warp-local node sets)
  dcontract<0>(T1, b0, b1, lane, nt0, d);
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int col0 = (nt0 + t) * 8 + 2 * bl;
    T1[daddr<0>(m, col0)] = d[t][0];
    T1[daddr<0>(m, col0 + 1)] = d[t][1];
  }
  dcontract<1>(T2, b0, b1, lane, nt0, d);
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int col0 = (nt0 + t) * 8 + 2 * bl;
    T1[daddr<1>(m, col0)] += d[t][0];
    T1[daddr<1>(m, col0 + 1)] += d[t][1];
  }
  __syncthreads();
  // backward t, the sum, the mass term, the store (two consecutive i: 16 B
  // in the natural layout); CG: pAp = sum p (A_e p) over the element (R10)
  dcontract<2>(U, b0, b1, lane, nt0, d);
  double pap = 0.0;
  if (live) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int col0 = (nt0 + t) * 8 + 2 * bl;
      const int i0 = col0 & 7, j = col0 >> 3, k = m;
      double o[2];
      o[0] = T1[dslot(i0, j, k)] + d[t][0];
      o[1] = T1[dslot(i0 + 1, j, k)] + d[t][1];
      const int n0 = i0 + 8 * j + 64 * k;
      const int64_t g = e * 512 + n0;
      double uu[2] = {0.0, 0.0};
      if (HM == 1 || CG) {  // u (CG: the new p, written by this CTA above)
        if (CG) {
          uu[0] = P.p[g];
          uu[1] = P.p[g + 1];
        } else {
          const double2 v = __ldg(reinterpret_cast<const double2*>(P.u + g));
          uu[0] = v.x;
          uu[1] = v.y;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (HM == 0) o[h] *= P.h1c;
        else o[h] = P.h1c * o[h] + P.h2c * __ldg(P.B + g + h) * uu[h];
        if (CG) pap += uu[h] * o[h];
      }
      if (CG && P.xl) {  // the CG operator output in the x-planes-last layout
        P.w[e * 512 + xlast_pos<8>(n0)] = o[0];
        P.w[e * 512 + xlast_pos<8>(n0 + 1)] = o[1];
      } else {
        *reinterpret_cast<double2*>(P.w + g) = make_double2(o[0], o[1]);
      }
    }
  }
  if constexpr (CG) {  // the element's pAp partial (its two warps), fixed order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pap += __shfl_down_sync(0xffffffffu, pap, o);
    if (lane == 0) s_red[le][half] = pap;
    __syncthreads();
    if (live && half == 0 && lane == 0) P.part[P.elem0 + q] = s_red[le][0] + s_red[le][1];
  }
}

cudaError_t launch_ax8_aff_dmma(const sem_mesh* m, const AxKP& P0, int HM, bool cg, int64_t count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  AxKP P = P0;
  P.npos = count;  // positions [elem0, elem0 + count) of this launch
  const unsigned grid = (unsigned)((count + kDElems - 1) / kDElems);
  if (cg) {
    if (HM == 0) k_ax8_aff_dmma<0, true><<<grid, 64 * kDElems, 0, s>>>(P);
    else k_ax8_aff_dmma<1, true><<<grid, 64 * kDElems, 0, s>>>(P);
  } else {
    if (HM == 0) k_ax8_aff_dmma<0, false><<<grid, 64 * kDElems, 0, s>>>(P);
    else k_ax8_aff_dmma<1, false><<<grid, 64 * kDElems, 0, s>>>(P);
  }
  return cudaGetLastError();
}

}  // namespace sem
