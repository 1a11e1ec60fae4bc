// Restarted GMRES(m) with right (Jacobi) preconditioning for the pressure
// system -- "we use restarted GMRES for the pressure solves";
// SURVEY.md 8(f) row f2, reading R14.  Same algorithm as the
// oracle's or_gmres (Saad 2003, Alg. 9.5; Givens rotations, section 6.5.3)
// except that the Arnoldi step orthogonalises by classical Gram-Schmidt with
// one re-orthogonalisation (CGS2: equal to modified Gram-Schmidt in exact
// arithmetic, and two fused vector passes instead of j+1 dependent ones):
//   w  = mask dssum(A_e z_j),  z_j = dinv v_j           (operator, fused gs)
//   h  = V^T w                                          k_gm_stream<0>
//   w1 = w - V h ; h2 = V^T w1 ; nn = <w1, w1>          k_gm_stream<1>
//   H(:, j) = h + h2 ; sigma = sqrt(nn - |h2|^2) ; Givens ; stopping test
//                                                       k_gm_givens
//   v_{j+1} = (w1 - V h2) / sigma ; z_{j+1} = dinv v_{j+1}   k_gm_stream<2>
// and per cycle: y = H^-1 g (k_gm_solve), x += dinv (V y) (k_gm_xupd), the
// true residual r = b - mask dssum(A_e x) and v_0 = r / |r| (k_gm_resid,
// k_gm_start).  Inner products are mult-weighted (reading R10); every
// reduction is deterministic (per-block partials, the last block sums them
// in block order).  All scalars stay on the device; the host only reads
// them once per cycle.
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "device_common.cuh"
#include "gmres.h"

namespace sem {

constexpr int kGmThreads = 256;

static unsigned gm_blocks(const sem_mesh* m) {
  return (unsigned)std::min<int64_t>((int64_t)m->nsm * 4, kGmMaxBlocks);
}

// The three Arnoldi vector passes as one TMA-staged streaming kernel: each
// CTA walks tiles of kGmTile consecutive nodes; thread 0 issues one bulk copy
// (cp.async.bulk, TMA engine) per operand chunk of a tile into a two-stage
// shared-memory ring (an mbarrier per stage), so two tiles' worth of the j+1
// basis chunks (up to 31 x 2 KB) stream in while the threads work on the
// previous tile from shared memory -- the loads need no registers, and the
// bytes in flight per SM do not depend on the number of basis vectors.  The
// ragged last tile (n not a multiple of kGmTile) reads global memory
// directly.  Modes:
//   0 dots    out[k] = <w, V_k>                         (aux = mult)
//   1 update  w -= sum c_k V_k ; out[k] = <w, V_k>, out[NV] = <w, w>  (aux = mult)
//   2 next    vout = (w - sum c_k V_k) / sigma ; z = aux v  (aux = dinv; z may be NULL)
// Tile: 256 nodes (2 KB chunks), 128 for NV = 32 so that three CTAs of
// 2 x 34 chunks fit one SM's shared memory (one CTA of 256 measured 3.2
// against 6.8 TB/s for NV = 16 at three CTAs per SM).
template <int MODE, int NV, int kGmTile = (NV > 16 ? 128 : 256)>
__global__ void __launch_bounds__(kGmTile) k_gm_stream(double* __restrict__ w, const double* __restrict__ V, int64_t ld,
                                                       int nvec, const double* __restrict__ c,
                                                       const double* __restrict__ aux, int64_t n, double* part,
                                                       unsigned* ticket, double* out, double* __restrict__ vout,
                                                       double* __restrict__ z, const GmScalars* gs) {
  constexpr int NACC = MODE == 1 ? NV + 1 : NV;
  extern __shared__ __align__(128) double smem[];  // [2][NV + 2][kGmTile]
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double s_c[NV];
  __shared__ double s_red[MODE == 2 ? 1 : 32 * NACC];
  __shared__ int s_flag;
  if (gs->cycle_stop) return;  // uniform over the launch
  if (MODE == 2 && !(gs->sigma > 0.0)) return;
  const int tid = threadIdx.x;
  const int64_t ntiles = (n + kGmTile - 1) / kGmTile, nfull = n / kGmTile;
  const int64_t stride = gridDim.x;
  if (MODE != 0 && tid < NV) s_c[tid] = tid < nvec ? c[tid] : 0.0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  constexpr uint32_t kChunk = kGmTile * sizeof(double);
  auto issue = [&](int64_t t, int st) {  // thread 0: every operand chunk of tile t into stage st
    double* dst = smem + (size_t)st * (NV + 2) * kGmTile;
    mbar_expect_tx(&bar[st], kChunk * (uint32_t)(nvec + 2));
    for (int k = 0; k < nvec; ++k) bulk_g2s_plain(dst + k * kGmTile, V + k * ld + t * kGmTile, kChunk, &bar[st]);
    bulk_g2s_plain(dst + NV * kGmTile, w + t * kGmTile, kChunk, &bar[st]);
    bulk_g2s_plain(dst + (NV + 1) * kGmTile, aux + t * kGmTile, kChunk, &bar[st]);
  };
  if (tid == 0) {
    if (blockIdx.x < nfull) issue(blockIdx.x, 0);
    if (blockIdx.x + stride < nfull) issue(blockIdx.x + stride, 1);
  }
  double acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
  const double is = MODE == 2 ? 1.0 / gs->sigma : 0.0;
  uint32_t ph0 = 0, ph1 = 0;
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += stride, ++it) {
    const int st = it & 1;
    const bool full = t < nfull;
    const int64_t q = t * kGmTile + tid;
    const double* sv = smem + (size_t)st * (NV + 2) * kGmTile;
    if (full) {
      mbar_wait(&bar[st], st ? ph1 : ph0);
      if (st) ph1 ^= 1; else ph0 ^= 1;
    }
    if (full || q < n) {
      auto Vk = [&](int k) { return full ? sv[k * kGmTile + tid] : V[k * ld + q]; };
      const double wq = full ? sv[NV * kGmTile + tid] : w[q];
      const double aq = full ? sv[(NV + 1) * kGmTile + tid] : aux[q];
      if (MODE == 0) {
        const double mw = aq * wq;
#pragma unroll
        for (int k = 0; k < NV; ++k)
          if (k < nvec) acc[k] += mw * Vk(k);
      } else {
        double w1 = wq;
#pragma unroll
        for (int k = 0; k < NV; ++k)
          if (k < nvec) w1 -= s_c[k] * Vk(k);
        if (MODE == 1) {
          w[q] = w1;
          const double mw = aq * w1;
#pragma unroll
          for (int k = 0; k < NV; ++k)
            if (k < nvec) acc[k] += mw * Vk(k);
          acc[NV] += mw * w1;
        } else {
          const double v = w1 * is;
          vout[q] = v;
          if (z) z[q] = aq * v;
        }
      }
    }
    __syncthreads();  // stage st fully read
    if (tid == 0 && t + 2 * stride < nfull) issue(t + 2 * stride, st);
  }
  if (MODE != 2) grid_sum_last_block<NACC>(acc, part, ticket, out, s_red, &s_flag);
}

template <int MODE, int NV>
static cudaError_t gm_stream_launch(sem_mesh* m, GmState* G, int nvec, double* w, const double* c,
                                    const double* aux, double* out, double* vout, double* z, cudaStream_t s) {
  constexpr int kGmTile = NV > 16 ? 128 : 256;
  const size_t smem = (size_t)2 * (NV + 2) * kGmTile * sizeof(double);
  static std::atomic<bool> attr_set[64];
  const int dev = m->device & 63;
  if (!attr_set[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(k_gm_stream<MODE, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true);
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gm_stream<MODE, NV>, kGmTile, smem);
  const int64_t ntiles = (m->nloc + kGmTile - 1) / kGmTile;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>({(int64_t)m->nsm * std::max(per_sm, 1), ntiles,
                                                              kGmMaxBlocks}));
  k_gm_stream<MODE, NV><<<(unsigned)grid, kGmTile, smem, s>>>(w, G->V, G->ld, nvec, c, aux, m->nloc, G->part,
                                                             G->ticket, out, vout, z, G->gs);
  return cudaGetLastError();
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
  GM_NV_DISPATCH(nvec, return (gm_stream_launch<0, NV>(m, G, nvec, m->w, nullptr, m->mult, G->gs->h, nullptr, nullptr,
                                                      s)));
}

cudaError_t gm_launch_update(sem_mesh* m, GmState* G, int nvec, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  // the reduction writes [h2 (NV), nn]: copy nn into place after (k_gm_givens reads gs->nn)
  GM_NV_DISPATCH(nvec, return (gm_stream_launch<1, NV>(m, G, nvec, m->w, G->gs->h, m->mult, G->red, nullptr, nullptr,
                                                      s)));
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
  GM_NV_DISPATCH(nvec, return (gm_stream_launch<2, NV>(m, G, nvec, m->w, G->gs->h2, m->dinv, nullptr,
                                                      G->V + (int64_t)(j + 1) * G->ld, flex ? nullptr : G->z, s)));
}

cudaError_t gm_launch_cycle_end(sem_mesh* m, GmState* G, double* x, bool flex, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_gm_solve<<<1, 1, 0, s>>>(G->gs);
  for (int k0 = 0; k0 < G->restart; k0 += 16) {
    SEM_COUNT_LAUNCH(m);
    k_gm_xupd<16><<<gm_blocks(m), kGmThreads, 0, s>>>(x, flex ? G->Z : G->V, flex ? m->nloc : G->ld, k0,
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
