// sm_100a kernels of the SEM hot path (arXiv 2405.05640).
//
//   k_geom      geometric factors G_ab, B (reading R4), once per mesh
//   k_mult_mask multiplicity / mask per local node (R7, R8)
//   k_gs_nodal  the gather-scatter pass over precomputed copy offsets (R7, R8),
//               run after every operator launch (natural layout, or the CG's
//               x-planes-last layout of the operator output; the in-launch
//               variants were measured slower)
//   k_if_*      interface exchange of the gather-scatter across ranks
//   k_diag      exact local Jacobi diagonal (R9)
//   CG vector kernels and deterministic two-stage reductions (R10)
//
// Data layout: fields [E][lx^3] fp64; G [E][6][n3p]
// (n3p = n3 rounded up to even so every element's 6 factors are one
// 16-byte-aligned contiguous block that a single cp.async.bulk (TMA) moves
// into shared memory).
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>

#include "device_common.cuh"
#include "p2p.cuh"

namespace sem {

__constant__ double c_D[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];  // c_D[lx][i*lx+l] = D_il
__constant__ double c_w[kMaxN + 2][kMaxN + 1];

cudaError_t upload_basis_ax(int N, const double* D, const double* w);
cudaError_t upload_basis_p(int N, const double* D);
cudaError_t upload_basis_pnpn(int N, const double* D, const double* w);

cudaError_t upload_basis(int N, const double* D, const double* w) {
  const int lx = N + 1;
  cudaError_t e = upload_basis_ax(N, D, w);
  if (e != cudaSuccess) return e;
  e = upload_basis_p(N, D);
  if (e != cudaSuccess) return e;
  e = upload_basis_pnpn(N, D, w);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(c_D, D, sizeof(double) * lx * lx,
                                     sizeof(double) * lx * (kMaxN + 1) * (kMaxN + 1));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_w, w, sizeof(double) * lx, sizeof(double) * lx * (kMaxN + 1));
}

// ---------------------------------------------------------------------------
// Geometry (R4): X = dx/dr by D contractions, J = det X, R = X^-1,
// G_ab = W J sum_m R_am R_bm, B = W J, W = w_i w_j w_k.
// ---------------------------------------------------------------------------
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_geom(const double* __restrict__ coords, int64_t E,
                                                   double* __restrict__ G, int64_t gstride,
                                                   double* __restrict__ B,
                                                   unsigned long long* bad) {
  constexpr int N3 = LX * LX * LX, N3P = (N3 + 1) & ~1, NT = LX * LX;
  __shared__ double sx[3][N3];
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  for (int q = tid; q < N3; q += NT)
#pragma unroll
    for (int c = 0; c < 3; ++c) sx[c][q] = coords[(size_t)c * E * N3 + (size_t)e * N3 + q];
  __syncthreads();
#pragma unroll 1
  for (int k = 0; k < LX; ++k) {
    double X[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        dr += c_D[LX][i * LX + l] * sx[c][l + LX * (j + LX * k)];
        ds += c_D[LX][j * LX + l] * sx[c][i + LX * (l + LX * k)];
        dt += c_D[LX][k * LX + l] * sx[c][i + LX * (j + LX * l)];
      }
      X[c][0] = dr;
      X[c][1] = ds;
      X[c][2] = dt;
    }
    const double C00 = X[1][1] * X[2][2] - X[1][2] * X[2][1];
    const double C01 = X[1][2] * X[2][0] - X[1][0] * X[2][2];
    const double C02 = X[1][0] * X[2][1] - X[1][1] * X[2][0];
    const double J = X[0][0] * C00 + X[0][1] * C01 + X[0][2] * C02;
    if (!(J > 0.0)) atomicMin(bad, (unsigned long long)e);
    // R[a][m] = adj(X)[a][m] / J
    const double iJ = 1.0 / J;
    double R[3][3];
    R[0][0] = C00 * iJ;
    R[1][0] = C01 * iJ;
    R[2][0] = C02 * iJ;
    R[0][1] = (X[0][2] * X[2][1] - X[0][1] * X[2][2]) * iJ;
    R[1][1] = (X[0][0] * X[2][2] - X[0][2] * X[2][0]) * iJ;
    R[2][1] = (X[0][1] * X[2][0] - X[0][0] * X[2][1]) * iJ;
    R[0][2] = (X[0][1] * X[1][2] - X[0][2] * X[1][1]) * iJ;
    R[1][2] = (X[0][2] * X[1][0] - X[0][0] * X[1][2]) * iJ;
    R[2][2] = (X[0][0] * X[1][1] - X[0][1] * X[1][0]) * iJ;
    const double WJ = c_w[LX][i] * c_w[LX][j] * c_w[LX][k] * J;
    const int p = tid + NT * k;
    double* Ge = G + (size_t)e * gstride;
    const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int a = ab[c][0], b = ab[c][1];
      Ge[c * N3P + p] = WJ * (R[a][0] * R[b][0] + R[a][1] * R[b][1] + R[a][2] * R[b][2]);
    }
    B[(size_t)e * N3 + p] = WJ;
  }
}

// mult (1/m) and mask (0/1) per local node
template <int LX>
__global__ void k_mult_mask(double* __restrict__ mult, double* __restrict__ mask, uint8_t* __restrict__ m8,
                            GsPlan plan, const int32_t* __restrict__ gcount, int64_t nitems) {
  constexpr int N3 = LX * LX * LX, M = LX - 2, MD = M > 0 ? M : 1;
  const int64_t fItems = plan.nF * M * M, eItems = plan.nEd * M;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nitems;
       it += (int64_t)gridDim.x * blockDim.x) {
    int64_t ent;
    int n;
    if (it < fItems) {
      ent = it / (MD * MD);
      n = (int)(it % (MD * MD));
    } else if (it < fItems + eItems) {
      ent = plan.nF + (it - fItems) / MD;
      n = (int)((it - fItems) % MD);
    } else {
      ent = plan.nF + plan.nEd + (it - fItems - eItems);
      n = 0;
    }
    const int c0 = plan.ent_ptr[ent], c1 = plan.ent_ptr[ent + 1];
    const int mcount = gcount ? gcount[ent] : (c1 - c0);
    const double mv = 1.0 / (double)mcount;
    const double kv = (plan.ent_flags[ent] & kEntMasked) ? 0.0 : 1.0;
    for (int c = c0; c < c1; ++c) {
      const int64_t cp = plan.ent_copy[c];
      const size_t o = (size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n);
      mult[o] = mv;
      mask[o] = kv;
      if (m8) m8[o] = (uint8_t)(mcount < 255 ? mcount : 0);
    }
  }
}

__global__ void k_fill(double* x, double v, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    x[q] = v;
}

static int64_t gs_items(const sem_mesh* m) {
  const int64_t M = m->lx - 2;
  return m->topo.nF * M * M + m->topo.nEd * M + m->topo.nV;
}

// grid-stride launches: at most 16 blocks per SM
static unsigned grid_for(const sem_mesh* m, int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > (int64_t)m->nsm * 16) b = (int64_t)m->nsm * 16;
  if (b < 1) b = 1;
  return (unsigned)b;
}

cudaError_t launch_geom_bad(const sem_mesh* m, unsigned long long* bad, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_geom<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(
                             m->coords, m->E, m->G, (int64_t)6 * m->n3p, m->B, bad)));
  return cudaGetLastError();
}

cudaError_t launch_mult_mask(const sem_mesh* m, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  if (m->m8) cudaMemsetAsync(m->m8, 1, (size_t)m->nloc, s);  // interior nodes: multiplicity 1
  k_fill<<<grid_for(m, m->nloc, 256), 256, 0, s>>>(m->mult, 1.0, m->nloc);
  SEM_COUNT_LAUNCH(m);
  k_fill<<<grid_for(m, m->nloc, 256), 256, 0, s>>>(m->mask, 1.0, m->nloc);
  const int64_t n = gs_items(m);
  if (n == 0) return cudaGetLastError();
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_mult_mask<LX><<<grid_for(m, n, 256), 256, 0, s>>>(m->mult, m->mask, m->m8, m->plan(), m->d_ent_gcount, n)));
  return cudaGetLastError();
}

// Nodal gather-scatter over one launch's classes: item -> (class, group);
// the group's m offsets are coalesced loads (pairs: one 8-byte load), its
// copies are summed in list
// (ascending element) order, and the sum (0 if masked) is stored to each.
// Items [0, n2) are the m <= 2 classes (faces, masked single copies): each
// thread takes kGsU of them, all loads in flight before the first use (the
// pass is latency bound); the rest (edges, vertices) one item per thread.
P2PArgs p2p_args(const sem_mesh* m);  // p2p.cu (peers == nullptr: one rank or NCCL)
#ifndef SEM_GS_U
#define SEM_GS_U 4
#endif
// programmatic dependent launch (option pdl): the dependents are released at
// the end of a kernel's main loop, so they reserve no SM resources while it runs
#ifndef SEM_PDL_LATE
#define SEM_PDL_LATE 1
#endif
#ifndef SEM_GS_MINB
#define SEM_GS_MINB 5
#endif
#ifndef SEM_GS_REV
#define SEM_GS_REV 1
#endif
constexpr int kGsU = SEM_GS_U;  // face groups per thread, all loads in flight (build flag for A/B)
// the pAp-fusing gs launch reduces through the scratch before the per-position
// partials (pap_part_offset() = kMaxVecBlocks * 4 entries): at most that many
// blocks (32 per SM measured best at 148 SMs; 2 and 8 per SM slower)
static int64_t gs_pap_blocks(const sem_mesh* m) { return std::min<int64_t>((int64_t)m->nsm * 32, kMaxVecBlocks * 4); }
__device__ __forceinline__ int gs_class(const GsLaunch& A, int it) {
  int t = 0;
  while (t + 1 < A.ncls && it >= A.c[t + 1].item0) ++t;
  return t;
}
// fused pAp reduction (one rank, CG): the operator's per-element partials
struct PapFuse {
  const double* in;  // nullptr: none
  int64_t n;
  double* part;
  unsigned* ticket;
  CGScalars* sc;
  P2PArgs p2p;       // several ranks: the sum is allreduced over NVLink in place
};
__global__ void __launch_bounds__(256, SEM_GS_MINB) k_gs_nodal(double* __restrict__ u, const uint32_t* __restrict__ idx,
                                                  const GsLaunch A, const PapFuse F) {
  if (A.pdl) {
    griddep_wait();
    if (!SEM_PDL_LATE) griddep_launch_dependents();
  }
  const int S = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  // face items: each block takes kGsU * blockDim consecutive items (groups
  // are sorted by their first copy's offset, so a block sweeps a contiguous
  // stretch of w); SEM_GS_REV: from the top of w down, where the operator
  // that just ran left the most recently written lines in L2
  const int BK = kGsU * blockDim.x;
  for (int b0 = blockIdx.x * BK; b0 < A.n2; b0 += gridDim.x * BK) {
    uint32_t o0[kGsU], o1[kGsU];
    bool ok[kGsU], msk[kGsU];
#pragma unroll
    for (int k = 0; k < kGsU; ++k) {
      int it = b0 + k * (int)blockDim.x + (int)threadIdx.x;
      ok[k] = it < A.n2;
      if (SEM_GS_REV) it = A.n2 - 1 - it;
      msk[k] = true;
      o0[k] = o1[k] = 0;
      if (ok[k]) {
        const int t = gs_class(A, it);
        const int g = it - A.c[t].item0;
        msk[k] = A.c[t].masked;
        // one load per item, so the loads of all kGsU items issue back to back
        if (A.c[t].m == 2) {
          const uint2 o = __ldg(reinterpret_cast<const uint2*>(idx + A.c[t].base) + g);
          o0[k] = o.x;
          o1[k] = o.y;
        } else {  // a masked single copy
          o0[k] = o1[k] = __ldg(idx + A.c[t].base + g);
        }
      }
    }
    double v0[kGsU], v1[kGsU];
#pragma unroll
    for (int k = 0; k < kGsU; ++k) {
      v0[k] = v1[k] = 0.0;
      if (ok[k] && !msk[k]) {
        v0[k] = u[o0[k]];
        v1[k] = u[o1[k]];
      }
    }
#pragma unroll
    for (int k = 0; k < kGsU; ++k)
      if (ok[k]) {
        double s = msk[k] ? 0.0 : (0.0 + v0[k]) + v1[k];
        if (A.scale) s *= 0.5;  // 1/m of a two-copy group (masked singles are 0)
        u[o0[k]] = s;
        u[o1[k]] = s;
      }
  }
  for (int it1 = A.n2 + tid; it1 < A.nitems; it1 += S) {
    const int it = SEM_GS_REV ? A.nitems - 1 - (it1 - A.n2) : it1;
    const int t = gs_class(A, it);
    const int count = A.c[t].count, mlt = A.c[t].m, masked = A.c[t].masked;
    const uint32_t* __restrict__ ix = idx + A.c[t].base + (it - A.c[t].item0);
    if (mlt <= 8) {
      uint32_t o[8];
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < mlt) o[c] = __ldg(ix + (int64_t)c * count);
      double s = 0.0;
      if (!masked) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < mlt) v[c] = u[o[c]];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < mlt) s += v[c];
        if (A.scale) s *= 1.0 / (double)mlt;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < mlt) u[o[c]] = s;
    } else {
      double s = 0.0;
      if (!masked) {
        for (int c = 0; c < mlt; ++c) s += u[__ldg(ix + (int64_t)c * count)];
        if (A.scale) s *= 1.0 / (double)mlt;
      }
      for (int c = 0; c < mlt; ++c) u[__ldg(ix + (int64_t)c * count)] = s;
    }
  }
  if (A.pdl && SEM_PDL_LATE) griddep_launch_dependents();  // the next kernel may stage its inputs
  // pAp = sum of the operator's partials (what k_reduce_parts does), and
  // the pending deferred-x alpha is consumed
  // Only the first nred blocks (one partial per thread) take part, so the
  // other blocks retire without a block barrier (measured: 20 % of the
  // pass's stall samples were that barrier when every block joined)
  const int64_t nneed = (F.n + blockDim.x - 1) / blockDim.x;
  const unsigned nred = nneed < (int64_t)gridDim.x ? (unsigned)nneed : gridDim.x;
  if (F.in && !F.sc->done && blockIdx.x < max(nred, 1u)) {
    __shared__ double s_red[32];
    __shared__ int s_flag;
    double v[1] = {0.0};
    const int64_t Sr = (int64_t)max(nred, 1u) * blockDim.x;
    for (int64_t q = tid; q < F.n; q += Sr) v[0] += F.in[q];
    grid_sum_last_block<1>(v, F.part, F.ticket, &F.sc->red[0], s_red, &s_flag, max(nred, 1u));
    if (F.p2p.peers && s_flag) {
      __syncthreads();
      if (threadIdx.x < 32) p2p_allreduce_warp(&F.sc->red[0], 1, F.p2p, threadIdx.x);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) F.sc->xalpha = 0.0;
  }
}

// the active classes of a list for mode (1 sum, 2 mask, 3 both): a class acts
// if it sums (m > 1) or masks; m <= 2 classes first; launched in batches of
// kGsMaxCls classes
cudaError_t launch_gs_nodal(const sem_mesh* m, double* w, const uint32_t* idx, const std::vector<GsClass>& cls,
                            int mode, cudaStream_t s, bool* pap_fused, bool pdl) {
  GsLaunch A;
  A.ncls = A.nitems = A.n2 = 0;
  A.pdl = 0;
  A.scale = (mode & 4) ? 1 : 0;
  bool first = true;
  auto flush = [&](bool last) -> cudaError_t {
    if (A.nitems == 0) return cudaSuccess;
    SEM_COUNT_LAUNCH(m);
    int64_t blocks = std::max(((int64_t)A.n2 + 256 * kGsU - 1) / (256 * kGsU),
                              ((int64_t)(A.nitems - A.n2) + 255) / 256);
    PapFuse F{nullptr, 0, nullptr, nullptr, nullptr, P2PArgs{nullptr, nullptr, nullptr, nullptr, 0, 1}};
    if (last && pap_fused) {  // the reduction scratch before the partials
      F = PapFuse{m->part + pap_part_offset(), m->pap_nparts, m->part, m->ticket, m->sc, p2p_args(m)};
      blocks = std::min<int64_t>(blocks, gs_pap_blocks(m));
      *pap_fused = true;
    }
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)m->nsm * 64));
    A.pdl = (pdl && first) ? 1 : 0;  // the first launch follows the operator
    first = false;
    cudaError_t e = launch_maybe_pdl(A.pdl != 0, k_gs_nodal, dim3((unsigned)blocks), dim3(256), 0, s, w, idx, A, F);
    A.ncls = A.nitems = A.n2 = 0;
    return e;
  };
  for (int pass = 0; pass < 2; ++pass) {
    for (const GsClass& g : cls) {
      if ((g.m <= 2) != (pass == 0)) continue;
      const bool add = (mode & 1) && g.m > 1, msk = (mode & 2) && g.masked;
      if (!add && !msk) continue;
      if (A.ncls == kGsMaxCls || (int64_t)A.nitems + g.count >= ((int64_t)1 << 31)) {
        cudaError_t e = flush(false);
        if (e != cudaSuccess) return e;
      }
      GsLaunchCls& L = A.c[A.ncls++];
      L.base = g.base;
      L.count = (int32_t)g.count;
      L.item0 = A.nitems;
      L.m = g.m;
      L.masked = msk ? 1 : 0;
      A.nitems += (int32_t)g.count;
      if (pass == 0) A.n2 = A.nitems;
    }
  }
  return flush(true);
}

// ---------------------------------------------------------------------------
// Interface exchange kernels (comm.cpp): own partial sums of the interface
// entities' local copies (ascending element order), pack per peer, and the
// rank-ordered total written back to every local copy (0 where masked).
// ---------------------------------------------------------------------------
template <int LX>
__global__ void k_if_partial(const double* __restrict__ u, GsPlan plan, const int32_t* __restrict__ if_ent,
                             const int32_t* __restrict__ node_ent, const int64_t* __restrict__ noff, int64_t nn,
                             double* __restrict__ U, int xl) {
  constexpr int N3 = LX * LX * LX;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nn; it += (int64_t)gridDim.x * blockDim.x) {
    const int q = node_ent[it];
    const int n = (int)(it - noff[q]);
    const int ent = if_ent[q];
    double sum = 0.0;
    for (int c = plan.ent_ptr[ent]; c < plan.ent_ptr[ent + 1]; ++c) {
      const int64_t cp = plan.ent_copy[c];
      const int lo = node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n);
      sum += u[(size_t)(cp >> 8) * N3 + (xl ? xlast_pos<LX>(lo) : lo)];
    }
    U[it] = sum;
  }
}

__global__ void k_if_pack(const double* __restrict__ U, const int32_t* __restrict__ idx, int64_t n,
                          double* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = U[idx[q]];
}

template <int LX>
__global__ void k_if_unpack(double* __restrict__ u, GsPlan plan, const int32_t* __restrict__ if_ent,
                            const int32_t* __restrict__ node_ent, const int64_t* __restrict__ noff,
                            const int32_t* __restrict__ src_ptr, const int64_t* __restrict__ src, int64_t nn,
                            const double* __restrict__ U, int mode, const unsigned long long* xseq,
                            int64_t nrecv, int xl, const int32_t* __restrict__ gcount) {
  constexpr int N3 = LX * LX * LX;
  // P2P exchange: the peers' partials sit in the receive region of this
  // exchange's parity (the wait kernel advanced *xseq)
  const int64_t shift = (xseq && ((*xseq) & 1)) ? nrecv : 0;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nn; it += (int64_t)gridDim.x * blockDim.x) {
    const int q = node_ent[it];
    const int n = (int)(it - noff[q]);
    const int ent = if_ent[q];
    const bool masked = (mode & 2) && (plan.ent_flags[ent] & kEntMasked);
    if (!(mode & 1) && !masked) continue;
    double sum = 0.0;
    if (mode & 1)
      for (int k = src_ptr[q]; k < src_ptr[q + 1]; ++k) {
        const int64_t o = src[k];
        sum += U[(o >= nn ? o + shift : o) + n];
      }
    if (masked) sum = 0.0;
    else if ((mode & 4) && gcount) sum *= 1.0 / (double)gcount[ent];  // as z *= mult would
    for (int c = plan.ent_ptr[ent]; c < plan.ent_ptr[ent + 1]; ++c) {
      const int64_t cp = plan.ent_copy[c];
      const int lo = node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n);
      u[(size_t)(cp >> 8) * N3 + (xl ? xlast_pos<LX>(lo) : lo)] = sum;
    }
  }
}

cudaError_t launch_if_partial(const sem_mesh* m, const double* u, cudaStream_t s) {
  if (m->n_if_nodes == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_if_partial<LX><<<grid_for(m, m->n_if_nodes, 256), 256, 0, s>>>(
                             u, m->plan(), m->d_if_ent, m->d_if_node_ent, m->d_if_noff, m->n_if_nodes, m->d_U,
                             m->xl_active ? 1 : 0)));
  return cudaGetLastError();
}

cudaError_t launch_if_pack(const sem_mesh* m, cudaStream_t s) {
  const int64_t n = m->peer_off.empty() ? 0 : m->peer_off.back();
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  k_if_pack<<<grid_for(m, n, 256), 256, 0, s>>>(m->d_U, m->d_send_idx, n, m->d_sendbuf);
  return cudaGetLastError();
}

cudaError_t launch_if_unpack(const sem_mesh* m, double* u, int mode, cudaStream_t s) {
  if (m->n_if_nodes == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_if_unpack<LX><<<grid_for(m, m->n_if_nodes, 256), 256, 0, s>>>(
                             u, m->plan(), m->d_if_ent, m->d_if_node_ent, m->d_if_noff, m->d_if_src_ptr,
                             m->d_if_src, m->n_if_nodes, m->d_U, mode, m->xp2p ? m->d_x_seq : nullptr,
                             m->peer_off.empty() ? 0 : m->peer_off.back(), m->xl_active ? 1 : 0, m->d_ent_gcount)));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Jacobi diagonal (R9): d = h1 [sum_l D_li^2 G11(l,j,k) + ... + 2 D_ii D_jj G12
//   + 2 D_ii D_kk G13 + 2 D_jj D_kk G23] + h2 B  (h1 at each term's node)
// ---------------------------------------------------------------------------
template <int LX>
__global__ void k_diag(const double* __restrict__ G, int64_t gstride, const double* __restrict__ B,
                       const double* __restrict__ h1, const double* __restrict__ h2, double h1c,
                       double h2c, double* __restrict__ d) {
  constexpr int N3 = LX * LX * LX, N3P = (N3 + 1) & ~1, NT = LX * LX;
  __shared__ double sg[3][N3];
  __shared__ double sD2[NT];  // D_li^2, indexed l * LX + i
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  const double* Ge = G + (size_t)e * gstride;
  sD2[tid] = c_D[LX][tid] * c_D[LX][tid];
  for (int q = tid; q < N3; q += NT) {
    const double h = h1 ? h1[(size_t)e * N3 + q] : h1c;
    sg[0][q] = Ge[q] * h;
    sg[1][q] = Ge[N3P + q] * h;
    sg[2][q] = Ge[2 * N3P + q] * h;
  }
  __syncthreads();
  // the thread's D^2 columns in registers (the lane-dependent constant-bank
  // reads of the first version serialised within the warp)
  double a2[LX], b2[LX];
#pragma unroll
  for (int l = 0; l < LX; ++l) {
    a2[l] = sD2[l * LX + i];
    b2[l] = sD2[l * LX + j];
  }
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      s += a2[l] * sg[0][l + LX * j + NT * k];
      s += b2[l] * sg[1][i + LX * l + NT * k];
      s += c_D[LX][l * LX + k] * c_D[LX][l * LX + k] * sg[2][i + LX * j + NT * l];
    }
    const double Dii = c_D[LX][i * LX + i], Djj = c_D[LX][j * LX + j], Dkk = c_D[LX][k * LX + k];
    const double hp = h1 ? h1[(size_t)e * N3 + p] : h1c;
    s += 2.0 * Dii * Djj * hp * Ge[3 * N3P + p];
    s += 2.0 * Dii * Dkk * hp * Ge[4 * N3P + p];
    s += 2.0 * Djj * Dkk * hp * Ge[5 * N3P + p];
    const double hm = h2 ? h2[(size_t)e * N3 + p] : h2c;
    if (hm != 0.0) s += hm * B[(size_t)e * N3 + p];
    d[(size_t)e * N3 + p] = s;
  }
}

cudaError_t launch_diag(const sem_mesh* m, const double* h1, const double* h2, double h1c,
                        double h2c, double* d, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_diag<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(
                             m->G, (int64_t)6 * m->n3p, m->B, h1, h2, h1c, h2c, d)));
  return cudaGetLastError();
}

__global__ void k_invert_diag(double* __restrict__ d, const double* __restrict__ mask, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    d[q] = (mask[q] == 0.0) ? 1.0 : 1.0 / d[q];
}
cudaError_t launch_invert_diag(const sem_mesh* m, double* d, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_invert_diag<<<grid_for(m, m->nloc, 256), 256, 0, s>>>(d, m->mask, m->nloc);
  return cudaGetLastError();
}

__global__ void k_mul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                      int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = a[q] * b[q];
}
cudaError_t launch_rhs_local(const sem_mesh* m, const double* f, double* b, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_mul<<<grid_for(m, m->nloc, 256), 256, 0, s>>>(m->B, f, b, m->nloc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// CG (R10).  Scalars live in device memory (CGScalars); kernels read them,
// so the host never synchronises inside an iteration.
// ---------------------------------------------------------------------------
constexpr int kVecThreads = 256;
// grid-stride vector kernels: 8 blocks of 256 per SM (<= kMaxVecBlocks, the
// reduction scratch)
static unsigned vec_blocks(const sem_mesh* m) { return (unsigned)std::min<int64_t>((int64_t)m->nsm * 8, kMaxVecBlocks); }

// generic weighted dot: out = sum mult a b  (b == nullptr -> sum mult a)
__global__ void __launch_bounds__(kVecThreads) k_wdot(const double* __restrict__ a, const double* __restrict__ b,
                                                      const double* __restrict__ mult, int64_t n, double* part,
                                                      unsigned* ticket, double* out) {
  __shared__ double s_red[32];
  __shared__ int s_flag;
  double v[1] = {0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    v[0] += mult[q] * a[q] * (b ? b[q] : 1.0);
  grid_sum_last_block<1>(v, part, ticket, out, s_red, &s_flag);
}

// r = mask b, x = 0, p = 0
__global__ void k_cg_init(const double* __restrict__ b, const double* __restrict__ mask, double* __restrict__ r,
                          double* __restrict__ x, double* __restrict__ p, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    r[q] = mask[q] * b[q];
    x[q] = 0.0;
    p[q] = 0.0;
  }
}

__global__ void k_sub_scalar(double* __restrict__ x, const double* __restrict__ sumv, double nuniq, int64_t n) {
  const double mean = sumv[0] / nuniq;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    x[q] -= mean;
}

// rtr = sum mult r r, rtz = sum mult r (dinv r) of the initial residual
__global__ void __launch_bounds__(kVecThreads) k_cg_start(const double* __restrict__ r, const double* __restrict__ dinv,
                                                          const double* __restrict__ mult, int64_t n, double* part,
                                                          unsigned* ticket, CGScalars* sc) {
  __shared__ double s_red[64];
  __shared__ int s_flag;
  double v[2] = {0.0, 0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double rq = r[q], mq = mult[q];
    v[0] += mq * rq * rq;
    v[1] += mq * rq * (dinv[q] * rq);
  }
  grid_sum_last_block<2>(v, part, ticket, &sc->red[1], s_red, &s_flag);
}

// after the update's rtr, rtz sums: convergence test, beta, the pending alpha
__device__ __forceinline__ void cg_scalar_step(CGScalars* sc) {
  if (sc->done) return;
  sc->iter += 1;
  sc->pAp = sc->red[0];
  sc->alpha = sc->rtz / sc->pAp;
  sc->rtr = sc->red[1];
  const double rtz_new = sc->red[2];
  const double rn = sqrt(sc->rtr);
  if (sc->tol > 0.0 && rn <= sc->tol * sc->bn) {
    sc->converged = 1;
    sc->done = 1;
  }
  if (sc->iter >= sc->maxit) sc->done = 1;
  sc->xalpha = sc->alpha;  // x += alpha p happens in the next operator launch (or k_cg_x_final)
  sc->beta = rtz_new / sc->rtz;
  sc->rtz_prev = sc->rtz;
  sc->rtz = rtz_new;
}

// phase 0: after k_cg_start (bn, rtz); phase 1: after k_cg_update
__global__ void k_cg_scalar(CGScalars* sc, int phase) {
  if (phase == 0) {
    sc->bn = sqrt(sc->red[1]);
    sc->rtz = sc->red[2];
    sc->rtr = sc->red[1];
    sc->beta = 0.0;
    sc->iter = 0;
    sc->breakdown = 0;
    sc->converged = 0;
    sc->done = (sc->bn == 0.0) || (sc->maxit <= 0);
    if (sc->bn == 0.0) sc->converged = 1;
    return;
  }
  cg_scalar_step(sc);
}

// r -= alpha w; partial rtr, rtz with alpha = rtz / pAp.  (x += alpha p is
// deferred: the next operator launch applies it while it reads p, and
// k_cg_x_final after the loop applies the last one.)
// the update's early exits (loop != 0: the iteration is the body of a
// conditional WHILE graph node; every exit path sets whether it goes on):
// false = nothing to do; else *alpha = rtz / pAp
__device__ __forceinline__ bool cg_update_prologue(CGScalars* sc, cudaGraphConditionalHandle loop, double* alpha) {
  if (sc->done) {
    if (loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(loop, 0);
    return false;
  }
  const double pAp = sc->red[0];
  if (!(pAp > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc->breakdown = 1;
      sc->done = 1;
      sc->pAp = pAp;
      if (loop) cudaGraphSetConditional(loop, 0);
    }
    return false;
  }
  *alpha = sc->rtz / pAp;
  return true;
}
// the update's rtr, rtz partials summed by the last block, which also takes
// the scalar step after allreducing them over NVLink (several ranks)
__device__ __forceinline__ void cg_update_tail(double (&v)[2], double* part, unsigned* ticket, CGScalars* sc,
                                               int fuse_scalar, const P2PArgs& p2p, cudaGraphConditionalHandle loop,
                                               double* s_red, int* s_flag) {
  grid_sum_last_block<2>(v, part, ticket, &sc->red[1], s_red, s_flag);
  if (fuse_scalar && *s_flag) {
    if (p2p.peers) {
      __syncthreads();
      if (threadIdx.x < 32) p2p_allreduce_warp(&sc->red[1], 2, p2p, threadIdx.x);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      cg_scalar_step(sc);
      if (loop) cudaGraphSetConditional(loop, sc->done ? 0 : 1);
    }
  }
}

// r -= alpha w; partial rtr, rtz with alpha = rtz / pAp.  (x += alpha p is
// deferred: the next operator launch applies it while it reads p, and
// k_cg_x_final after the loop applies the last one.)  XLX > 0: w (only) is
// in the x-planes-last layout of order XLX (option cg_layout): natural node
// g = e n3 + q reads w[e n3 + xlast_pos(q)].
template <int XLX>
__device__ __forceinline__ int64_t w_index(int64_t g) {
  if constexpr (XLX == 0) {
    return g;
  } else {
    constexpr int N3 = XLX * XLX * XLX;
    const int64_t e = g / N3;
    return e * N3 + xlast_pos<XLX>((int)(g - e * N3));
  }
}
template <int XLX>
__global__ void __launch_bounds__(kVecThreads) k_cg_update(double* __restrict__ r, const double* __restrict__ w,
                                                           const double* __restrict__ dinv,
                                                           const double* __restrict__ mult,
                                                           const uint8_t* __restrict__ m8, int64_t n, double* part,
                                                           unsigned* ticket, CGScalars* sc, int fuse_scalar,
                                                           const P2PArgs p2p, cudaGraphConditionalHandle loop,
                                                           int pdl) {
  __shared__ double s_red[64];
  __shared__ int s_flag;
  if (pdl) {
    griddep_wait();
    if (!SEM_PDL_LATE) griddep_launch_dependents();
  }
  double alpha;
  if (!cg_update_prologue(sc, loop, &alpha)) return;
  double v[2] = {0.0, 0.0};
  if (m8 && ((n & 1) == 0)) {
    // vectorised: 16-byte loads/stores, multiplicity as bytes with a shared
    // table of 1/m (the same IEEE values as the oracle's mult = 1/m)
    __shared__ double s_inv[256];
    s_inv[threadIdx.x] = threadIdx.x ? 1.0 / (double)threadIdx.x : 0.0;
    __syncthreads();
    const int64_t n2 = n >> 1;
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* w2 = reinterpret_cast<const double2*>(w);
    const double2* d2 = reinterpret_cast<const double2*>(dinv);
    const uchar2* mm = reinterpret_cast<const uchar2*>(m8);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n2; q += (int64_t)gridDim.x * blockDim.x) {
      double2 wv;
      if constexpr (XLX == 0) {
        wv = w2[q];
      } else {  // even n3 (the vector path): the pair stays in one element
        wv.x = w[w_index<XLX>(2 * q)];
        wv.y = w[w_index<XLX>(2 * q + 1)];
      }
      const double2 dv = d2[q];
      double2 rv = r2[q];
      const uchar2 mv = mm[q];
      rv.x = rv.x - alpha * wv.x;
      rv.y = rv.y - alpha * wv.y;
      r2[q] = rv;
      const double m0 = s_inv[mv.x], m1 = s_inv[mv.y];
      v[0] += m0 * rv.x * rv.x;
      v[1] += m0 * rv.x * (dv.x * rv.x);
      v[0] += m1 * rv.y * rv.y;
      v[1] += m1 * rv.y * (dv.y * rv.y);
    }
  } else {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
      const double rq = r[q] - alpha * w[w_index<XLX>(q)];
      r[q] = rq;
      const double mq = mult[q];
      v[0] += mq * rq * rq;
      v[1] += mq * rq * (dinv[q] * rq);
    }
  }
  if (pdl && SEM_PDL_LATE) griddep_launch_dependents();  // the next operator may start its G copies
  cg_update_tail(v, part, ticket, sc, fuse_scalar, p2p, loop, s_red, &s_flag);
}

// the last deferred update x += xalpha p (after the iteration loop)
__global__ void k_cg_x_final(double* __restrict__ x, const double* __restrict__ p, int64_t n,
                             const CGScalars* sc) {
  const double xa = sc->xalpha;
  if (xa == 0.0) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    x[q] += xa * p[q];
}

// deterministic sum of n partials into sc->red[0] (pAp)
__global__ void __launch_bounds__(kVecThreads) k_reduce_parts(const double* __restrict__ in, int64_t n, double* part,
                                                              unsigned* ticket, double* out, CGScalars* sc) {
  __shared__ double s_red[32];
  __shared__ int s_flag;
  if (sc && sc->done) return;
  double v[1] = {0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    v[0] += in[q];
  grid_sum_last_block<1>(v, part, ticket, out, s_red, &s_flag);
  // the operator launches before this one consumed the deferred x update
  if (sc && blockIdx.x == 0 && threadIdx.x == 0) sc->xalpha = 0.0;
}

__global__ void k_cg_config(CGScalars* sc, double tol, int maxit, int singular) {
  sc->tol = tol;
  sc->maxit = maxit;
  sc->singular = singular;
}

// the stopping parameters of a device-driven solve (no host copy)
cudaError_t launch_cg_config(sem_mesh* m, double tol, int maxit, int singular, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_config<<<1, 1, 0, s>>>(m->sc, tol, maxit, singular);
  return cudaGetLastError();
}

cudaError_t launch_cg_init(sem_mesh* m, const double* b, double* x, double tol, int maxit, int singular,
                           cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_init<<<vec_blocks(m), kVecThreads, 0, s>>>(b, m->mask, m->r, x, m->p, m->nloc);
  return cudaGetLastError();
}

cudaError_t launch_wdot(sem_mesh* m, const double* a, const double* b, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_wdot<<<vec_blocks(m), kVecThreads, 0, s>>>(a, b, m->mult, m->nloc, m->part, m->ticket, &m->sc->red[slot]);
  return cudaGetLastError();
}

cudaError_t launch_sub_mean(sem_mesh* m, double* x, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_sub_scalar<<<vec_blocks(m), kVecThreads, 0, s>>>(x, &m->sc->red[slot], (double)m->n_unique, m->nloc);
  return cudaGetLastError();
}

cudaError_t launch_cg_start(sem_mesh* m, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_start<<<vec_blocks(m), kVecThreads, 0, s>>>(m->r, m->dinv, m->mult, m->nloc, m->part, m->ticket, m->sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_pap_reduce(sem_mesh* m, cudaStream_t s) {
  // the fused operator left one partial per element in m->part + npart_off
  SEM_COUNT_LAUNCH(m);
  k_reduce_parts<<<vec_blocks(m), kVecThreads, 0, s>>>(m->part + pap_part_offset(), m->pap_nparts, m->part, m->ticket,
                                                    &m->sc->red[0], m->sc);
  return cudaGetLastError();
}

// one resident wave of the update (grid-stride: a second partial wave of
// equal-work blocks would double its tail); per device and instantiation
// (XLX 0: natural w; 2..12: the x-planes-last w of that order)
template <int XLX>
static unsigned update_blocks(const sem_mesh* m) {
  static std::atomic<int> per_sm[64];
  const int dev = (m->device >= 0 && m->device < 64) ? m->device : 0;
  int b = per_sm[dev].load(std::memory_order_acquire);
  if (b == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_cg_update<XLX>, kVecThreads, 0) != cudaSuccess || b < 1) {
      cudaGetLastError();
      b = 4;
    }
    per_sm[dev].store(b, std::memory_order_release);
  }
  return (unsigned)std::min<int64_t>((int64_t)m->nsm * std::min(b, 8), kMaxVecBlocks);
}

cudaError_t launch_cg_update(sem_mesh* m, cudaStream_t s, bool fuse_scalar, cudaGraphConditionalHandle loop,
                             bool pdl) {
  SEM_COUNT_LAUNCH(m);
  const uint8_t* m8 = m->m8;
  const double* mult = m->mult;
  const double* dinv = m->dinv;
  const bool vec = m8 && (((uintptr_t)m->r | (uintptr_t)m->w | (uintptr_t)dinv) & 15) == 0;
  if (m->xl_active) {  // w in the x-planes-last layout (option cg_layout)
    cudaError_t e = cudaErrorInvalidValue;
    SEM_LX_DISPATCH_INT(m->lx, e, (launch_maybe_pdl(pdl, k_cg_update<LX>, dim3(update_blocks<LX>(m)), dim3(kVecThreads), 0,
                                                    s, m->r, (const double*)m->w, dinv, mult,
                                                    (const uint8_t*)(vec ? m8 : nullptr), m->nloc, m->part, m->ticket,
                                                    m->sc, fuse_scalar ? 1 : 0, p2p_args(m), loop, pdl ? 1 : 0)));
    return e;
  }
  return launch_maybe_pdl(pdl, k_cg_update<0>, dim3(update_blocks<0>(m)), dim3(kVecThreads), 0, s, m->r, (const double*)m->w,
                          dinv, mult, (const uint8_t*)(vec ? m8 : nullptr),
                          m->nloc, m->part, m->ticket, m->sc, fuse_scalar ? 1 : 0, p2p_args(m), loop, pdl ? 1 : 0);
}

cudaError_t launch_cg_x_final(sem_mesh* m, double* x, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_x_final<<<vec_blocks(m), kVecThreads, 0, s>>>(x, m->p, m->nloc, m->sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_scalar_step(sem_mesh* m, int phase, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_scalar<<<1, 1, 0, s>>>(m->sc, phase);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kVecThreads) k_count_nz(const double* __restrict__ a, int64_t n, double* part,
                                                          unsigned* ticket, double* out) {
  __shared__ double s_red[32];
  __shared__ int s_flag;
  double v[1] = {0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    v[0] += (a[q] != 0.0) ? 1.0 : 0.0;
  grid_sum_last_block<1>(v, part, ticket, out, s_red, &s_flag);
}

cudaError_t launch_count_nonzero(const double* a, int64_t n, sem_mesh* m, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_count_nz<<<vec_blocks(m), kVecThreads, 0, s>>>(a, n, m->part, m->ticket, &m->sc->red[slot]);
  return cudaGetLastError();
}

int64_t part_capacity(int64_t E) { return kMaxVecBlocks * 4 + 3 * E + 64; }
int64_t pap_part_offset() { return kMaxVecBlocks * 4; }

}  // namespace sem
