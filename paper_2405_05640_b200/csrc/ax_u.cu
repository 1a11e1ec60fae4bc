// CG in the "U layout": the CG vectors hold
// every UNIQUE node once -- each element's interior block (lx-2)^3, then each
// shared entity's nodes (face (lx-2)^2, edge lx-2, vertex 1) in canonical
// order -- instead of the E*lx^3 local copies.  The operator kernel gathers
// an element's operands from the unique vectors into its shared-memory tile
// (reorienting face/edge nodes), computes A_e, writes the interior result
// straight into the unique output and hands the shared-node partials to a
// contiguous buffer S (one slot per copy, canonical order), which a
// segmented sum (k_segsum) reduces into the unique output: the dssum
// (reading R7) becomes a contiguous, deterministic reduction and every CG
// vector pass moves (lx-1)^3/lx^3 (= 0.67 at lx = 8) of the local-layout
// bytes.  Same mathematics as R5/R10; see DESIGN.md.
#include <stdint.h>

#include "device_common.cuh"

namespace sem {

__constant__ double c_Du[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];

cudaError_t upload_basis_u(int N, const double* D) {
  const int lx = N + 1;
  return cudaMemcpyToSymbol(c_Du, D, sizeof(double) * lx * lx,
                            sizeof(double) * lx * (kMaxN + 1) * (kMaxN + 1));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// slot/n decomposition of the 6 M^2 + 12 M + 8 surface items of an element
template <int LX>
__device__ __forceinline__ void surf_item(int it, int* slot, int* n) {
  constexpr int M = LX - 2, MD = M > 0 ? M : 1, NFI = 6 * M * M, NEI = 12 * M;
  if (it < NFI) {
    *slot = it / (MD * MD);
    *n = it % (MD * MD);
  } else if (it < NFI + NEI) {
    *slot = kEdgeSlot0 + (it - NFI) / MD;
    *n = (it - NFI) % MD;
  } else {
    *slot = kVertSlot0 + (it - NFI - NEI);
    *n = 0;
  }
}

struct AxUKP {
  const double* G;
  int64_t gstride;
  const double* B;
  const double* h1;
  const double* h2;
  double h1c, h2c;
  const int64_t* gdesc;  // [E][26] ent_off << 4 | writer << 3 | orient
  const int64_t* wdesc;  // [E][26] target << 2 | direct << 1 | zero
  const double* r;       // unique vectors
  const double* dinv;
  double* p;
  double* w;
  double* S;
  const CGScalars* sc;
  double* part;
  const int32_t* elist;
  int64_t elem0;
};

template <int LX>
__host__ __device__ constexpr int axu_smem_doubles() {
  return ((LX * LX * LX + 1) & ~1) * 9 + ((LX * LX + 1) & ~1) + 32 + 2 * kSlots + 4 /*barriers*/ +
         (6 * (LX - 2) * (LX - 2) + 12 * (LX - 2) + 8 + 3) / 4 /*perm*/;
}

// canonical staging offset of slot s (interior first, then 6 faces, 12
// edges, 8 vertices), and its node count
template <int LX>
__device__ __forceinline__ int stage_base(int slot) {
  constexpr int M = LX - 2, M3 = M * M * M;
  if (slot < kEdgeSlot0) return M3 + slot * M * M;
  if (slot < kVertSlot0) return M3 + 6 * M * M + (slot - kEdgeSlot0) * M;
  return M3 + 6 * M * M + 12 * M + (slot - kVertSlot0);
}

template <int LX, int HM>
__global__ void __launch_bounds__(LX* LX) k_ax_u(AxUKP P) {
  constexpr int N3 = LX * LX * LX, N3P = (N3 + 1) & ~1, NT = LX * LX, M = LX - 2, M3 = M * M * M;
  constexpr int NSURF = 6 * M * M + 12 * M + 8, MD = M > 0 ? M : 1;
  constexpr bool kBulkSeg = (M % 2 == 0);  // face/edge segments are 16-byte multiples
  extern __shared__ __align__(128) double sm[];
  double* sA = sm;                 // stage r (canonical), then the p tile (local order)
  double* sB = sm + N3P;           // stage dinv, then p_new (canonical)
  double* sC = sm + 2 * N3P;       // stage p_old, then the w tile (local order)
  double* sg = sm + 3 * N3P;       // [6][N3P] G, later q_r, q_s
  double* sD = sg + 6 * N3P;
  double* s_red = sD + ((NT + 1) & ~1);
  int64_t* s_gd = (int64_t*)(s_red + 32);  // [26]
  int64_t* s_wd = s_gd + kSlots;           // [26]
  uint64_t* bar = (uint64_t*)(s_wd + kSlots);  // [0] descriptors + interiors, [1] segments, [2] G
  uint16_t* s_perm = (uint16_t*)(bar + 4);        // [NSURF] local offsets of the canonical surface items

  if (P.sc->done) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t q = P.elem0 + blockIdx.x;
  const int64_t e = P.elist ? (int64_t)P.elist[q] : q;
  const size_t ib = (size_t)e * M3;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init(bar + 2, 1);
  }
  for (int t = tid; t < NT; t += NT) sD[t] = c_Du[LX][t];
  __syncthreads();
  if (tid == 0) {
    const uint64_t pol = policy_evict_first();
    const uint32_t ib_bytes = kBulkSeg ? M3 * 8 : 0;
    // the descriptors gate the second-level gathers: they travel alone so
    // the segment copies can start before the 24 KB of G have landed
    mbar_expect_tx(bar, 2 * kSlots * 8 + 3 * ib_bytes);
    bulk_g2s(s_gd, P.gdesc + (size_t)e * kSlots, kSlots * 8, bar, pol);
    bulk_g2s(s_wd, P.wdesc + (size_t)e * kSlots, kSlots * 8, bar, pol);
    if (kBulkSeg && M3 > 0) {
      bulk_g2s(sA, P.r + ib, ib_bytes, bar, pol);
      bulk_g2s(sB, P.dinv + ib, ib_bytes, bar, pol);
      bulk_g2s(sC, P.p + ib, ib_bytes, bar, pol);
    }
    mbar_expect_tx(bar + 2, 6 * N3P * 8);
    bulk_g2s(sg, P.G + (size_t)e * P.gstride, 6 * N3P * 8, bar + 2, pol);
  }
  if (!kBulkSeg)
    for (int t = tid; t < M3; t += NT) {
      sA[t] = P.r[ib + t];
      sB[t] = P.dinv[ib + t];
      sC[t] = P.p[ib + t];
    }
  mbar_wait(bar, 0);
  // shared-node segments: faces and edges by bulk copy (contiguous in the
  // unique vectors, canonical order; issued by the lanes of warp 0), vertices
  // and odd sizes by plain loads
  if (kBulkSeg && tid < 32) {
    if (tid == 0) mbar_expect_tx(bar + 1, 3 * (6 * M * M + 12 * M) * 8);
    __syncwarp(NT >= 32 ? 0xffffffffu : ((1u << NT) - 1u));
    for (int s = tid; s < kVertSlot0; s += (NT < 32 ? NT : 32)) {
      const size_t src = (size_t)(s_gd[s] >> 4);
      const uint32_t nb = (s < kEdgeSlot0 ? M * M : M) * 8;
      const int d = stage_base<LX>(s);
      bulk_g2s_plain(sA + d, P.r + src, nb, bar + 1);
      bulk_g2s_plain(sB + d, P.dinv + src, nb, bar + 1);
      bulk_g2s_plain(sC + d, P.p + src, nb, bar + 1);
    }
  }
  for (int it = kBulkSeg ? (6 * M * M + 12 * M) + tid : tid; it < NSURF; it += NT) {
    int slot, n;
    surf_item<LX>(it, &slot, &n);
    const size_t src = (size_t)(s_gd[slot] >> 4) + n;
    const int d = M3 + it;
    sA[d] = P.r[src];
    sB[d] = P.dinv[src];
    sC[d] = P.p[src];
  }
  // local tile offset of every canonical surface item (used twice)
  for (int it = tid; it < NSURF; it += NT) {
    int slot, n;
    surf_item<LX>(it, &slot, &n);
    s_perm[it] = (uint16_t)node_offset<LX>(slot, (int)(s_gd[slot] & 7), n);
  }
  if (kBulkSeg) mbar_wait(bar + 1, 0);
  mbar_wait(bar + 2, 0);
  __syncthreads();
  // p_new = dinv r + beta p in canonical order; written back once per unique
  // node straight from the stage (interior block, and this element's writer
  // slots -- contiguous runs), and reoriented into the local tile (sA)
  const double beta = P.sc->beta;
  for (int t = tid; t < M3 + NSURF; t += NT) sB[t] = sB[t] * sA[t] + beta * sC[t];
  __syncthreads();
  for (int t = tid; t < M3; t += NT) {
    const double v = sB[t];
    P.p[ib + t] = v;
    const int ti = t % MD, tj = (t / MD) % MD, tk = t / (MD * MD);
    sA[(1 + ti) + LX * ((1 + tj) + LX * (1 + tk))] = v;
  }
  for (int it = tid; it < NSURF; it += NT) {
    int slot, n;
    surf_item<LX>(it, &slot, &n);
    const int64_t gd = s_gd[slot];
    const double v = sB[M3 + it];
    if (gd & 8) P.p[(size_t)(gd >> 4) + n] = v;
    sA[s_perm[it]] = v;
  }
  __syncthreads();
  double* su = sA;

  double Dr[LX], Ds[LX], DTr[LX], DTs[LX], uc[LX], wc[LX];
#pragma unroll
  for (int l = 0; l < LX; ++l) {
    Dr[l] = sD[i * LX + l];
    Ds[l] = sD[j * LX + l];
    DTr[l] = sD[l * LX + i];
    DTs[l] = sD[l * LX + j];
    uc[l] = su[tid + NT * l];
    wc[l] = 0.0;
  }
  const size_t eo = (size_t)e * N3;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      ur = fma(Dr[l], su[l + LX * j + NT * k], ur);
      us = fma(Ds[l], su[i + LX * l + NT * k], us);
      ut = fma(c_Du[LX][k * LX + l], uc[l], ut);
    }
    const double g11 = sg[p], g22 = sg[N3P + p], g33 = sg[2 * N3P + p];
    const double g12 = sg[3 * N3P + p], g13 = sg[4 * N3P + p], g23 = sg[5 * N3P + p];
    double qr = g11 * ur + g12 * us + g13 * ut;
    double qs = g12 * ur + g22 * us + g23 * ut;
    double qt = g13 * ur + g23 * us + g33 * ut;
    if (HM == 2) {
      const double h = P.h1 ? P.h1[eo + p] : P.h1c;
      qr *= h;
      qs *= h;
      qt *= h;
    }
    sg[p] = qr;
    sg[N3P + p] = qs;
#pragma unroll
    for (int mm = 0; mm < LX; ++mm) wc[mm] = fma(c_Du[LX][k * LX + mm], qt, wc[mm]);
  }
  __syncthreads();
  double pap = 0.0;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double s = wc[k];
#pragma unroll
    for (int l = 0; l < LX; ++l) s = fma(DTr[l], sg[l + LX * j + NT * k], s);
#pragma unroll
    for (int l = 0; l < LX; ++l) s = fma(DTs[l], sg[N3P + i + LX * l + NT * k], s);
    if (HM == 0) {
      s *= P.h1c;
    } else if (HM == 1) {
      s = P.h1c * s + P.h2c * P.B[eo + p] * uc[k];
    } else {
      const double hm = P.h2 ? P.h2[eo + p] : P.h2c;
      if (hm != 0.0) s += hm * P.B[eo + p] * uc[k];
    }
    pap += uc[k] * s;
    sC[p] = s;  // w tile
  }
  __syncthreads();
  for (int t = tid; t < M3; t += NT) {
    const int ti = t % MD, tj = (t / MD) % MD, tk = t / (MD * MD);
    P.w[ib + t] = sC[(1 + ti) + LX * ((1 + tj) + LX * (1 + tk))];
  }
  for (int it = tid; it < NSURF; it += NT) {
    int slot, n;
    surf_item<LX>(it, &slot, &n);
    const int64_t wd = s_wd[slot];
    const double v = sC[s_perm[it]];
    if (wd & 2) P.w[(size_t)(wd >> 2) + n] = (wd & 1) ? 0.0 : v;  // single local copy
    else P.S[(size_t)(wd >> 2) + n] = v;
  }
  double v[1] = {pap};
  block_sum<1>(v, s_red);
  if (tid == 0) P.part[q] = v[0];
}

// Segmented sum S -> w (unique): every entity with >= 2 local copies gets
// the sum of its copies in ascending element order (0 if masked).
// Segment descriptors: {uoff, soff | masked << 62, mult} (faces: mult 2).
template <int LX>
__global__ void __launch_bounds__(256) k_segsum(double* __restrict__ w, const double* __restrict__ S,
                                                const int64_t* __restrict__ fseg, int64_t f0, int64_t nf,
                                                const int64_t* __restrict__ xseg, int64_t e0, int64_t ne,
                                                int64_t v0, int64_t nv, const CGScalars* sc) {
  constexpr int M = LX - 2, MD = M > 0 ? M : 1;
  if (sc && sc->done) return;
  const int64_t fItems = nf * M * M, eItems = ne * M, nitems = fItems + eItems + nv;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nitems;
       it += (int64_t)gridDim.x * blockDim.x) {
    if (it < fItems) {
      const int64_t f = f0 + it / (MD * MD);
      const int n = (int)(it % (MD * MD));
      const int64_t uo = fseg[2 * f], so = fseg[2 * f + 1];
      double s = (0.0 + S[(so & ~kFaceMasked) + n]) + S[(so & ~kFaceMasked) + M * M + n];
      w[uo + n] = (so & kFaceMasked) ? 0.0 : s;
      continue;
    }
    int64_t x;
    int n, nodes;
    if (it < fItems + eItems) {
      x = e0 + (it - fItems) / MD;
      n = (int)((it - fItems) % MD);
      nodes = M;
    } else {
      x = v0 + (it - fItems - eItems);
      n = 0;
      nodes = 1;
    }
    const int64_t uo = xseg[3 * x], so = xseg[3 * x + 1] & ~kFaceMasked;
    const int mult = (int)xseg[3 * x + 2];
    double s = 0.0;
    for (int c = 0; c < mult; ++c) s += S[so + (int64_t)c * nodes + n];
    w[uo + n] = (xseg[3 * x + 1] & kFaceMasked) ? 0.0 : s;
  }
}

// x += alpha p; r -= alpha w on all unique local nodes; rtr, rtz (z = dinv r)
// over the owned prefix [0, nown) (interface replicas owned by another rank
// sit after it).
constexpr int kUThreads = 256;
constexpr unsigned kUBlocks = 148 * 8;
__global__ void __launch_bounds__(kUThreads) k_cg_update_u(double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p, const double* __restrict__ w,
                                                           const double* __restrict__ dinv, int64_t nu, int64_t nown,
                                                           double* part, unsigned* ticket, CGScalars* sc) {
  __shared__ double s_red[64];
  __shared__ int s_flag;
  if (sc->done) return;
  const double pAp = sc->red[0];
  if (!(pAp > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc->breakdown = 1;
      sc->done = 1;
      sc->pAp = pAp;
    }
    return;
  }
  const double alpha = sc->rtz / pAp;
  double v[2] = {0.0, 0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nu; q += (int64_t)gridDim.x * blockDim.x) {
    x[q] += alpha * p[q];
    const double rq = r[q] - alpha * w[q];
    r[q] = rq;
    if (q < nown) {
      v[0] += rq * rq;
      v[1] += rq * (dinv[q] * rq);
    }
  }
  grid_sum_last_block<2>(v, part, ticket, &sc->red[1], s_red, &s_flag);
}

// sum over the owned prefix: out = sum a (b == null) or sum a b
__global__ void __launch_bounds__(kUThreads) k_dot_u(const double* __restrict__ a, const double* __restrict__ b,
                                                     int64_t nown, double* part, unsigned* ticket, double* out) {
  __shared__ double s_red[32];
  __shared__ int s_flag;
  double v[1] = {0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nown; q += (int64_t)gridDim.x * blockDim.x)
    v[0] += a[q] * (b ? b[q] : 1.0);
  grid_sum_last_block<1>(v, part, ticket, out, s_red, &s_flag);
}

__global__ void k_sub_mean_u(double* __restrict__ x, const double* __restrict__ sumv, double nuniq, int64_t n) {
  const double mean = sumv[0] / nuniq;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    x[q] -= mean;
}

// local <-> unique conversions, one CTA per element.  l2u: every unique node
// takes the value of the copy that writes it (the element's interior, and
// its writer slots), times mask if given.  u2l: every local copy takes its
// unique value.
template <int LX>
__global__ void __launch_bounds__(LX* LX) k_l2u(const double* __restrict__ loc, const double* __restrict__ mask,
                                                const int64_t* __restrict__ gdesc, double* __restrict__ u) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX, M = LX - 2, M3 = M * M * M;
  constexpr int NSURF = 6 * M * M + 12 * M + 8, MD = M > 0 ? M : 1;
  const int tid = threadIdx.x + LX * threadIdx.y;
  const int64_t e = blockIdx.x;
  const size_t eo = (size_t)e * N3, ib = (size_t)e * M3;
  for (int t = tid; t < M3; t += NT) {
    const int p = (1 + t % MD) + LX * ((1 + (t / MD) % MD) + LX * (1 + t / (MD * MD)));
    u[ib + t] = loc[eo + p] * (mask ? mask[eo + p] : 1.0);
  }
  for (int it = tid; it < NSURF; it += NT) {
    int slot, n;
    surf_item<LX>(it, &slot, &n);
    const int64_t gd = gdesc[(size_t)e * kSlots + slot];
    if (!(gd & 8)) continue;
    const int p = node_offset<LX>(slot, (int)(gd & 7), n);
    u[(size_t)(gd >> 4) + n] = loc[eo + p] * (mask ? mask[eo + p] : 1.0);
  }
}

template <int LX>
__global__ void __launch_bounds__(LX* LX) k_u2l(const double* __restrict__ u, const int64_t* __restrict__ gdesc,
                                                double* __restrict__ loc) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX, M = LX - 2, M3 = M * M * M;
  constexpr int NSURF = 6 * M * M + 12 * M + 8, MD = M > 0 ? M : 1;
  const int tid = threadIdx.x + LX * threadIdx.y;
  const int64_t e = blockIdx.x;
  const size_t eo = (size_t)e * N3, ib = (size_t)e * M3;
  for (int t = tid; t < M3; t += NT) {
    const int p = (1 + t % MD) + LX * ((1 + (t / MD) % MD) + LX * (1 + t / (MD * MD)));
    loc[eo + p] = u[ib + t];
  }
  for (int it = tid; it < NSURF; it += NT) {
    int slot, n;
    surf_item<LX>(it, &slot, &n);
    const int64_t gd = gdesc[(size_t)e * kSlots + slot];
    loc[eo + node_offset<LX>(slot, (int)(gd & 7), n)] = u[(size_t)(gd >> 4) + n];
  }
}

// interface exchange in the U layout: own partial = the entity's segment
__global__ void k_ifu_gather(const double* __restrict__ w, const int64_t* __restrict__ uoff,
                             const int32_t* __restrict__ node_ent, const int64_t* __restrict__ noff, int64_t nn,
                             double* __restrict__ U) {
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nn; it += (int64_t)gridDim.x * blockDim.x) {
    const int q = node_ent[it];
    U[it] = w[uoff[q] + (it - noff[q])];
  }
}

__global__ void k_ifu_scatter(double* __restrict__ w, const int64_t* __restrict__ uoff,
                              const int32_t* __restrict__ node_ent, const int64_t* __restrict__ noff,
                              const int32_t* __restrict__ src_ptr, const int64_t* __restrict__ src,
                              const uint8_t* __restrict__ ent_flags, const int32_t* __restrict__ if_ent, int64_t nn,
                              const double* __restrict__ U) {
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nn; it += (int64_t)gridDim.x * blockDim.x) {
    const int q = node_ent[it];
    const int64_t n = it - noff[q];
    double s = 0.0;
    for (int k = src_ptr[q]; k < src_ptr[q + 1]; ++k) s += U[src[k] + n];
    if (ent_flags[if_ent[q]] & kEntMasked) s = 0.0;
    w[uoff[q] + n] = s;
  }
}

static unsigned gridu(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

#define SEM_LX_CASES(CALL)                                            \
  switch (m->lx) {                                                    \
    case 2: { constexpr int LX = 2; CALL; } break;                    \
    case 3: { constexpr int LX = 3; CALL; } break;                    \
    case 4: { constexpr int LX = 4; CALL; } break;                    \
    case 5: { constexpr int LX = 5; CALL; } break;                    \
    case 6: { constexpr int LX = 6; CALL; } break;                    \
    case 7: { constexpr int LX = 7; CALL; } break;                    \
    case 8: { constexpr int LX = 8; CALL; } break;                    \
    case 9: { constexpr int LX = 9; CALL; } break;                    \
    case 10: { constexpr int LX = 10; CALL; } break;                  \
    case 11: { constexpr int LX = 11; CALL; } break;                  \
    case 12: { constexpr int LX = 12; CALL; } break;                  \
    default: return cudaErrorInvalidValue;                            \
  }

template <int LX, int HM>
static cudaError_t launch_axu_t(const sem_mesh* m, const AxUKP& P, int64_t count, cudaStream_t s) {
  const size_t smem = sizeof(double) * axu_smem_doubles<LX>();
  auto kern = k_ax_u<LX, HM>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (count <= 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  kern<<<(unsigned)count, dim3(LX, LX), smem, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_ax_u(const sem_mesh* m, const AxArgs& a, int64_t elem0, int64_t count, cudaStream_t s) {
  AxUKP P;
  P.G = m->G;
  P.gstride = (int64_t)6 * m->n3p;
  P.B = m->B;
  P.h1 = a.h1;
  P.h2 = a.h2;
  P.h1c = a.h1c;
  P.h2c = a.h2c;
  P.gdesc = m->d_gdesc;
  P.wdesc = m->d_wdesc;
  P.r = m->ur;
  P.dinv = m->udinv;
  P.p = m->up;
  P.w = m->uw;
  P.S = m->d_Su;
  P.sc = m->sc;
  P.part = a.part;
  P.elist = m->d_elist_all;
  P.elem0 = elem0;
  const int HM = (a.h1 || a.h2) ? 2 : (a.h2c == 0.0 ? 0 : 1);
  SEM_LX_CASES((HM == 0 ? launch_axu_t<LX, 0>(m, P, count, s)
                        : HM == 1 ? launch_axu_t<LX, 1>(m, P, count, s) : launch_axu_t<LX, 2>(m, P, count, s)));
  return cudaGetLastError();
}

cudaError_t launch_segsum(const sem_mesh* m, int64_t c0, int64_t c1, cudaStream_t s) {
  const int64_t f0 = m->useg_f[c0], nf = m->useg_f[c1] - f0;
  const int64_t e0 = m->useg_e[c0], ne = m->useg_e[c1] - e0;
  const int64_t v0 = m->useg_v[c0], nv = m->useg_v[c1] - v0;
  const int64_t M = m->lx - 2, n = nf * M * M + ne * M + nv;
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_CASES((k_segsum<LX><<<gridu(n), 256, 0, s>>>(m->uw, m->d_Su, m->d_fseg, f0, nf, m->d_xseg, e0, ne,
                                                      m->nseg_e + v0, nv, m->sc)));
  return cudaGetLastError();
}

cudaError_t launch_cg_update_u(sem_mesh* m, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_update_u<<<kUBlocks, kUThreads, 0, s>>>(m->ux, m->ur, m->up, m->uw, m->udinv, m->n_u, m->n_own, m->part,
                                               m->ticket, m->sc);
  return cudaGetLastError();
}

cudaError_t launch_dot_u(sem_mesh* m, const double* a, const double* b, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_dot_u<<<kUBlocks, kUThreads, 0, s>>>(a, b, m->n_own, m->part, m->ticket, &m->sc->red[slot]);
  return cudaGetLastError();
}

cudaError_t launch_sub_mean_u(sem_mesh* m, double* x, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_sub_mean_u<<<kUBlocks, kUThreads, 0, s>>>(x, &m->sc->red[slot], (double)m->n_unique, m->n_u);
  return cudaGetLastError();
}

cudaError_t launch_l2u(const sem_mesh* m, const double* loc, const double* mask, double* u, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_CASES((k_l2u<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(loc, mask, m->d_gdesc, u)));
  return cudaGetLastError();
}

cudaError_t launch_u2l(const sem_mesh* m, const double* u, double* loc, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_CASES((k_u2l<LX><<<(unsigned)m->E, dim3(LX, LX), 0, s>>>(u, m->d_gdesc, loc)));
  return cudaGetLastError();
}

cudaError_t launch_ifu_gather(const sem_mesh* m, const double* w, cudaStream_t s) {
  if (m->n_if_nodes == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  k_ifu_gather<<<gridu(m->n_if_nodes), 256, 0, s>>>(w, m->d_if_uoff, m->d_if_node_ent, m->d_if_noff, m->n_if_nodes,
                                                    m->d_U);
  return cudaGetLastError();
}

cudaError_t launch_ifu_scatter(const sem_mesh* m, double* w, cudaStream_t s) {
  if (m->n_if_nodes == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  k_ifu_scatter<<<gridu(m->n_if_nodes), 256, 0, s>>>(w, m->d_if_uoff, m->d_if_node_ent, m->d_if_noff,
                                                     m->d_if_src_ptr, m->d_if_src, m->d_ent_flags, m->d_if_ent,
                                                     m->n_if_nodes, m->d_U);
  return cudaGetLastError();
}

}  // namespace sem

namespace sem {
__global__ void __launch_bounds__(kUThreads) k_cg_start_u(const double* __restrict__ r, const double* __restrict__ dinv,
                                                          int64_t nown, double* part, unsigned* ticket, CGScalars* sc) {
  __shared__ double s_red[64];
  __shared__ int s_flag;
  double v[2] = {0.0, 0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nown; q += (int64_t)gridDim.x * blockDim.x) {
    const double rq = r[q];
    v[0] += rq * rq;
    v[1] += rq * (dinv[q] * rq);
  }
  grid_sum_last_block<2>(v, part, ticket, &sc->red[1], s_red, &s_flag);
}
__global__ void k_zero2(double* __restrict__ a, double* __restrict__ b, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    a[q] = 0.0;
    b[q] = 0.0;
  }
}
cudaError_t launch_cg_start_u(sem_mesh* m, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_start_u<<<kUBlocks, kUThreads, 0, s>>>(m->ur, m->udinv, m->n_own, m->part, m->ticket, m->sc);
  return cudaGetLastError();
}
cudaError_t launch_zero2(sem_mesh* m, double* a, double* b, int64_t n, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_zero2<<<kUBlocks, kUThreads, 0, s>>>(a, b, n);
  return cudaGetLastError();
}
}  // namespace sem
