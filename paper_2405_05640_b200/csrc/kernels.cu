// sm_100a kernels of the SEM hot path (arXiv 2405.05640).
//
//   k_geom      geometric factors G_ab, B (reading R4), once per mesh
//   k_ax        local operator A_e u (R5), optionally fused with
//                 - the CG prologue p <- dinv r + beta p and the pAp partial,
//                 - the gather-scatter dssum + mask (R7, R8) done by the
//                   LAST element to finish each shared face/edge/vertex
//   k_gs        standalone gather-scatter (ADD / MASK)
//   k_diag      exact local Jacobi diagonal (R9)
//   CG vector kernels and deterministic two-stage reductions (R10)
//
// Data layout: fields [E][lx^3] fp64; G [E][6][n3p]
// (n3p = n3 rounded up to even so every element's 6 factors are one
// 16-byte-aligned contiguous block that a single cp.async.bulk (TMA) moves
// into shared memory).
#include <stdint.h>

#include "internal.h"

#define SEM_COUNT_LAUNCH(m) (const_cast<sem_mesh*>(m)->nlaunch++)

namespace sem {

__constant__ double c_D[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];  // c_D[lx][i*lx+l] = D_il
__constant__ double c_w[kMaxN + 2][kMaxN + 1];

cudaError_t upload_basis(int N, const double* D, const double* w) {
  const int lx = N + 1;
  cudaError_t e = cudaMemcpyToSymbol(c_D, D, sizeof(double) * lx * lx,
                                     sizeof(double) * lx * (kMaxN + 1) * (kMaxN + 1));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_w, w, sizeof(double) * lx, sizeof(double) * lx * (kMaxN + 1));
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + 1D bulk async copy (TMA engine), L2 policy
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Local node offset of canonical node n of an entity copy (slot, orient);
// device twin of copy_node_offset() in topo.cpp.
template <int LX>
__device__ __forceinline__ int node_offset(int slot, int orient, int n) {
  constexpr int N = LX - 1, M = LX - 2, MD = M > 0 ? M : 1;
  int i, j, k;
  if (slot < kEdgeSlot0) {
    const int a = n % MD, b = n / MD;
    const int du = (orient & 4) ? b : a, dv = (orient & 4) ? a : b;
    const int u = 1 + ((orient & 1) ? M - 1 - du : du);
    const int v = 1 + ((orient & 2) ? M - 1 - dv : dv);
    const int side = (slot & 1) ? N : 0, ax = slot >> 1;
    i = ax == 0 ? side : u;
    j = ax == 0 ? u : (ax == 1 ? side : v);
    k = ax == 2 ? side : v;
  } else if (slot < kVertSlot0) {
    const int ed = slot - kEdgeSlot0, ax = ed >> 2, q = ed & 3;
    const int t = 1 + ((orient & 1) ? M - 1 - n : n);
    const int p = (q & 1) * N, r = (q >> 1) * N;
    i = ax == 0 ? t : p;
    j = ax == 0 ? p : (ax == 1 ? t : r);
    k = ax == 2 ? t : r;
  } else {
    const int c = slot - kVertSlot0;
    i = (c & 1) * N;
    j = ((c >> 1) & 1) * N;
    k = (c >> 2) * N;
  }
  return i + LX * (j + LX * k);
}

// deterministic block sum of NV values (fixed tree); result valid in thread 0
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* s_red /* >= 32*NV */) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nt = blockDim.x * blockDim.y * blockDim.z;
  const int nw = (nt + 31) >> 5;
  const int lane = tid & 31;
  const int active = min(32, nt - (tid & ~31));  // lanes present in this warp
  const unsigned wmask = active == 32 ? 0xffffffffu : ((1u << active) - 1u);
#pragma unroll
  for (int q = 0; q < NV; ++q)
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_down_sync(wmask, v[q], o);
      if (lane + o < active) v[q] += t;
    }
  if ((tid & 31) == 0)
    for (int q = 0; q < NV; ++q) s_red[q * 32 + (tid >> 5)] = v[q];
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += s_red[q * 32 + w];
      v[q] = s;
    }
}

// Partials written per block, the last block to arrive (ticket) sums them in
// block order -> deterministic.  part: [nblk][NV]; out: NV doubles.
template <int NV>
__device__ __forceinline__ void grid_sum_last_block(double (&v)[NV], double* part, unsigned* ticket,
                                                    double* out, double* s_red, int* s_flag) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nt = blockDim.x * blockDim.y * blockDim.z;
  const unsigned nblk = gridDim.x;
  block_sum<NV>(v, s_red);
  if (tid == 0) {
    for (int q = 0; q < NV; ++q) part[(size_t)blockIdx.x * NV + q] = v[q];
    __threadfence();
    const unsigned t = atomicInc(ticket, nblk - 1);
    *s_flag = (t == nblk - 1);
  }
  __syncthreads();
  if (*s_flag) {
    __threadfence();
    double acc[NV];
    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
    for (unsigned b = tid; b < nblk; b += nt)
      for (int q = 0; q < NV; ++q) acc[q] += __ldcg(&part[(size_t)b * NV + q]);
    __syncthreads();
    block_sum<NV>(acc, s_red);
    if (tid == 0)
      for (int q = 0; q < NV; ++q) out[q] = acc[q];
  }
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

// ---------------------------------------------------------------------------
// Fused local operator.  One CTA of lx*lx threads per element; thread (i,j)
// owns the column (i,j,:) in registers (t-direction contractions never touch
// shared memory); the r/s contractions read the element's u tile in shared
// memory.  G (6 factors) and u arrive by one TMA bulk copy per element.
//   HM = 0: h1 = h1c constant, h2 = 0 (Poisson when h1c = 1)
//   HM = 1: h1c, h2c constants
//   HM = 2: h1/h2 arrays (NULL array -> its constant)
//   GS:     dssum + mask by the last arriver of each shared entity
//   CG:     u := p = dinv r + beta p (written back), pAp partial per CTA
// ---------------------------------------------------------------------------
struct AxKP {
  const double* u;
  double* w;
  const double* G;
  const double* B;
  int64_t gstride;
  const double* h1;
  const double* h2;
  double h1c, h2c;
  const double* r;
  const double* dinv;
  double* p;
  const CGScalars* sc;
  double* part;
  const int32_t* elist;
  int u_bulk;  // u element blocks are 16-byte aligned -> TMA bulk copy
  GsPlan plan;
};

// Shared-memory scratch of the gather-scatter epilogue.
struct GsSmem {
  int64_t cp[kSlots][8];   // staged copies (element, slot, orient) of each last-arrived entity
  int pre[kSlots + 1];     // prefix of node counts over slots
  int mult[kSlots];        // copies of the entity (0 = nothing to do)
  int ent[kSlots];
  uint8_t fl[kSlots];
};

// Gather-scatter (dssum + mask, readings R7/R8) of element e's shared nodes,
// done by the LAST element to finish each shared entity.  Every thread of
// the CTA has already stored its part of w.  One atom.acq_rel per entity
// (release: this CTA's w stores, made visible CTA-wide by the barrier;
// acquire: the other copies' stores); the last arriver sums all copies in
// ascending element order and writes the sum (0 if masked) to every copy.
template <int LX>
__device__ __forceinline__ void gs_last_arriver(double* __restrict__ w, const GsPlan& plan, int64_t e, int tid,
                                                GsSmem* S) {
  constexpr int N3 = LX * LX * LX, NT = LX * LX, M = LX - 2;
  __syncthreads();
  for (int ts = tid; ts < kSlots; ts += NT) {
    const int ent = plan.elem_ent[(size_t)e * kSlots + ts];
    const int c0 = plan.ent_ptr[ent], mult = plan.ent_ptr[ent + 1] - c0;
    const uint8_t fl = plan.ent_flags[ent];
    int todo = 0;
    if (mult > 1 || (fl & kEntMasked)) {
      unsigned old;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(plan.ent_cnt + ent) : "memory");
      if (old == (unsigned)(mult - 1)) {
        plan.ent_cnt[ent] = 0u;  // every copy has arrived: nobody else touches it in this launch
        todo = mult;
        if (mult <= 8)
          for (int c = 0; c < mult; ++c) S->cp[ts][c] = plan.ent_copy[c0 + c];
      }
    }
    S->mult[ts] = todo;
    S->ent[ts] = c0;
    S->fl[ts] = fl;
    S->pre[ts + 1] = todo ? (ts < kEdgeSlot0 ? M * M : (ts < kVertSlot0 ? M : 1)) : 0;
  }
  __syncthreads();
  if (NT >= 32) {
    if (tid < 32) {  // warp-inclusive scan of the 26 node counts
      int v = tid < kSlots ? S->pre[tid + 1] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if ((tid & 31) >= o) v += t;
      }
      if (tid < kSlots) S->pre[tid + 1] = v;
      if (tid == 0) S->pre[0] = 0;
    }
  } else if (tid == 0) {
    S->pre[0] = 0;
    for (int s = 0; s < kSlots; ++s) S->pre[s + 1] += S->pre[s];
  }
  __syncthreads();
  const int total = S->pre[kSlots];
  for (int it = tid; it < total; it += NT) {
    int lo = 0, hi = kSlots;  // find s with pre[s] <= it < pre[s+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (S->pre[mid] <= it) lo = mid;
      else hi = mid;
    }
    const int s = lo, n = it - S->pre[s], mult = S->mult[s];
    const bool masked = S->fl[s] & kEntMasked;
    if (mult <= 8) {
      size_t off[8];
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < mult) {
          const int64_t cp = S->cp[s][c];
          off[c] = (size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n);
          v[c] = __ldcg(&w[off[c]]);
        }
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < mult) sum += v[c];
      if (masked) sum = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < mult) w[off[c]] = sum;
    } else {
      const int c0 = S->ent[s];
      double sum = 0.0;
      for (int c = 0; c < mult; ++c) {
        const int64_t cp = plan.ent_copy[c0 + c];
        sum += __ldcg(&w[(size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n)]);
      }
      if (masked) sum = 0.0;
      for (int c = 0; c < mult; ++c) {
        const int64_t cp = plan.ent_copy[c0 + c];
        w[(size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n)] = sum;
      }
    }
  }
}

template <int LX>
constexpr int ax_smem_doubles() {
  return ((LX * LX * LX + 1) & ~1) * 7 + ((LX * LX + 1) & ~1) + 32 /*red*/ + 2 /*bar*/ +
         (int)((sizeof(GsSmem) + 7) / 8);
}

template <int LX, int HM, bool GS, bool CG>
__global__ void __launch_bounds__(LX* LX) k_ax(AxKP P) {
  constexpr int N3 = LX * LX * LX, N3P = (N3 + 1) & ~1, NT = LX * LX, M = LX - 2;
  extern __shared__ __align__(128) double sm[];
  double* su = sm;                   // [N3P]    u (or p)
  double* sg = su + N3P;             // [6][N3P] G, later q_r (slot 0) and q_s (slot 1)
  double* sD = sg + 6 * N3P;         // [LX*LX]
  double* s_red = sD + ((NT + 1) & ~1);  // [32]
  uint64_t* bar = (uint64_t*)(s_red + 32);
  GsSmem* s_gs = (GsSmem*)(bar + 2);

  if (CG && P.sc->done) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = P.elist ? (int64_t)P.elist[blockIdx.x] : (int64_t)blockIdx.x;
  const size_t eo = (size_t)e * N3;
  const bool kBulkU = !CG && P.u_bulk;

  if (tid == 0) mbar_init(bar, 1);
  for (int q = tid; q < NT; q += NT) sD[q] = c_D[LX][q];
  __syncthreads();
  if (tid == 0) {
    const uint64_t pol = policy_evict_first();
    mbar_expect_tx(bar, 6 * N3P * 8 + (kBulkU ? N3 * 8 : 0));
    bulk_g2s(sg, P.G + (size_t)e * P.gstride, 6 * N3P * 8, bar, pol);
    if (kBulkU) bulk_g2s(su, P.u + eo, N3 * 8, bar, pol);
  }
  if (CG) {
    const double beta = P.sc->beta;
    for (int q = tid; q < N3; q += NT) {
      const double pn = P.dinv[eo + q] * P.r[eo + q] + beta * P.p[eo + q];
      P.p[eo + q] = pn;
      su[q] = pn;
    }
  } else if (!kBulkU) {
    for (int q = tid; q < N3; q += NT) su[q] = P.u[eo + q];
  }
  __syncthreads();
  mbar_wait(bar, 0);

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
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      ur = fma(Dr[l], su[l + LX * j + NT * k], ur);
      us = fma(Ds[l], su[i + LX * l + NT * k], us);
      ut = fma(c_D[LX][k * LX + l], uc[l], ut);
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
    for (int mm = 0; mm < LX; ++mm) wc[mm] = fma(c_D[LX][k * LX + mm], qt, wc[mm]);
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
    if (CG) pap += uc[k] * s;
    P.w[eo + p] = s;
  }
  if (CG) {
    double v[1] = {pap};
    block_sum<1>(v, s_red);
    if (tid == 0) P.part[blockIdx.x] = v[0];
  }
  if (!GS) return;

  // ---- gather-scatter by the last arriver of each shared entity ----------
  gs_last_arriver<LX>(P.w, P.plan, e, tid, s_gs);
}

template <int LX, int HM, bool GS, bool CG>
static cudaError_t launch_ax_t(const sem_mesh* m, const AxKP& P, int64_t nelem, cudaStream_t s) {
  const size_t smem = sizeof(double) * ax_smem_doubles<LX>();
  auto kern = k_ax<LX, HM, GS, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (nelem == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  kern<<<(unsigned)nelem, dim3(LX, LX), smem, s>>>(P);
  return cudaGetLastError();
}

template <int LX>
static cudaError_t launch_ax_lx(const sem_mesh* m, const AxKP& P, int HM, bool gs, bool cg,
                                int64_t nelem, cudaStream_t s) {
  if (cg) {
    switch (HM) {
      case 0: return launch_ax_t<LX, 0, true, true>(m, P, nelem, s);
      case 1: return launch_ax_t<LX, 1, true, true>(m, P, nelem, s);
      default: return launch_ax_t<LX, 2, true, true>(m, P, nelem, s);
    }
  }
  if (gs) {
    switch (HM) {
      case 0: return launch_ax_t<LX, 0, true, false>(m, P, nelem, s);
      case 1: return launch_ax_t<LX, 1, true, false>(m, P, nelem, s);
      default: return launch_ax_t<LX, 2, true, false>(m, P, nelem, s);
    }
  }
  switch (HM) {
    case 0: return launch_ax_t<LX, 0, false, false>(m, P, nelem, s);
    case 1: return launch_ax_t<LX, 1, false, false>(m, P, nelem, s);
    default: return launch_ax_t<LX, 2, false, false>(m, P, nelem, s);
  }
}

cudaError_t launch_ax(const sem_mesh* m, const AxArgs& a, bool gs, bool cg, cudaStream_t s) {
  AxKP P;
  P.u = a.u;
  P.w = a.w;
  P.G = m->G;
  P.B = m->B;
  P.gstride = (int64_t)6 * m->n3p;
  P.h1 = a.h1;
  P.h2 = a.h2;
  P.h1c = a.h1c;
  P.h2c = a.h2c;
  P.r = a.r;
  P.dinv = a.dinv;
  P.p = a.p;
  P.sc = a.sc;
  P.part = a.part;
  P.elist = nullptr;
  P.u_bulk = (m->n3 % 2 == 0) && a.u && (((uintptr_t)a.u & 15) == 0);
  P.plan = m->plan();
  int HM = 2;
  if (!a.h1 && !a.h2) HM = (a.h2c == 0.0) ? 0 : 1;
  const int64_t nelem = m->E;
  switch (m->lx) {
    case 2: return launch_ax_lx<2>(m, P, HM, gs, cg, nelem, s);
    case 3: return launch_ax_lx<3>(m, P, HM, gs, cg, nelem, s);
    case 4: return launch_ax_lx<4>(m, P, HM, gs, cg, nelem, s);
    case 5: return launch_ax_lx<5>(m, P, HM, gs, cg, nelem, s);
    case 6: return launch_ax_lx<6>(m, P, HM, gs, cg, nelem, s);
    case 7: return launch_ax_lx<7>(m, P, HM, gs, cg, nelem, s);
    case 8: return launch_ax_lx<8>(m, P, HM, gs, cg, nelem, s);
    case 9: return launch_ax_lx<9>(m, P, HM, gs, cg, nelem, s);
    case 10: return launch_ax_lx<10>(m, P, HM, gs, cg, nelem, s);
    case 11: return launch_ax_lx<11>(m, P, HM, gs, cg, nelem, s);
    case 12: return launch_ax_lx<12>(m, P, HM, gs, cg, nelem, s);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Standalone gather-scatter over entity nodes (one thread per entity node).
// ---------------------------------------------------------------------------
template <int LX>
__global__ void k_gs(double* __restrict__ u, GsPlan plan, int op, int64_t nitems) {
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
    const uint8_t fl = plan.ent_flags[ent];
    double sum = 0.0;
    if (op == SEM_GS_ADD) {
      if (c1 - c0 == 1) continue;
      for (int c = c0; c < c1; ++c) {
        const int64_t cp = plan.ent_copy[c];
        sum += u[(size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n)];
      }
    } else {
      if (!(fl & kEntMasked)) continue;
    }
    for (int c = c0; c < c1; ++c) {
      const int64_t cp = plan.ent_copy[c];
      u[(size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n)] = sum;
    }
  }
}

// mult (1/m) and mask (0/1) per local node
template <int LX>
__global__ void k_mult_mask(double* __restrict__ mult, double* __restrict__ mask, GsPlan plan,
                            int64_t nitems) {
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
    const double mv = 1.0 / (double)(c1 - c0);
    const double kv = (plan.ent_flags[ent] & kEntMasked) ? 0.0 : 1.0;
    for (int c = c0; c < c1; ++c) {
      const int64_t cp = plan.ent_copy[c];
      const size_t o = (size_t)(cp >> 8) * N3 + node_offset<LX>((int)((cp >> 3) & 31), (int)(cp & 7), n);
      mult[o] = mv;
      mask[o] = kv;
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

#define SEM_LX_DISPATCH(LXV, CALL)                  \
  switch (LXV) {                                    \
    case 2: { constexpr int LX = 2; CALL; } break;  \
    case 3: { constexpr int LX = 3; CALL; } break;  \
    case 4: { constexpr int LX = 4; CALL; } break;  \
    case 5: { constexpr int LX = 5; CALL; } break;  \
    case 6: { constexpr int LX = 6; CALL; } break;  \
    case 7: { constexpr int LX = 7; CALL; } break;  \
    case 8: { constexpr int LX = 8; CALL; } break;  \
    case 9: { constexpr int LX = 9; CALL; } break;  \
    case 10: { constexpr int LX = 10; CALL; } break; \
    case 11: { constexpr int LX = 11; CALL; } break; \
    case 12: { constexpr int LX = 12; CALL; } break; \
    default: return cudaErrorInvalidValue;          \
  }

static unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
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

cudaError_t launch_gs(const sem_mesh* m, double* u, int op, cudaStream_t s) {
  const int64_t n = gs_items(m);
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_gs<LX><<<grid_for(n, 256), 256, 0, s>>>(u, m->plan(), op, n)));
  return cudaGetLastError();
}

cudaError_t launch_mult_mask(const sem_mesh* m, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_fill<<<grid_for(m->nloc, 256), 256, 0, s>>>(m->mult, 1.0, m->nloc);
  SEM_COUNT_LAUNCH(m);
  k_fill<<<grid_for(m->nloc, 256), 256, 0, s>>>(m->mask, 1.0, m->nloc);
  const int64_t n = gs_items(m);
  if (n == 0) return cudaGetLastError();
  SEM_COUNT_LAUNCH(m);
  SEM_LX_DISPATCH(m->lx, (k_mult_mask<LX><<<grid_for(n, 256), 256, 0, s>>>(m->mult, m->mask, m->plan(), n)));
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
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t e = blockIdx.x;
  const double* Ge = G + (size_t)e * gstride;
  for (int q = tid; q < N3; q += NT) {
    const double h = h1 ? h1[(size_t)e * N3 + q] : h1c;
    sg[0][q] = Ge[q] * h;
    sg[1][q] = Ge[N3P + q] * h;
    sg[2][q] = Ge[2 * N3P + q] * h;
  }
  __syncthreads();
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double s = 0.0;
    for (int l = 0; l < LX; ++l) {
      const double a = c_D[LX][l * LX + i], b = c_D[LX][l * LX + j], c = c_D[LX][l * LX + k];
      s += a * a * sg[0][l + LX * j + NT * k];
      s += b * b * sg[1][i + LX * l + NT * k];
      s += c * c * sg[2][i + LX * j + NT * l];
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
  k_invert_diag<<<grid_for(m->nloc, 256), 256, 0, s>>>(d, m->mask, m->nloc);
  return cudaGetLastError();
}

__global__ void k_mul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                      int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = a[q] * b[q];
}
cudaError_t launch_rhs_local(const sem_mesh* m, const double* f, double* b, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_mul<<<grid_for(m->nloc, 256), 256, 0, s>>>(m->B, f, b, m->nloc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// CG (R10).  Scalars live in device memory (CGScalars); kernels read them,
// so the host never synchronises inside an iteration.
// ---------------------------------------------------------------------------
constexpr int kVecThreads = 256;
constexpr unsigned kVecBlocks = 148 * 8;

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

// x += alpha p; r -= alpha w; partial rtr, rtz with alpha = rtz / pAp
__global__ void __launch_bounds__(kVecThreads) k_cg_update(double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p, const double* __restrict__ w,
                                                           const double* __restrict__ dinv,
                                                           const double* __restrict__ mult, int64_t n, double* part,
                                                           unsigned* ticket, CGScalars* sc) {
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
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    x[q] += alpha * p[q];
    const double rq = r[q] - alpha * w[q];
    r[q] = rq;
    const double mq = mult[q];
    v[0] += mq * rq * rq;
    v[1] += mq * rq * (dinv[q] * rq);
  }
  grid_sum_last_block<2>(v, part, ticket, &sc->red[1], s_red, &s_flag);
}

// deterministic sum of n partials into sc->red[0] (pAp)
__global__ void __launch_bounds__(kVecThreads) k_reduce_parts(const double* __restrict__ in, int64_t n, double* part,
                                                              unsigned* ticket, double* out, const CGScalars* sc) {
  __shared__ double s_red[32];
  __shared__ int s_flag;
  if (sc && sc->done) return;
  double v[1] = {0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    v[0] += in[q];
  grid_sum_last_block<1>(v, part, ticket, out, s_red, &s_flag);
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
  sc->beta = rtz_new / sc->rtz;
  sc->rtz_prev = sc->rtz;
  sc->rtz = rtz_new;
}

cudaError_t launch_cg_init(sem_mesh* m, const double* b, double* x, double tol, int maxit, int singular,
                           cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_init<<<kVecBlocks, kVecThreads, 0, s>>>(b, m->mask, m->r, x, m->p, m->nloc);
  return cudaGetLastError();
}

cudaError_t launch_wdot(sem_mesh* m, const double* a, const double* b, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_wdot<<<kVecBlocks, kVecThreads, 0, s>>>(a, b, m->mult, m->nloc, m->part, m->ticket, &m->sc->red[slot]);
  return cudaGetLastError();
}

cudaError_t launch_sub_mean(sem_mesh* m, double* x, int slot, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_sub_scalar<<<kVecBlocks, kVecThreads, 0, s>>>(x, &m->sc->red[slot], (double)m->n_unique, m->nloc);
  return cudaGetLastError();
}

cudaError_t launch_cg_start(sem_mesh* m, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_start<<<kVecBlocks, kVecThreads, 0, s>>>(m->r, m->dinv, m->mult, m->nloc, m->part, m->ticket, m->sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_pap_reduce(sem_mesh* m, cudaStream_t s) {
  // the fused operator left one partial per element in m->part + npart_off
  SEM_COUNT_LAUNCH(m);
  k_reduce_parts<<<kVecBlocks, kVecThreads, 0, s>>>(m->part + kVecBlocks * 4, m->E, m->part, m->ticket,
                                                    &m->sc->red[0], m->sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_update(sem_mesh* m, double* x, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_cg_update<<<kVecBlocks, kVecThreads, 0, s>>>(x, m->r, m->p, m->w, m->dinv, m->mult, m->nloc, m->part,
                                                 m->ticket, m->sc);
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
  k_count_nz<<<kVecBlocks, kVecThreads, 0, s>>>(a, n, m->part, m->ticket, &m->sc->red[slot]);
  return cudaGetLastError();
}

int64_t part_capacity(int64_t E) { return (int64_t)kVecBlocks * 4 + E + 64; }
int64_t pap_part_offset() { return (int64_t)kVecBlocks * 4; }

}  // namespace sem
