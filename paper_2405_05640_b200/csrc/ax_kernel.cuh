// Operator kernel templates (reading R5, CG fusion R10), included by
// ax_lx.cu, which is compiled once per order
// (-DSEM_AX_LX=lx) so the orders build in parallel; ax.cu dispatches.
#pragma once
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "ax.cuh"

namespace sem {

// per translation unit (one order each): uploaded by ax_upload_basis_lx<LX>
static __constant__ double c_D[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];  // c_D[lx][i*lx+l] = D_il
static __constant__ double c_W[kMaxN + 2][kMaxN + 1];                    // GLL weights per lx
// the same D in global memory: the per-CTA copy into shared memory reads it
// with a thread-dependent index, which the constant cache would serialise
static __device__ double g_D[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];

// Affine elements (opt-in SEM_AFFINE=1): the Jacobian is
// constant over the element, so G_ab(node) = C_ab * w_i w_j w_k with six
// constants per element.  One warp per element checks that every node's
// G_ab / (w_i w_j w_k) equals node 0's to 1e-12 relative (else *nonaffine)
// and stores C_ab = node 0's ratio.
template <int LX>
__global__ void __launch_bounds__(32) k_affine_detect(const double* __restrict__ G, int64_t gstride, int n3p,
                                                      double* __restrict__ C, int* nonaffine) {
  constexpr int N3 = LX * LX * LX;
  const int64_t e = blockIdx.x;
  const double* g = G + e * gstride;
  const double w0 = c_W[LX][0] * c_W[LX][0] * c_W[LX][0];
  double ref[6];
  for (int c = 0; c < 6; ++c) ref[c] = g[(size_t)c * n3p] / w0;
  const double scale = fabs(ref[0]) + fabs(ref[1]) + fabs(ref[2]);
  bool ok = true;
  for (int p = threadIdx.x; p < N3; p += 32) {
    const int i = p % LX, j = (p / LX) % LX, k = p / (LX * LX);
    const double W = c_W[LX][i] * c_W[LX][j] * c_W[LX][k];
    for (int c = 0; c < 6; ++c) ok = ok && fabs(g[(size_t)c * n3p + p] / W - ref[c]) <= 1e-12 * scale;
  }
  if (!__all_sync(0xffffffffu, ok) && threadIdx.x == 0) atomicOr(nonaffine, 1);
  if (threadIdx.x < 6) C[e * 6 + threadIdx.x] = ref[threadIdx.x];
}

// ---------------------------------------------------------------------------
// Local operator A_e u (reading R5).  One CTA of lx*lx threads per element;
// thread (i,j) owns the column (i,j,:) in registers, so the t-direction
// contractions never touch shared memory, while the r/s contractions read
// the element's u tile in shared memory.  The element's 6 geometric factors
// and its operand arrays arrive by cp.async.bulk (TMA engine) into shared
// memory with an mbarrier complete_tx, with an L2 evict_first policy (they
// stream once); w leaves with plain coalesced stores (it stays in L2 for the
// gather-scatter pass that follows on the gs stream).
//   HM = 0: h1 = h1c constant, h2 = 0 (Poisson when h1c = 1)
//   HM = 1: h1c, h2c constants
//   HM = 2: h1/h2 arrays (NULL array -> its constant)
//   CG:     u := p = dinv r + beta p (written back), pAp = sum_l p_l (A_e p)_l
//           per element (reading R10's unassembled identity)
// Elements: position q in [elem0, elem0 + gridDim.x) of the processing order
// (elist, or identity).
// ---------------------------------------------------------------------------


// CG operands (r, dinv, p) are read straight into registers (each thread its
// column, coalesced) while the TMA brings G: the shared-memory footprint stays
// that of the plain operator (7 CTAs per SM at lx = 8)
constexpr bool kCGRegOperands = true;
// L2 eviction hints on the operand loads / stores (see k_ax)
#ifndef SEM_L2_HINTS
#define SEM_L2_HINTS 1
#endif
constexpr bool kL2Hints = SEM_L2_HINTS;

// tile doubles: u (CG: p; + r, dinv without register operands), G x 6 (AFF:
// 2 work slots), D, the reduction scratch, the mbarrier
// constant-coefficient Helmholtz at lx >= SEM_BSMEM_LX (even n3): the mass
// diagonal B rides in the TMA with u and G instead of per-column loads
#ifndef SEM_PDL_LATE
#define SEM_PDL_LATE 1
#endif
#ifndef SEM_AX_SMALL
#define SEM_AX_SMALL 1  // lx <= 4: several elements per CTA (k_ax_small)
#endif
#ifndef SEM_BSMEM_LX
#define SEM_BSMEM_LX 10
#endif
template <int LX, int HM, bool AFF>
__host__ __device__ constexpr bool ax_b_smem() {
  return HM == 1 && !AFF && LX >= SEM_BSMEM_LX && (LX * LX * LX) % 2 == 0;
}
template <int LX, bool CG, bool AFF = false, int HM = 0>
__host__ __device__ constexpr int ax_smem_doubles() {
  return ((LX * LX * LX + 1) & ~1) * ((CG && !kCGRegOperands ? 3 : 1) + (AFF ? 2 : 6) + (ax_b_smem<LX, HM, AFF>() ? 1 : 0)) +
         ((LX * LX + 1) & ~1) + 32 /*red*/ + 2 /*bar*/;
}

// experiment switches (build flags; defaults = the measured best)
#ifndef SEM_MINB_LX10
#define SEM_MINB_LX10 3
#endif
#ifndef SEM_DREG_MAX_LX
#define SEM_DREG_MAX_LX 10
#endif
// resident CTAs per SM the register allocation is capped for (measured per
// order and mode; the CG variant holds its operand columns as well)
template <int LX, bool CG>
__host__ __device__ constexpr int ax_min_blocks() {
  // lx >= 10: 3 CTAs/SM without spills measured 9 % faster on c5 than 4
  // CTAs/SM at 128 registers with spills
  if (LX == 10) return SEM_MINB_LX10;
  if (CG) return LX >= 10 ? 3 : (LX == 9 ? 4 : (LX == 8 ? 7 : (LX == 6 ? 12 : 1)));
  return LX >= 10 ? 3 : (LX == 9 ? 5 : (LX == 8 ? 7 : (LX == 7 ? 10 : (LX == 6 ? 12 : 16))));
}

template <int LX, int HM, bool CG, bool AFF>
__global__ void __launch_bounds__(LX* LX, ax_min_blocks<LX, CG>()) k_ax(AxKP P) {
  constexpr int N3 = LX * LX * LX, N3P = (N3 + 1) & ~1, NT = LX * LX;
  constexpr int NU = (CG && !kCGRegOperands) ? 3 : 1;
  extern __shared__ __align__(128) double sm[];
  double* su = sm;                   // [N3P] u (CG: p)
  double* sr = sm + N3P;             // CG: [N3P] r, [N3P] dinv
  double* sg = sm + NU * N3P;        // [6][N3P] G (AFF: [2]), later q_r (slot 0), q_s (slot 1)
  constexpr bool BSM = ax_b_smem<LX, HM, AFF>();
  double* sB = sg + (AFF ? 2 : 6) * N3P;  // BSM: [N3P] B
  double* sD = sB + (BSM ? N3P : 0);      // [LX*LX]
  double* s_red = sD + ((NT + 1) & ~1);  // [32]
  uint64_t* bar = (uint64_t*)(s_red + 32);

  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t q = P.elem0 + blockIdx.x;
  const int64_t e = P.elist ? (int64_t)P.elist[q] : q;
  const size_t eo = (size_t)e * N3;
  const bool bulk_ops = P.bulk && !(CG && kCGRegOperands);
  const bool use_bar = !AFF || bulk_ops;
  if (!P.pdl && ((CG && P.sc->done) || (P.skip && *P.skip))) return;  // uniform over the launch
  if (tid == 0) {
    mbar_init(bar, 1);
    // G does not depend on the kernel before: its TMA goes out first (bytes
    // expected without arriving), so with programmatic dependent launch
    // (P.pdl) the first wave's factors stream in while the previous kernel
    // drains; the single arrival comes with the operand copies below
    if (use_bar && !AFF) {
      mbar_expect_tx_only(bar, 6 * N3P * 8 + (BSM ? N3 * 8 : 0));
      bulk_g2s(sg, P.G + (size_t)e * P.gstride, 6 * N3P * 8, bar, policy_evict_first());
      if (BSM) bulk_g2s(sB, P.B + eo, N3 * 8, bar, policy_evict_first());
    }
  }
  if (P.pdl) {
    griddep_wait();  // the previous kernel's results are visible from here on
    if ((CG && P.sc->done) || (P.skip && *P.skip)) {  // uniform over the launch
      if (use_bar) {  // no CTA exits with a copy into its shared memory in flight
        __syncthreads();
        if (tid == 0) mbar_arrive(bar);
        mbar_wait(bar, 0);
      }
      return;
    }
    if (!SEM_PDL_LATE) griddep_launch_dependents();
  }
  for (int t = tid; t < NT; t += NT) sD[t] = __ldg(&g_D[LX][t]);
  __syncthreads();
  if (tid == 0 && use_bar) {
    if (bulk_ops) {
      const uint64_t pol = policy_evict_first();
      mbar_expect_tx(bar, NU * N3 * 8);  // arrives
      if (CG) {
        bulk_g2s(su, P.p + eo, N3 * 8, bar, pol);
        bulk_g2s(sr, P.r + eo, N3 * 8, bar, pol);
        bulk_g2s(sr + N3P, P.dinv + eo, N3 * 8, bar, pol);
      } else {
        bulk_g2s(su, P.u + eo, N3 * 8, bar, pol);
      }
    } else {
      mbar_arrive(bar);
    }
  }
  // L2 priorities: the streamed operands go first, w stays (the gather-
  // scatter of this chunk reads it back while the next chunk streams)
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_w = kL2Hints ? policy_evict_last() : pol_first;
  double pcol[CG && kCGRegOperands ? LX : 1];
  if (CG && kCGRegOperands) {  // p <- dinv r + beta p, column by column, from registers
    const double beta = P.sc->beta;
    double rv[LX], dv[LX], pv[LX], xv[LX];
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const size_t o = eo + tid + NT * k;
      if (kL2Hints) {
        rv[k] = ld_hint(P.r + o, pol_first);
        dv[k] = ld_hint(P.dinv + o, pol_first);
        pv[k] = ld_hint_rw(P.p + o, pol_first);
      } else {
        rv[k] = __ldg(P.r + o);
        dv[k] = __ldg(P.dinv + o);
        pv[k] = P.p[o];
      }
      if (P.x) xv[k] = kL2Hints ? ld_hint_rw(P.x + o, pol_first) : P.x[o];
    }
    if (P.x) {  // x += alpha_{i-1} p_{i-1}: the previous iteration's update, deferred
      const double xa = P.sc->xalpha;
#pragma unroll
      for (int k = 0; k < LX; ++k) {
        const size_t o = eo + tid + NT * k;
        if (kL2Hints) st_hint(P.x + o, xv[k] + xa * pv[k], pol_first);
        else P.x[o] = xv[k] + xa * pv[k];
      }
    }
#pragma unroll
    for (int k = 0; k < LX; ++k) pcol[CG && kCGRegOperands ? k : 0] = dv[k] * rv[k] + beta * pv[k];
  } else if (!P.bulk) {
    for (int t = tid; t < N3; t += NT) {
      if (CG) {
        su[t] = P.p[eo + t];
        sr[t] = P.r[eo + t];
        sr[N3P + t] = P.dinv[eo + t];
      } else {
        su[t] = P.u[eo + t];
      }
    }
  }
  if (use_bar) mbar_wait(bar, 0);
  if (CG && kCGRegOperands) {
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const int p = tid + NT * k;
      su[p] = pcol[CG && kCGRegOperands ? k : 0];
      if (kL2Hints) st_hint(P.p + eo + p, pcol[CG && kCGRegOperands ? k : 0], pol_first);
      else P.p[eo + p] = pcol[CG && kCGRegOperands ? k : 0];
    }
  } else if (CG) {  // p <- dinv r + beta p, column by column
    const double beta = P.sc->beta;
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const int p = tid + NT * k;
      const double pn = sr[N3P + p] * sr[p] + beta * su[p];
      su[p] = pn;
      P.p[eo + p] = pn;
    }
  }
  __syncthreads();

  // lx <= 10: the thread's two rows of D (gradient phase), then its two
  // columns (divergence phase) live in registers -- two lx-vectors at a time,
  // so the contractions issue one shared-memory load per FMA (the u / q
  // tile); lx >= 11 reads D from shared memory (register budget)
  constexpr bool kDReg = LX <= SEM_DREG_MAX_LX;
  constexpr int DN = kDReg ? LX : 1;
  double Da[DN], Db[DN], uc[LX], wc[LX];
#pragma unroll
  for (int l = 0; l < LX; ++l) {
    if constexpr (kDReg) {
      Da[kDReg ? l : 0] = sD[i * LX + l];
      Db[kDReg ? l : 0] = sD[j * LX + l];
    }
    uc[l] = su[tid + NT * l];
    wc[l] = 0.0;
  }
  double ca[AFF ? 6 : 1], wij = 0.0;
  if constexpr (AFF) {
#pragma unroll
    for (int c = 0; c < 6; ++c) ca[AFF ? c : 0] = __ldg(P.gaff + e * 6 + c);
    wij = c_W[LX][i] * c_W[LX][j];
  }
#define DA1(l) (kDReg ? Da[kDReg ? (l) : 0] : sD[i * LX + (l)])
#define DB1(l) (kDReg ? Db[kDReg ? (l) : 0] : sD[j * LX + (l)])
#define DA2(l) (kDReg ? Da[kDReg ? (l) : 0] : sD[(l) * LX + i])
#define DB2(l) (kDReg ? Db[kDReg ? (l) : 0] : sD[(l) * LX + j])
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double ur = 0.0, us = 0.0, ut = 0.0;
    // even lx: the r-direction row u(:, j, k) is contiguous -> 16-byte shared
    // loads (half the load instructions for that contraction; same order)
    if constexpr (LX % 2 == 0) {
#pragma unroll
      for (int l = 0; l < LX; l += 2) {
        const double2 v = *reinterpret_cast<const double2*>(su + l + LX * j + NT * k);
        ur = fma(DA1(l), v.x, ur);
        ur = fma(DA1(l + 1), v.y, ur);
      }
    } else {
#pragma unroll
      for (int l = 0; l < LX; ++l) ur = fma(DA1(l), su[l + LX * j + NT * k], ur);
    }
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      us = fma(DB1(l), su[i + LX * l + NT * k], us);
      ut = fma(c_D[LX][k * LX + l], uc[l], ut);
    }
    double g11, g22, g33, g12, g13, g23;
    if constexpr (AFF) {
      const double W = wij * c_W[LX][k];
      g11 = ca[0] * W;
      g22 = ca[1] * W;
      g33 = ca[2] * W;
      g12 = ca[3] * W;
      g13 = ca[4] * W;
      g23 = ca[5] * W;
    } else {
      g11 = sg[p];
      g22 = sg[N3P + p];
      g33 = sg[2 * N3P + p];
      g12 = sg[3 * N3P + p];
      g13 = sg[4 * N3P + p];
      g23 = sg[5 * N3P + p];
    }
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
  // constant-coefficient Helmholtz: the column's B values are requested
  // before the barrier, so their latency hides behind it and the D reloads
  double bcol[HM == 1 ? LX : 1];
  if constexpr (HM == 1 && !BSM) {
#pragma unroll
    for (int k = 0; k < LX; ++k) bcol[HM == 1 ? k : 0] = __ldg(P.B + eo + tid + NT * k);
  }
  __syncthreads();
  if constexpr (kDReg) {
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      Da[kDReg ? l : 0] = sD[l * LX + i];
      Db[kDReg ? l : 0] = sD[l * LX + j];
    }
  }
  double pap = 0.0;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double s = wc[k];
    if constexpr (LX % 2 == 0) {
#pragma unroll
      for (int l = 0; l < LX; l += 2) {
        const double2 v = *reinterpret_cast<const double2*>(sg + l + LX * j + NT * k);
        s = fma(DA2(l), v.x, s);
        s = fma(DA2(l + 1), v.y, s);
      }
    } else {
#pragma unroll
      for (int l = 0; l < LX; ++l) s = fma(DA2(l), sg[l + LX * j + NT * k], s);
    }
#pragma unroll
    for (int l = 0; l < LX; ++l) s = fma(DB2(l), sg[N3P + i + LX * l + NT * k], s);
    // the column of u again from the tile (its registers are free by now)
    const double uk = su[p];
    if (HM == 0) {
      s *= P.h1c;
    } else if (HM == 1) {
      s = P.h1c * s + P.h2c * (BSM ? sB[p] : bcol[HM == 1 ? k : 0]) * uk;
    } else {
      const double hm = P.h2 ? P.h2[eo + p] : P.h2c;
      if (hm != 0.0) s += hm * P.B[eo + p] * uk;
    }
    if (CG) pap += uk * s;
    // the CG operator's output in the x-planes-last layout when P.xl
    const size_t ow = eo + ((CG && P.xl) ? xlast_pos<LX>(p) : p);
    if (kL2Hints) st_hint(P.w + ow, s, pol_w);
    else P.w[ow] = s;
  }
#undef DA1
#undef DB1
#undef DA2
#undef DB2
  if (P.pdl && SEM_PDL_LATE) griddep_launch_dependents();
  if (CG) {
    double v[1] = {pap};
    block_sum<1>(v, s_red);
    if (tid == 0) P.part[q] = v[0];
  }
}

constexpr int kMaxDevices = 64;


// Low orders (lx <= 4: the multigrid's coarse levels).  One CTA of lx^2
// threads per element leaves the SM's block slots full of 4- or 16-thread
// CTAs (launch- and latency-bound); here a CTA of 128 threads takes
// 128 / lx^2 elements, thread (i, j) of element le owning its column as in
// k_ax; operands straight from global memory (no TMA at 64-512 B per
// element).  Same arithmetic (reading R5; CG: R10's fused prologue and the
// element's pAp partial, summed in a fixed order).
template <int LX>
struct AxSmall {
  static constexpr int NT = LX * LX, N3 = LX * LX * LX, EPB = 128 / NT, THREADS = EPB * NT;
};
template <int LX, int HM, bool CG>
__global__ void __launch_bounds__(128) k_ax_small(AxKP P) {
  using S = AxSmall<LX>;
  constexpr int NT = S::NT, N3 = S::N3, EPB = S::EPB;
  __shared__ double su[EPB][N3], sqr[EPB][N3], sqs[EPB][N3];
  __shared__ double sD[NT], s_p[S::THREADS];
  if ((CG && P.sc->done) || (P.skip && *P.skip)) return;  // uniform over the launch
  const int t = threadIdx.x, le = t / NT, tid = t - le * NT, i = tid % LX, j = tid / LX;
  if (t < NT) sD[t] = __ldg(&g_D[LX][t]);
  const int64_t ql = (int64_t)blockIdx.x * EPB + le;
  const bool live = le < EPB && ql < P.npos;
  const int64_t q = P.elem0 + ql;
  const int64_t e = live ? (P.elist ? (int64_t)P.elist[q] : q) : 0;
  const size_t eo = (size_t)e * N3;
  double uc[LX], g[6][LX];
  if (live) {
    const double beta = CG ? P.sc->beta : 0.0, xa = CG ? P.sc->xalpha : 0.0;
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const int p = tid + NT * k;
      double v;
      if (CG) {
        const double pv = P.p[eo + p];
        if (P.x) P.x[eo + p] += xa * pv;
        v = __ldg(P.dinv + eo + p) * __ldg(P.r + eo + p) + beta * pv;
        P.p[eo + p] = v;
      } else {
        v = __ldg(P.u + eo + p);
      }
      uc[k] = v;
      su[le][p] = v;
#pragma unroll
      for (int c = 0; c < 6; ++c) g[c][k] = __ldg(P.G + (size_t)e * P.gstride + (size_t)c * ((N3 + 1) & ~1) + p);
    }
  }
  __syncthreads();
  double wc[LX];
#pragma unroll
  for (int k = 0; k < LX; ++k) wc[k] = 0.0;
  if (live) {
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const int p = tid + NT * k;
      double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        ur = fma(sD[i * LX + l], su[le][l + LX * j + NT * k], ur);
        us = fma(sD[j * LX + l], su[le][i + LX * l + NT * k], us);
        ut = fma(c_D[LX][k * LX + l], uc[l], ut);
      }
      double qr = g[0][k] * ur + g[3][k] * us + g[4][k] * ut;
      double qs = g[3][k] * ur + g[1][k] * us + g[5][k] * ut;
      double qt = g[4][k] * ur + g[5][k] * us + g[2][k] * ut;
      if (HM == 2) {
        const double h = P.h1 ? P.h1[eo + p] : P.h1c;
        qr *= h;
        qs *= h;
        qt *= h;
      }
      sqr[le][p] = qr;
      sqs[le][p] = qs;
#pragma unroll
      for (int mm = 0; mm < LX; ++mm) wc[mm] = fma(c_D[LX][k * LX + mm], qt, wc[mm]);
    }
  }
  __syncthreads();
  double pap = 0.0;
  if (live) {
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const int p = tid + NT * k;
      double s = wc[k];
#pragma unroll
      for (int l = 0; l < LX; ++l) s = fma(sD[l * LX + i], sqr[le][l + LX * j + NT * k], s);
#pragma unroll
      for (int l = 0; l < LX; ++l) s = fma(sD[l * LX + j], sqs[le][i + LX * l + NT * k], s);
      const double uk = uc[k];
      if (HM == 0) {
        s *= P.h1c;
      } else if (HM == 1) {
        s = P.h1c * s + P.h2c * __ldg(P.B + eo + p) * uk;
      } else {
        const double hm = P.h2 ? P.h2[eo + p] : P.h2c;
        if (hm != 0.0) s += hm * P.B[eo + p] * uk;
      }
      if (CG) pap += uk * s;
      P.w[eo + ((CG && P.xl) ? xlast_pos<LX>(p) : p)] = s;
    }
  }
  if (CG) {  // the element's pAp partial, its threads summed in order
    if (t < S::THREADS) s_p[t] = pap;
    __syncthreads();
    if (live && tid == 0) {
      double a = 0.0;
      for (int r = 0; r < NT; ++r) a += s_p[le * NT + r];
      P.part[q] = a;
    }
  }
}

template <int LX, int HM, bool CG, bool AFF>
static cudaError_t launch_ax_t(const sem_mesh* m, const AxKP& P, int64_t count, cudaStream_t s) {
  const size_t smem = sizeof(double) * ax_smem_doubles<LX, CG, AFF, HM>();
  auto kern = k_ax<LX, HM, CG, AFF>;
  // the dynamic shared memory attribute is per device (set once each)
  static std::atomic<bool> attr_set[kMaxDevices];
  const int dev = m->device;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true, std::memory_order_release);
  }
  if (count <= 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  if constexpr (LX <= 4 && !AFF) {  // several elements per CTA (k_ax_small)
    if (SEM_AX_SMALL) {
      AxKP Q = P;
      Q.npos = count;
      const unsigned grid = (unsigned)((count + AxSmall<LX>::EPB - 1) / AxSmall<LX>::EPB);
      k_ax_small<LX, HM, CG><<<grid, 128, 0, s>>>(Q);
      return cudaGetLastError();
    }
  }
  if (!P.pdl) {
    kern<<<(unsigned)count, dim3(LX, LX), smem, s>>>(P);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)count);
  cfg.blockDim = dim3(LX, LX);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, P);
}

template <int LX, bool AFF>
static cudaError_t launch_ax_lx2(const sem_mesh* m, const AxKP& P, int HM, bool cg, int64_t count,
                                cudaStream_t s) {
  if (cg) {
    switch (HM) {
      case 0: return launch_ax_t<LX, 0, true, AFF>(m, P, count, s);
      case 1: return launch_ax_t<LX, 1, true, AFF>(m, P, count, s);
      default: return launch_ax_t<LX, 2, true, AFF>(m, P, count, s);
    }
  }
  switch (HM) {
    case 0: return launch_ax_t<LX, 0, false, AFF>(m, P, count, s);
    case 1: return launch_ax_t<LX, 1, false, AFF>(m, P, count, s);
    default: return launch_ax_t<LX, 2, false, AFF>(m, P, count, s);
  }
}



// ---- the per-order entry points (explicitly instantiated in ax_lx.cu) -----
template <int LX>
cudaError_t ax_upload_basis_lx(const double* D, const double* w) {
  cudaError_t e = cudaMemcpyToSymbol(c_D, D, sizeof(double) * LX * LX,
                                     sizeof(double) * LX * (kMaxN + 1) * (kMaxN + 1));
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(g_D, D, sizeof(double) * LX * LX, sizeof(double) * LX * (kMaxN + 1) * (kMaxN + 1));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_W, w, sizeof(double) * LX, sizeof(double) * LX * (kMaxN + 1));
}

template <int LX>
cudaError_t ax_launch_lx(const sem_mesh* m, const AxKP& P, int HM, bool cg, int64_t count, cudaStream_t s) {
  return P.gaff ? launch_ax_lx2<LX, true>(m, P, HM, cg, count, s) : launch_ax_lx2<LX, false>(m, P, HM, cg, count, s);
}

template <int LX>
cudaError_t ax_affine_detect_lx(const sem_mesh* m, double* C, int* nonaffine, cudaStream_t s) {
  k_affine_detect<LX><<<(unsigned)m->E, 32, 0, s>>>(m->G, (int64_t)6 * m->n3p, m->n3p, C, nonaffine);
  return cudaGetLastError();
}

template <int LX>
int ax_occupancy_lx() {
  int b = 0;
  const size_t smem = sizeof(double) * ax_smem_doubles<LX, true, false>();
  cudaFuncSetAttribute(k_ax<LX, 0, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_ax<LX, 0, true, false>, LX * LX, smem) != cudaSuccess)
    b = ax_min_blocks<LX, true>();
  cudaGetLastError();
  return b;
}

}  // namespace sem
