// Single-reduction ("pipelined") Jacobi-PCG: the Chronopoulos-Gear
// formulation of CG (PAPER.md:72 mentions Neko's
// "pipelined Krylov methods").  Same iterates as the standard PCG of
// reading R10 in exact arithmetic; per iteration ONE fused pass per element
//     u_i = dinv r_i ; p_i = u_i + beta_i p_{i-1} ; s_i = w_i + beta_i s_{i-1}
//     x += alpha_i p_i ; r_{i+1} = r_i - alpha_i s_i ; u = dinv r_{i+1}
//     w_{i+1}^e = A_e u            (then mask . dssum by the gs pipeline)
// and ONE reduction of (gamma = <r,u>, delta = <w,u>, <r,r>), with
// delta = sum_l u_l (A_e u)_l on the unassembled output (u is continuous and
// zero at masked nodes), so no separate vector pass and one allreduce.
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "device_common.cuh"

namespace sem {

__constant__ double c_Dp[kMaxN + 2][(kMaxN + 1) * (kMaxN + 1)];

cudaError_t upload_basis_p(int N, const double* D) {
  const int lx = N + 1;
  return cudaMemcpyToSymbol(c_Dp, D, sizeof(double) * lx * lx,
                            sizeof(double) * lx * (kMaxN + 1) * (kMaxN + 1));
}

struct AxPKP {
  const double* G;
  int64_t gstride;
  const double* B;
  const double* h1;
  const double* h2;
  double h1c, h2c;
  double* r;
  const double* dinv;
  const double* win;   // w_i (assembled)
  double* wout;        // w_{i+1} (local, assembled afterwards by the gs pipeline)
  double* p;
  double* s;
  double* x;
  const double* mult;
  const uint8_t* m8;
  const CGScalars* sc;
  double* part;        // [E][3] (gamma, delta, rtr) partial per element position
  const int32_t* elist;
  int64_t elem0;
  int first;           // first pass: r, x given; p = s = 0, u = dinv r (no update)
};

template <int LX>
__host__ __device__ constexpr int axp_smem_doubles() {
  return ((LX * LX * LX + 1) & ~1) * 7 + ((LX * LX + 1) & ~1) + 3 * 32 + 2;
}

template <int LX, int HM>
__global__ void __launch_bounds__(LX* LX, (LX >= 9 ? 4 : (LX == 8 ? 7 : 1))) k_ax_pcg(AxPKP P) {
  constexpr int N3 = LX * LX * LX, N3P = (N3 + 1) & ~1, NT = LX * LX;
  extern __shared__ __align__(128) double sm[];
  double* su = sm;               // u tile
  double* sg = su + N3P;         // [6][N3P] G, later q_r, q_s
  double* sD = sg + 6 * N3P;
  double* s_red = sD + ((NT + 1) & ~1);  // [3][32]
  uint64_t* bar = (uint64_t*)(s_red + 3 * 32);
  __shared__ double s_inv[256];

  if (P.sc->done) return;
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const int64_t q = P.elem0 + blockIdx.x;
  const int64_t e = P.elist ? (int64_t)P.elist[q] : q;
  const size_t eo = (size_t)e * N3;
  if (tid == 0) mbar_init(bar, 1);
  for (int t = tid; t < NT; t += NT) sD[t] = c_Dp[LX][t];
  for (int t = tid; t < 256; t += NT) s_inv[t] = t ? 1.0 / (double)t : 0.0;
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(bar, 6 * N3P * 8);
    bulk_g2s(sg, P.G + (size_t)e * P.gstride, 6 * N3P * 8, bar, policy_evict_first());
  }
  // element-wise CG-CG update, column (i,j,:) per thread, coalesced loads
  const double alpha = P.sc->alpha, beta = P.sc->beta;
  double gam = 0.0, rtr = 0.0;
  double uc[LX];
  {
    // all loads of the column first (independent, in flight together), then
    // the updates and stores
    const double* __restrict__ gr = P.r;
    const double* __restrict__ gd = P.dinv;
    const double* __restrict__ gw = P.win;
    const double* __restrict__ gp = P.p;
    const double* __restrict__ gs = P.s;
    const double* __restrict__ gx = P.x;
    double dv[LX], rv[LX], pv[LX], wv[LX], sv[LX], xv[LX];
    double mq[LX];
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const size_t o = eo + tid + NT * k;
      dv[k] = __ldg(gd + o);
      rv[k] = gr[o];
      mq[k] = P.m8 ? s_inv[P.m8[o]] : P.mult[o];
      if (!P.first) {
        pv[k] = gp[o];
        wv[k] = gw[o];
        sv[k] = gs[o];
        xv[k] = gx[o];
      }
    }
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const size_t o = eo + tid + NT * k;
      double r = rv[k];
      if (!P.first) {
        const double pn = dv[k] * r + beta * pv[k];
        const double sn = wv[k] + beta * sv[k];
        P.p[o] = pn;
        P.s[o] = sn;
        P.x[o] = xv[k] + alpha * pn;
        r = r - alpha * sn;
        P.r[o] = r;
      }
      const double u = dv[k] * r;
      gam += mq[k] * r * u;
      rtr += mq[k] * r * r;
      uc[k] = u;
      su[tid + NT * k] = u;
    }
  }
  mbar_wait(bar, 0);
  __syncthreads();

  constexpr bool kDReg = LX <= 8;
  double Dr[kDReg ? LX : 1], Ds[kDReg ? LX : 1], DTr[kDReg ? LX : 1], DTs[kDReg ? LX : 1], wc[LX];
#pragma unroll
  for (int l = 0; l < LX; ++l) {
    if constexpr (kDReg) {
      Dr[l] = sD[i * LX + l];
      Ds[l] = sD[j * LX + l];
      DTr[l] = sD[l * LX + i];
      DTs[l] = sD[l * LX + j];
    }
    wc[l] = 0.0;
  }
#define DR(l) (kDReg ? Dr[kDReg ? (l) : 0] : sD[i * LX + (l)])
#define DS(l) (kDReg ? Ds[kDReg ? (l) : 0] : sD[j * LX + (l)])
#define DTR(l) (kDReg ? DTr[kDReg ? (l) : 0] : sD[(l) * LX + i])
#define DTS(l) (kDReg ? DTs[kDReg ? (l) : 0] : sD[(l) * LX + j])
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      ur = fma(DR(l), su[l + LX * j + NT * k], ur);
      us = fma(DS(l), su[i + LX * l + NT * k], us);
      ut = fma(c_Dp[LX][k * LX + l], uc[l], ut);
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
    for (int mm = 0; mm < LX; ++mm) wc[mm] = fma(c_Dp[LX][k * LX + mm], qt, wc[mm]);
  }
  __syncthreads();
  double del = 0.0;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int p = tid + NT * k;
    double sacc = wc[k];
#pragma unroll
    for (int l = 0; l < LX; ++l) sacc = fma(DTR(l), sg[l + LX * j + NT * k], sacc);
#pragma unroll
    for (int l = 0; l < LX; ++l) sacc = fma(DTS(l), sg[N3P + i + LX * l + NT * k], sacc);
    if (HM == 0) {
      sacc *= P.h1c;
    } else if (HM == 1) {
      sacc = P.h1c * sacc + P.h2c * P.B[eo + p] * uc[k];
    } else {
      const double hm = P.h2 ? P.h2[eo + p] : P.h2c;
      if (hm != 0.0) sacc += hm * P.B[eo + p] * uc[k];
    }
    del += uc[k] * sacc;
    P.wout[eo + p] = sacc;
  }
#undef DR
#undef DS
#undef DTR
#undef DTS
  double v[3] = {gam, del, rtr};
  block_sum<3>(v, s_red);
  if (tid == 0) {
    P.part[3 * q] = v[0];
    P.part[3 * q + 1] = v[1];
    P.part[3 * q + 2] = v[2];
  }
}

template <int LX, int HM>
static cudaError_t launch_axp_t(const sem_mesh* m, const AxPKP& P, int64_t count, cudaStream_t s) {
  const size_t smem = sizeof(double) * axp_smem_doubles<LX>();
  auto kern = k_ax_pcg<LX, HM>;
  static std::atomic<bool> attr[64];  // per device
  const int dev = m->device;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!attr[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev].store(true, std::memory_order_release);
  }
  if (count <= 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  kern<<<(unsigned)count, dim3(LX, LX), smem, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_ax_pcg(const sem_mesh* m, const AxArgs& a, double* x, const double* win, double* wout,
                          int first, int64_t elem0, int64_t count, cudaStream_t s) {
  AxPKP P;
  P.G = m->G;
  P.gstride = (int64_t)6 * m->n3p;
  P.B = m->B;
  P.h1 = a.h1;
  P.h2 = a.h2;
  P.h1c = a.h1c;
  P.h2c = a.h2c;
  P.r = m->r;
  P.dinv = m->dinv;
  P.win = win;
  P.wout = wout;
  P.p = m->p;
  P.s = m->s_cg;
  P.x = x;
  P.mult = m->mult;
  P.m8 = m->m8;
  P.sc = m->sc;
  P.part = a.part;
  P.elist = m->d_elist_all;
  P.elem0 = elem0;
  P.first = first;
  const int HM = (a.h1 || a.h2) ? 2 : (a.h2c == 0.0 ? 0 : 1);
  switch (m->lx) {
#define SEM_AXP(LXV)                                                                   \
  case LXV:                                                                            \
    return HM == 0 ? launch_axp_t<LXV, 0>(m, P, count, s)                              \
                   : (HM == 1 ? launch_axp_t<LXV, 1>(m, P, count, s) : launch_axp_t<LXV, 2>(m, P, count, s));
    SEM_AXP(2) SEM_AXP(3) SEM_AXP(4) SEM_AXP(5) SEM_AXP(6) SEM_AXP(7) SEM_AXP(8) SEM_AXP(9) SEM_AXP(10)
    SEM_AXP(11) SEM_AXP(12)
#undef SEM_AXP
  }
  return cudaErrorInvalidValue;
}

// deterministic sum of the [n][3] element partials into red[0..2]
__global__ void __launch_bounds__(256) k_reduce3(const double* __restrict__ in, int64_t n, double* part,
                                                 unsigned* ticket, double* out, const CGScalars* sc) {
  __shared__ double s_red[96];
  __shared__ int s_flag;
  if (sc->done) return;
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    v[0] += in[3 * q];
    v[1] += in[3 * q + 1];
    v[2] += in[3 * q + 2];
  }
  grid_sum_last_block<3>(v, part, ticket, out, s_red, &s_flag);
}

cudaError_t launch_reduce3(sem_mesh* m, const double* in, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_reduce3<<<(unsigned)std::min<int64_t>((int64_t)m->nsm * 4, kMaxVecBlocks * 4), 256, 0, s>>>(in, m->E, m->part, m->ticket, &m->sc->red[0], m->sc);
  return cudaGetLastError();
}

// scalar step of the single-reduction CG.  red = (gamma, delta, rtr) of the
// pass that produced r_{i+1}, u_{i+1}, w_{i+1}.  phase 0: after the set-up
// pass (bn, alpha_0 = gamma/delta, beta_0 = 0); phase 1: after iteration i.
__global__ void k_pcg_scalar(CGScalars* sc, int phase) {
  const double gam = sc->red[0], del = sc->red[1], rtr = sc->red[2];
  if (phase == 0) {
    sc->bn = sqrt(rtr);
    sc->rtr = rtr;
    sc->iter = 0;
    sc->breakdown = 0;
    sc->converged = 0;
    sc->done = (sc->bn == 0.0) || (sc->maxit <= 0);
    if (sc->bn == 0.0) {
      sc->converged = 1;
      return;
    }
    if (!(del > 0.0)) {
      sc->breakdown = 1;
      sc->done = 1;
      return;
    }
    sc->rtz = gam;
    sc->beta = 0.0;
    sc->alpha = gam / del;
    return;
  }
  if (sc->done) return;
  sc->iter += 1;
  sc->rtr = rtr;
  if (sc->tol > 0.0 && sqrt(rtr) <= sc->tol * sc->bn) {
    sc->converged = 1;
    sc->done = 1;
    return;
  }
  if (sc->iter >= sc->maxit) {
    sc->done = 1;
    return;
  }
  const double beta = gam / sc->rtz;
  const double den = del - beta * gam / sc->alpha;
  if (!(den > 0.0)) {
    sc->breakdown = 1;
    sc->done = 1;
    return;
  }
  sc->beta = beta;
  sc->alpha = gam / den;
  sc->rtz = gam;
}

cudaError_t launch_pcg_scalar(sem_mesh* m, int phase, cudaStream_t s) {
  SEM_COUNT_LAUNCH(m);
  k_pcg_scalar<<<1, 1, 0, s>>>(m->sc, phase);
  return cudaGetLastError();
}

}  // namespace sem
