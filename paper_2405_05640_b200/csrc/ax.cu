// Dispatch of the operator kernel (ax_kernel.cuh, one translation unit per
// order: ax_lx.cu compiled with -DSEM_AX_LX=lx): basis upload, launch
// parameters, affine detection, occupancy.  See DESIGN.md section 4 (the
// operator kernel, its CG fusion and the element layout of its output).
#include <stdint.h>

#include <algorithm>

#include "ax.cuh"

namespace sem {

cudaError_t upload_basis_ax(int N, const double* D, const double* w) {
  cudaError_t e = cudaErrorInvalidValue;
  SEM_LX_DISPATCH_INT(N + 1, e, ax_upload_basis_lx<LX>(D, w));
  return e;
}

cudaError_t launch_affine_detect(const sem_mesh* m, double* C, int* nonaffine, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  cudaError_t e = cudaErrorInvalidValue;
  SEM_LX_DISPATCH_INT(m->lx, e, ax_affine_detect_lx<LX>(m, C, nonaffine, s));
  return e;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

cudaError_t launch_ax_range(const sem_mesh* m, const AxArgs& a, bool cg, int64_t elem0, int64_t count,
                            cudaStream_t s) {
  AxKP P;
  P.skip = a.skip;
  P.pdl = a.pdl ? 1 : 0;
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
  P.elist = m->d_elist_all;
  P.elem0 = elem0;
  P.x = cg ? a.x : nullptr;
  P.gaff = m->affine ? m->d_gaff : nullptr;
  P.xl = (cg && m->xl_active) ? 1 : 0;
  if (cg)
    P.bulk = (m->n3 % 2 == 0) && aligned16(a.r) && aligned16(a.dinv) && aligned16(a.p);
  else
    P.bulk = (m->n3 % 2 == 0) && aligned16(a.u);
  int HM = 2;
  if (!a.h1 && !a.h2) HM = (a.h2c == 0.0) ? 0 : 1;
  if (cudaSetDevice(m->device) != cudaSuccess) return cudaErrorInvalidDevice;
  cudaError_t e = cudaErrorInvalidValue;
  SEM_LX_DISPATCH_INT(m->lx, e, ax_launch_lx<LX>(m, P, HM, cg, count, s));
  return e;
}

int ax_ctas_per_sm(const sem_mesh* m) {
  int n = 0;
  SEM_LX_DISPATCH_INT(m->lx, n, ax_occupancy_lx<LX>());
  return n > 0 ? n : 1;
}

}  // namespace sem
