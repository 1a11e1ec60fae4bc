// Operator launch parameters (ax.cu dispatch, ax_kernel.cuh kernels).
#pragma once
#include <stdint.h>

#include "device_common.cuh"

namespace sem {

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
  int64_t elem0;
  int bulk;  // operand element blocks are 16-byte aligned -> TMA bulk copy
  double* x;  // CG: x += sc->xalpha p_old (deferred update of the previous iteration)
  const double* gaff;  // AFF: [E][6] per-element constants C_ab (G_ab = C_ab w_i w_j w_k)
  const int* skip;     // != nullptr and *skip: the launch does nothing (GMRES cycle end)
  int pdl;             // launched as a programmatic dependent of the previous kernel
  int xl;              // CG: w in the x-planes-last element layout
  int64_t npos;        // k_ax_small: positions in this launch
};

template <int LX>
cudaError_t ax_upload_basis_lx(const double* D, const double* w);
template <int LX>
cudaError_t ax_launch_lx(const sem_mesh* m, const AxKP& P, int HM, bool cg, int64_t count, cudaStream_t s);
template <int LX>
cudaError_t ax_affine_detect_lx(const sem_mesh* m, double* C, int* nonaffine, cudaStream_t s);
template <int LX>
int ax_occupancy_lx();

}  // namespace sem
