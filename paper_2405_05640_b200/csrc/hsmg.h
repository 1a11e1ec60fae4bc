// Hybrid-Schwarz multigrid preconditioner of the pressure solve (SURVEY 8(f)
// f2; reading R16 in DESIGN.md).  Internal.
#pragma once
#include "internal.h"

namespace sem {

constexpr int kHsmgMaxLevels = 3;

// level l: order N[l]; lev[0] is the caller's mesh when there are several
// levels (smoother and residual at the fine order); the coarsest level
// (order 1) is always an owned mesh, so its CG work arrays never alias the
// Krylov solver's
struct HsmgState {
  int nlev = 0;
  int N[kHsmgMaxLevels] = {0, 0, 0};
  sem_mesh* lev[kHsmgMaxLevels] = {nullptr, nullptr, nullptr};
  bool owned[kHsmgMaxLevels] = {false, false, false};
  double* r[kHsmgMaxLevels] = {};    // level residuals (r[0]: the caller's input)
  double* z[kHsmgMaxLevels] = {};    // level corrections (z[0]: the caller's output)
  double* t[kHsmgMaxLevels] = {};    // A_l z_l
  double* L = nullptr;               // [E][3] element lengths (R16)
  double* fdm[kHsmgMaxLevels] = {};  // per level: S [lx*lx] (S[l*lx + c]) then lam = 4 mu [lx]
  double* J[kHsmgMaxLevels] = {};    // J_l [lx_l][lx_{l+1}] (J[a*lxc + b])
  double h1c = -1.0, h2c = -1.0;     // coefficients of the coarse Jacobi inverse in lev[nlev-1]->dinv
};

// host math (hsmg_setup.cpp)
int hsmg_level_orders(int N, int* orders);  // R16: N, N/2 (if > 1), 1 -> count
bool hsmg_fdm_1d(int N, double* S, double* lam);  // S [lx*lx], lam = 4 mu [lx]
void hsmg_lagrange(int nfrom, const double* xfrom, int nto, const double* xto, double* J);  // J[a*(nfrom+1)+b]
void hsmg_interp_coords(int64_t E, int lxf, int lxc, const double* K, const double* cf, double* cc);
void hsmg_element_lengths(int64_t E, int lx, const double* coords, double* L);

// kernels (hsmg.cu)
cudaError_t launch_fdm(const sem_mesh* m, const double* r, double* z, const double* L, const double* fdm, double h1c,
                       double h2c, const int* skip, cudaStream_t s);
cudaError_t launch_restrict(const sem_mesh* mf, int lxc, const double* r, const double* w, const double* J,
                            double* rc, const int* skip, cudaStream_t s);
cudaError_t launch_prolong_add(const sem_mesh* mf, int lxc, const double* zc, const double* J, double* zf,
                               const int* skip, cudaStream_t s);

}  // namespace sem
