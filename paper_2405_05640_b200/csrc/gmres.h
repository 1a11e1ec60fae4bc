// Restarted GMRES state (gmres.cu kernels, api.cpp driver).  Internal.
#pragma once
#include <vector>

#include "internal.h"

namespace sem {

constexpr int kGmMaxRestart = 30;      // restart length m <= 30 (basis of m + 1 vectors)
constexpr int64_t kGmMaxBlocks = 1024; // reduction partials per pass

// device-resident scalars of one solve
struct GmScalars {
  double H[(kGmMaxRestart + 1) * kGmMaxRestart];  // H[i * restart + j]
  double cs[kGmMaxRestart], sn[kGmMaxRestart], g[kGmMaxRestart + 1], y[kGmMaxRestart];
  double h[kGmMaxRestart + 1], h2[kGmMaxRestart + 1];
  double nn, sigma, bn, beta, tol;
  int j, k, it, maxit, restart, done, converged, cycle_stop, breakdown;
};

struct GmState {
  int restart = 0;
  int64_t ld = 0;            // basis stride: nloc rounded up to 32 (16-byte aligned bulk copies)
  double* V = nullptr;       // [restart + 1][ld] Krylov basis
  double* z = nullptr;       // [nloc] dinv v_j (operator input)
  double* Z = nullptr;       // [restart][nloc] M v_j of the flexible variant (SEM_PC_HSMG)
  double* b = nullptr;       // [nloc] masked (and projected) right-hand side
  double* part = nullptr;    // [kGmMaxBlocks][33] reduction partials
  unsigned* ticket = nullptr;
  double* red = nullptr;     // [33] update-pass sums (h2, nn)
  GmScalars* gs = nullptr;   // device
  GmScalars* gs_host = nullptr;  // pinned
  // one CUDA graph per Arnoldi step j (its kernels depend on j only), captured
  // on first use and replayed by every later cycle and solve with the same key
  std::vector<cudaGraphExec_t> exec;
  double key_h1c = 0.0, key_h2c = 0.0;
  const void* key_h1 = nullptr;
  const void* key_h2 = nullptr;
  int key_flex = -1, key_coarse = 0;
  // early end of a cycle: the host reads step j-1's cycle_stop (pinned copy,
  // event) while step j runs, so at most one no-op step follows the stop
  int* stop_host = nullptr;  // pinned [2]
  cudaEvent_t ev_stop[2] = {nullptr, nullptr};
  void drop_graphs() {
    for (cudaGraphExec_t& e : exec)
      if (e) cudaGraphExecDestroy(e);
    exec.clear();
  }
};

cudaError_t gm_launch_dots(sem_mesh* m, GmState* G, int nvec, cudaStream_t s);
cudaError_t gm_launch_update(sem_mesh* m, GmState* G, int nvec, cudaStream_t s);
cudaError_t gm_launch_unpack(sem_mesh* m, GmState* G, int nvec, cudaStream_t s);
cudaError_t gm_launch_givens(sem_mesh* m, GmState* G, cudaStream_t s);
cudaError_t gm_launch_next(sem_mesh* m, GmState* G, int j, bool flex, cudaStream_t s);
cudaError_t gm_launch_cycle_end(sem_mesh* m, GmState* G, double* x, bool flex, cudaStream_t s);
cudaError_t gm_launch_resid(sem_mesh* m, GmState* G, const double* b, cudaStream_t s);
cudaError_t gm_launch_start(sem_mesh* m, GmState* G, int first, bool flex, cudaStream_t s);

}  // namespace sem
