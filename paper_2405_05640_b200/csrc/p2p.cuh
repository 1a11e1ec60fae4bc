// NVLink peer-memory scalar allreduce, as a warp-level routine that the CG
// kernels' last block can run in place (p2p.cu: set-up and the standalone
// kernel).  See p2p.cu for the protocol.
#pragma once
#include <stdint.h>

namespace sem {

constexpr int kP2PVals = 4;  // values per call (CG: 1 or 2)

struct P2PArgs {
  uint8_t* const* peers;  // [nranks] mailbox bases (own included); nullptr: not in use
  uint8_t* local;         // own mailbox
  unsigned long long* seq;
  unsigned* err;          // sticky failure word of the communicator (sem_comm::d_err)
  int rank, nranks;
};
constexpr unsigned kP2PErrTimeout = 1u;   // a peer did not arrive within ~2 s

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Executed by one full warp (lane = threadIdx.x & 31); vals in global memory,
// n <= kP2PVals.  On return vals holds the rank-ordered sums on every rank.
// A timed-out wait sets the communicator's sticky error word and returns
// NaN (which also ends a CG solve); the host turns the word into SEM_ENCCL
// and retires the communicator (the ranks' sequence counters are no longer
// in step).
__device__ __forceinline__ void p2p_allreduce_warp(double* vals, int n, const P2PArgs& A, int lane) {
  const unsigned long long seq = *A.seq + 1;
  const int par = (int)(seq & 1);
  const size_t vbytes = (size_t)2 * A.nranks * kP2PVals * sizeof(double);
  bool ok = true;
  if (lane < A.nranks) {
    double* dst = reinterpret_cast<double*>(A.peers[lane]) + ((size_t)par * A.nranks + A.rank) * kP2PVals;
    for (int i = 0; i < n; ++i) dst[i] = vals[i];
    unsigned long long* flag = reinterpret_cast<unsigned long long*>(A.peers[lane] + vbytes) +
                               ((size_t)par * A.nranks + A.rank);
    st_release_sys(flag, seq);
    const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(A.local + vbytes) +
                                     ((size_t)par * A.nranks + lane);
    const long long t0 = clock64();
    while (ld_acquire_sys(mine) != seq)
      if (clock64() - t0 > (1ll << 32)) {  // ~2 s: record the failure instead of hanging
        ok = false;
        break;
      }
  }
  // __syncwarp orders memory among the lanes: lane 0's reads below observe
  // what every lane acquired above
  __syncwarp();
  ok = __all_sync(0xffffffffu, ok);
  if (!ok && lane == 0) atomicOr(A.err, kP2PErrTimeout);
  if (lane == 0) {
    const double* src = reinterpret_cast<const double*>(A.local) + (size_t)par * A.nranks * kP2PVals;
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int r = 0; r < A.nranks; ++r) acc += src[(size_t)r * kP2PVals + i];
      vals[i] = ok ? acc : __longlong_as_double(0x7ff8000000000000ll);
    }
    *A.seq = seq;
  }
  __syncwarp();
}

}  // namespace sem
