// CG scalar allreduce over NVLink peer memory (reading R10 across ranks: the
// dot products of PAPER.md's CG are global sums).  Each rank owns a small
// mailbox in device memory, mapped into every peer with CUDA IPC.  One warp
// per call: lane p stores this rank's values into slot [parity][rank] of
// peer p's mailbox, then (release) the slot's sequence flag; it then waits
// (acquire) for every peer's flag in the local mailbox and lane 0 sums the
// slots in ASCENDING RANK ORDER -- every rank computes bit-identical sums.
// Mailboxes alternate by call parity: a rank can only reuse a parity after
// every peer finished reading it (the next call needs all their flags).
// A bounded spin (~2 s) turns a lost peer into NaN results (CG breakdown)
// instead of a hang.  Replaces a 1-2 value ncclAllReduce (~10-20 us in a
// graph) with one ~2-4 us kernel; NCCL stays the fallback.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "device_common.cuh"

namespace sem {

constexpr int kP2PVals = 4;  // values per call (CG: 1 or 2)

struct P2PArgs {
  uint8_t* const* peers;  // [nranks] mailbox bases (own included)
  uint8_t* local;         // own mailbox
  unsigned long long* seq;
  int rank, nranks;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(32) k_p2p_allreduce(double* vals, int n, P2PArgs A) {
  const int lane = threadIdx.x;
  const unsigned long long seq = *A.seq + 1;
  const int par = (int)(seq & 1);
  const size_t vbytes = (size_t)2 * A.nranks * kP2PVals * sizeof(double);
  if (lane < A.nranks) {
    double* dst = reinterpret_cast<double*>(A.peers[lane]) + ((size_t)par * A.nranks + A.rank) * kP2PVals;
    for (int i = 0; i < n; ++i) dst[i] = vals[i];
    unsigned long long* flag = reinterpret_cast<unsigned long long*>(A.peers[lane] + vbytes) +
                               ((size_t)par * A.nranks + A.rank);
    st_release_sys(flag, seq);
    const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(A.local + vbytes) +
                                     ((size_t)par * A.nranks + lane);
    const long long t0 = clock64();
    bool ok = true;
    while (ld_acquire_sys(mine) != seq)
      if (clock64() - t0 > (1ll << 32)) {
        ok = false;
        break;
      }
    if (!ok) vals[0] = __longlong_as_double(0x7ff8000000000000ll);  // NaN: CG breakdown, no hang
  }
  __syncwarp();
  if (lane == 0) {
    if (vals[0] == vals[0]) {
      const double* src = reinterpret_cast<const double*>(A.local) + (size_t)par * A.nranks * kP2PVals;
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int r = 0; r < A.nranks; ++r) acc += src[(size_t)r * kP2PVals + i];
        vals[i] = acc;
      }
    } else {
      for (int i = 0; i < n; ++i) vals[i] = __longlong_as_double(0x7ff8000000000000ll);
    }
    *A.seq = seq;
  }
}

#ifdef SEM_WITH_NCCL
// Collective (every rank calls it): allocate and zero the mailbox, exchange
// IPC handles (ncclAllGather), open the peers' mailboxes.  Leaves c->p2p
// false (NCCL allreduce) if any step fails or SEM_P2P=0.
void p2p_setup(sem_comm* c) {
  c->p2p = false;
  const char* env = getenv("SEM_P2P");
  const bool want = !(env && atoi(env) == 0);
  const int R = c->nranks;
  const size_t bytes = (size_t)2 * R * kP2PVals * sizeof(double) + (size_t)2 * R * sizeof(unsigned long long);
  bool ok = want && R > 1 && R <= 32;
  cudaIpcMemHandle_t h{};
  if (ok) ok = cudaMalloc((void**)&c->p2p_local, bytes) == cudaSuccess;
  if (ok) ok = cudaMemset(c->p2p_local, 0, bytes) == cudaSuccess;
  if (ok) ok = cudaMalloc((void**)&c->p2p_seq, sizeof(unsigned long long)) == cudaSuccess;
  if (ok) ok = cudaMemset(c->p2p_seq, 0, sizeof(unsigned long long)) == cudaSuccess;
  if (ok) ok = cudaIpcGetMemHandle(&h, c->p2p_local) == cudaSuccess;
  cudaGetLastError();
  // every rank takes part in the collectives below, whatever its own state
  const int nw = (int)((sizeof(h) + 7) / 8);
  int64_t *d_in = nullptr, *d_out = nullptr;
  std::vector<int64_t> mine((size_t)nw + 1, 0), all((size_t)(nw + 1) * R, 0);
  memcpy(mine.data(), &h, sizeof(h));
  mine[nw] = ok ? 1 : 0;
  if (cudaMalloc((void**)&d_in, sizeof(int64_t) * (nw + 1)) != cudaSuccess ||
      cudaMalloc((void**)&d_out, sizeof(int64_t) * (nw + 1) * R) != cudaSuccess) {
    cudaFree(d_in);
    ok = false;
    cudaGetLastError();
    return;  // (no collective issued by this rank: the NCCL set-up itself is broken)
  }
  cudaMemcpy(d_in, mine.data(), sizeof(int64_t) * (nw + 1), cudaMemcpyHostToDevice);
  const bool gathered = ncclAllGather(d_in, d_out, (size_t)(nw + 1), ncclInt64, c->nccl, 0) == ncclSuccess;
  cudaMemcpy(all.data(), d_out, sizeof(int64_t) * (nw + 1) * R, cudaMemcpyDeviceToHost);
  for (int r = 0; r < R && gathered; ++r) ok = ok && all[(size_t)r * (nw + 1) + nw] == 1;
  ok = ok && gathered;
  std::vector<uint8_t*> peers((size_t)R, nullptr);
  for (int r = 0; r < R && ok; ++r) {
    if (r == c->rank) {
      peers[r] = (uint8_t*)c->p2p_local;
      continue;
    }
    cudaIpcMemHandle_t hr;
    memcpy(&hr, &all[(size_t)r * (nw + 1)], sizeof(hr));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      ok = false;
      cudaGetLastError();
      break;
    }
    peers[r] = (uint8_t*)p;
    c->p2p_opened.push_back(p);
  }
  // agree: P2P only if every rank opened every peer
  int64_t* d_ok = d_in;
  const int64_t okv = ok ? 1 : 0;
  cudaMemcpy(d_ok, &okv, sizeof(int64_t), cudaMemcpyHostToDevice);
  bool all_ok = ncclAllReduce(d_ok, d_ok, 1, ncclInt64, ncclMin, c->nccl, 0) == ncclSuccess;
  int64_t agreed = 0;
  cudaMemcpy(&agreed, d_ok, sizeof(int64_t), cudaMemcpyDeviceToHost);
  all_ok = all_ok && agreed == 1;
  cudaFree(d_in);
  cudaFree(d_out);
  if (all_ok && cudaMalloc((void**)&c->d_p2p_peers, sizeof(uint8_t*) * R) == cudaSuccess &&
      cudaMemcpy(c->d_p2p_peers, peers.data(), sizeof(uint8_t*) * R, cudaMemcpyHostToDevice) == cudaSuccess)
    c->p2p = true;
  cudaGetLastError();
}

void p2p_free(sem_comm* c) {
  for (void* p : c->p2p_opened) cudaIpcCloseMemHandle(p);
  c->p2p_opened.clear();
  if (c->d_p2p_peers) cudaFree(c->d_p2p_peers);
  if (c->p2p_local) cudaFree(c->p2p_local);
  if (c->p2p_seq) cudaFree(c->p2p_seq);
  c->d_p2p_peers = nullptr;
  c->p2p_local = nullptr;
  c->p2p_seq = nullptr;
  c->p2p = false;
}
#endif

cudaError_t launch_p2p_allreduce(sem_mesh* m, double* vals, int n, cudaStream_t s) {
  if (n > kP2PVals) return cudaErrorInvalidValue;
  sem_comm* c = m->comm;
  SEM_COUNT_LAUNCH(m);
  P2PArgs A{c->d_p2p_peers, (uint8_t*)c->p2p_local, c->p2p_seq, c->rank, c->nranks};
  k_p2p_allreduce<<<1, 32, 0, s>>>(vals, n, A);
  return cudaGetLastError();
}

}  // namespace sem
