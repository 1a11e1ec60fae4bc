// CG scalar allreduce over NVLink peer memory (reading R10 across ranks: the
// dot products of PAPER.md's CG are global sums).  Each rank owns a small
// mailbox in device memory, mapped into every peer with CUDA IPC.  One warp
// per call: lane p stores this rank's values into slot [parity][rank] of
// peer p's mailbox, then (release) the slot's sequence flag; it then waits
// (acquire) for every peer's flag in the local mailbox and lane 0 sums the
// slots in ASCENDING RANK ORDER -- every rank computes bit-identical sums.
// Mailboxes alternate by call parity: a rank can only reuse a parity after
// every peer finished reading it (the next call needs all their flags).
// A bounded spin (~2 s) turns a lost peer into a sticky device error word
// (checked by the host: SEM_ENCCL, communicator retired) and NaN results
// instead of a hang.  Replaces a 1-2 value ncclAllReduce (~10-20 us in a
// graph) with one ~2-4 us kernel; NCCL stays the fallback.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <type_traits>

#include <string>
#include <vector>

#include "device_common.cuh"
#include "p2p.cuh"

namespace sem {

__global__ void __launch_bounds__(32) k_p2p_allreduce(double* vals, int n, P2PArgs A) {
  p2p_allreduce_warp(vals, n, A, threadIdx.x);
}

#ifdef SEM_WITH_NCCL
// Handshake buffers of the set-up collectives: static device memory, so a
// rank whose allocations fail still takes part in every collective (it
// reports ok = 0 instead of leaving its peers blocked).
constexpr int kHsWords = 64 + 3 + 64;            // IPC handle words + counts + per-rank offsets
__device__ int64_t g_hs_in[kHsWords];
__device__ int64_t g_hs_out[kHsWords * 64];       // <= 64 ranks
static bool handshake_buffers(int64_t** d_in, int64_t** d_out) {
  return cudaGetSymbolAddress((void**)d_in, g_hs_in) == cudaSuccess &&
         cudaGetSymbolAddress((void**)d_out, g_hs_out) == cudaSuccess;
}

// Collective (every rank calls it): allocate and zero the mailbox, exchange
// IPC handles (ncclAllGather), open the peers' mailboxes.  Leaves c->p2p
// false (NCCL allreduce) if any step fails or the communicator was created
// with p2p = 0.
void p2p_setup(sem_comm* c) {
  c->p2p = false;
  const bool want = c->want_p2p;
  const int R = c->nranks;
  const size_t bytes = (size_t)2 * R * kP2PVals * sizeof(double) + (size_t)2 * R * sizeof(unsigned long long);
  bool ok = want && R > 1 && R <= 32;
  cudaIpcMemHandle_t h{};
  const int nw = (int)((sizeof(h) + 7) / 8);
  int64_t *d_in = nullptr, *d_out = nullptr;
  if (!handshake_buffers(&d_in, &d_out) || R > 64 || nw + 1 > kHsWords) {
    cudaGetLastError();
    return;  // (cannot happen: static buffers; every rank sees the same R)
  }
  if (ok) ok = cudaMalloc((void**)&c->p2p_local, bytes) == cudaSuccess;
  if (ok) ok = cudaMemset(c->p2p_local, 0, bytes) == cudaSuccess;
  if (ok) ok = cudaMalloc((void**)&c->p2p_seq, sizeof(unsigned long long)) == cudaSuccess;
  if (ok) ok = cudaMemset(c->p2p_seq, 0, sizeof(unsigned long long)) == cudaSuccess;
  if (ok) ok = cudaIpcGetMemHandle(&h, c->p2p_local) == cudaSuccess;
  cudaGetLastError();
  // every rank takes part in the collectives below, whatever its own state
  std::vector<int64_t> mine((size_t)nw + 1, 0), all((size_t)(nw + 1) * R, 0);
  memcpy(mine.data(), &h, sizeof(h));
  mine[nw] = ok ? 1 : 0;
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

// ---------------------------------------------------------------------------
// Interface exchange over NVLink peer memory (the gather-scatter across ranks,
// reading R7): the pack kernel stores this rank's interface partials straight
// into every peer's receive region (its exchange buffer U, CUDA IPC mapped),
// alternating two regions by call parity, and its last block releases one
// sequence flag per peer; the receiver waits (acquire) for its peers' flags
// before the unpack sums all ranks' partials in rank order.  The transfer
// overlaps the interior operator launch that follows the pack.  A rank can be
// at most one exchange ahead of a peer (its next unpack needs the peer's next
// pack, which follows the peer's unpack), so two regions suffice.
// U layout: [own partials (nn) | recv parity 0 (nrecv) | parity 1 | flags[R]].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_if_pack_p2p(const double* __restrict__ U, const int32_t* __restrict__ idx,
                                                     const int32_t* __restrict__ peer_of, int64_t n,
                                                     const int64_t* __restrict__ peer_off, double* const* dst,
                                                     const int64_t* __restrict__ dst_stride,
                                                     unsigned long long* const* dst_flag, int npeers,
                                                     const unsigned long long* seqp, unsigned* ticket) {
  __shared__ int s_last;
  const unsigned long long seq = *seqp + 1;
  const int par = (int)(seq & 1);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int pe = peer_of[q];
    dst[pe][par * dst_stride[pe] + (q - peer_off[pe])] = U[idx[q]];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicInc(ticket, gridDim.x - 1) == gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    for (int pe = threadIdx.x; pe < npeers; pe += blockDim.x) st_release_sys(dst_flag[pe], seq);
  }
}

// The flags only grow, and a fast peer may already have released its NEXT
// exchange (into the other receive region) when this rank starts waiting:
// wait for flag >= seq.  A lost peer (~2 s) poisons its receive slots with
// NaN and sets the communicator's sticky error word instead of hanging.
__global__ void __launch_bounds__(32) k_if_wait_p2p(const unsigned long long* flags, const int32_t* peer_rank,
                                                    int npeers, unsigned long long* seqp, double* recv,
                                                    const int64_t* peer_off, unsigned* err) {
  const unsigned long long seq = *seqp + 1;
  const int64_t nrecv = peer_off[npeers];
  for (int pe = threadIdx.x; pe < npeers; pe += 32) {
    const long long t0 = clock64();
    while (ld_acquire_sys(flags + peer_rank[pe]) < seq)
      if (clock64() - t0 > (1ll << 32)) {
        double* r = recv + (int64_t)(seq & 1) * nrecv;
        for (int64_t q = peer_off[pe]; q < peer_off[pe + 1]; ++q) r[q] = __longlong_as_double(0x7ff8000000000000ll);
        atomicOr(err, kP2PErrTimeout);
        break;
      }
  }
  __syncwarp();
  if (threadIdx.x == 0) *seqp = seq;
}

#ifdef SEM_WITH_NCCL
// Collective over the mesh's ranks (called by comm_setup_device after U is
// allocated with both receive regions and the flags): publish U's IPC handle,
// nn, nrecv and where each source rank's data goes; open the peers' U.
void p2p_xchg_setup(sem_mesh* m) {
  sem_comm* c = m->comm;
  m->xp2p = false;
  const bool want = c->want_p2p;
  const int R = c->nranks;
  const IfacePlan& P = m->iface;
  cudaIpcMemHandle_t h{};
  bool ok = want && c->p2p && cudaIpcGetMemHandle(&h, m->d_U) == cudaSuccess;
  cudaGetLastError();
  const int nw = (int)((sizeof(h) + 7) / 8), W = nw + 3 + R;
  std::vector<int64_t> mine((size_t)W, -1), all((size_t)W * R, -1);
  memcpy(mine.data(), &h, sizeof(h));
  mine[nw] = ok ? 1 : 0;
  mine[nw + 1] = m->n_if_nodes;
  mine[nw + 2] = m->peer_off.empty() ? 0 : m->peer_off.back();
  for (size_t pe = 0; pe < P.peers.size(); ++pe) mine[(size_t)nw + 3 + P.peers[pe]] = m->peer_off[pe];
  int64_t *d_in = nullptr, *d_out = nullptr;
  if (!handshake_buffers(&d_in, &d_out) || W > kHsWords || R > 64) {
    cudaGetLastError();
    return;  // (cannot happen: static buffers, W <= 16 + 3 + 32)
  }
  cudaMemcpy(d_in, mine.data(), sizeof(int64_t) * W, cudaMemcpyHostToDevice);
  const bool gathered = ncclAllGather(d_in, d_out, (size_t)W, ncclInt64, c->nccl, 0) == ncclSuccess;
  cudaMemcpy(all.data(), d_out, sizeof(int64_t) * W * R, cudaMemcpyDeviceToHost);
  ok = ok && gathered;
  for (int r = 0; r < R && ok; ++r) ok = all[(size_t)r * W + nw] == 1;
  const int np = (int)P.peers.size();
  std::vector<double*> dst((size_t)np, nullptr);
  std::vector<int64_t> stride((size_t)np, 0);
  std::vector<unsigned long long*> flag((size_t)np, nullptr);
  std::vector<int32_t> prank((size_t)np, 0);
  for (int pe = 0; pe < np && ok; ++pe) {
    const int r = P.peers[pe];
    const int64_t* rec = &all[(size_t)r * W];
    cudaIpcMemHandle_t hr;
    memcpy(&hr, rec, sizeof(hr));
    void* base = nullptr;
    if (cudaIpcOpenMemHandle(&base, hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      ok = false;
      cudaGetLastError();
      break;
    }
    m->x_opened.push_back(base);
    const int64_t nn_r = rec[nw + 1], nrecv_r = rec[nw + 2], off_me = rec[nw + 3 + c->rank];
    if (off_me < 0) {
      ok = false;
      break;
    }
    dst[pe] = (double*)base + nn_r + off_me;
    stride[pe] = nrecv_r;
    flag[pe] = (unsigned long long*)((double*)base + nn_r + 2 * nrecv_r) + c->rank;
    prank[pe] = r;
  }
  std::vector<int32_t> peer_of(m->peer_off.empty() ? 0 : (size_t)m->peer_off.back());
  for (int pe = 0; pe < np; ++pe)
    for (int64_t q = m->peer_off[pe]; q < m->peer_off[pe + 1]; ++q) peer_of[(size_t)q] = pe;
  auto up = [&](auto** d, const auto& hv) -> bool {
    using V = typename std::remove_reference<decltype(hv)>::type::value_type;
    if (hv.empty()) return true;
    if (cudaMalloc((void**)d, sizeof(V) * hv.size()) != cudaSuccess) return false;
    return cudaMemcpy(*d, hv.data(), sizeof(V) * hv.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (ok) ok = up(&m->d_x_dst, dst) && up(&m->d_x_stride, stride) && up(&m->d_x_flag, flag) &&
               up(&m->d_x_prank, prank) && up(&m->d_x_peer_of, peer_of) && up(&m->d_x_peer_off, m->peer_off);
  if (ok) ok = cudaMalloc((void**)&m->d_x_seq, sizeof(unsigned long long) + sizeof(unsigned)) == cudaSuccess &&
               cudaMemset(m->d_x_seq, 0, sizeof(unsigned long long) + sizeof(unsigned)) == cudaSuccess;
  // agree (every rank must take the same path)
  const int64_t okv = ok ? 1 : 0;
  cudaMemcpy(d_in, &okv, sizeof(int64_t), cudaMemcpyHostToDevice);
  bool agreed = ncclAllReduce(d_in, d_in, 1, ncclInt64, ncclMin, c->nccl, 0) == ncclSuccess;
  int64_t v = 0;
  cudaMemcpy(&v, d_in, sizeof(int64_t), cudaMemcpyDeviceToHost);
  m->xp2p = agreed && v == 1;
  cudaGetLastError();
}
#endif

void p2p_xchg_free(sem_mesh* m) {
  for (void* q : m->x_opened) cudaIpcCloseMemHandle(q);
  m->x_opened.clear();
  void* ptrs[] = {m->d_x_dst, m->d_x_stride, m->d_x_flag, m->d_x_prank, m->d_x_peer_of, m->d_x_peer_off, m->d_x_seq};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  m->xp2p = false;
}

cudaError_t launch_if_pack_p2p(const sem_mesh* m, cudaStream_t s) {
  const int64_t n = m->peer_off.empty() ? 0 : m->peer_off.back();
  if (n == 0) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  const unsigned long long* seq = m->d_x_seq;
  unsigned* ticket = reinterpret_cast<unsigned*>(m->d_x_seq + 1);
  unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)m->nsm * 4);
  k_if_pack_p2p<<<blocks, 256, 0, s>>>(m->d_U, m->d_send_idx, m->d_x_peer_of, n, m->d_x_peer_off, m->d_x_dst,
                                        m->d_x_stride, m->d_x_flag, (int)m->iface.peers.size(), seq, ticket);
  return cudaGetLastError();
}

cudaError_t launch_if_wait_p2p(const sem_mesh* m, cudaStream_t s) {
  if (m->iface.peers.empty()) return cudaSuccess;
  SEM_COUNT_LAUNCH(m);
  const int64_t nrecv = m->peer_off.back();
  const unsigned long long* flags = (const unsigned long long*)(m->d_U + m->n_if_nodes + 2 * nrecv);
  k_if_wait_p2p<<<1, 32, 0, s>>>(flags, m->d_x_prank, (int)m->iface.peers.size(), m->d_x_seq,
                                  m->d_U + m->n_if_nodes, m->d_x_peer_off, m->comm->d_err);
  return cudaGetLastError();
}

P2PArgs p2p_args(const sem_mesh* m) {
  const sem_comm* c = m->comm;
  if (!c || !c->p2p) return P2PArgs{nullptr, nullptr, nullptr, nullptr, 0, 1};
  return P2PArgs{c->d_p2p_peers, (uint8_t*)c->p2p_local, c->p2p_seq, c->d_err, c->rank, c->nranks};
}

cudaError_t launch_p2p_allreduce(sem_mesh* m, double* vals, int n, cudaStream_t s) {
  if (n > kP2PVals) return cudaErrorInvalidValue;
  sem_comm* c = m->comm;
  SEM_COUNT_LAUNCH(m);
  P2PArgs A{c->d_p2p_peers, (uint8_t*)c->p2p_local, c->p2p_seq, c->d_err, c->rank, c->nranks};
  k_p2p_allreduce<<<1, 32, 0, s>>>(vals, n, A);
  return cudaGetLastError();
}

}  // namespace sem
