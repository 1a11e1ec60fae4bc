// Multi-GPU plumbing (PAPER.md:74 elements "distributed among the MPI
// ranks"; "only unit-depth communication is necessary in a
// so-called gather-scatter phase"): NCCL communicator bootstrap, the
// interface plan, the interface exchange of the gather-scatter and the CG
// scalar allreduce.
//
// Exchange (reading R7 across ranks): every rank sums its local copies of an
// interface entity (ascending local element order) into a partial, sends the
// partial to every rank sharing the entity and receives theirs (grouped
// ncclSend/ncclRecv over NVLink, straight from device buffers); the total is
// the sum of the per-rank partials in ASCENDING RANK ORDER, so every rank
// computes bit-identical values for its copies.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.h"

namespace sem {

#ifdef SEM_WITH_NCCL
#define SEM_NCCL_TRY(expr)                                                                          \
  do {                                                                                              \
    ncclResult_t _r = (expr);                                                                       \
    if (_r != ncclSuccess) return fail(SEM_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)
#endif

cudaError_t launch_if_partial(const sem_mesh* m, const double* u, cudaStream_t s);
cudaError_t launch_if_pack(const sem_mesh* m, cudaStream_t s);
cudaError_t launch_if_unpack(const sem_mesh* m, double* u, int mode, cudaStream_t s);
cudaError_t launch_mult_mask(const sem_mesh* m, cudaStream_t s);
cudaError_t launch_p2p_allreduce(sem_mesh* m, double* vals, int n, cudaStream_t s);
cudaError_t launch_if_pack_p2p(const sem_mesh* m, cudaStream_t s);
cudaError_t launch_if_wait_p2p(const sem_mesh* m, cudaStream_t s);
void p2p_xchg_free(sem_mesh* m);
#ifdef SEM_WITH_NCCL
void p2p_xchg_setup(sem_mesh* m);
#endif
#ifdef SEM_WITH_NCCL
void p2p_setup(sem_comm* c);
void p2p_free(sem_comm* c);
#endif

#ifdef SEM_WITH_NCCL
// host <-> device helpers for small setup collectives (synchronous)
static sem_status allgather_i64(sem_comm* c, const std::vector<int64_t>& mine, int64_t per_rank,
                                std::vector<int64_t>* all) {
  int64_t *d_in = nullptr, *d_out = nullptr;
  const size_t nb = sizeof(int64_t) * (size_t)std::max<int64_t>(per_rank, 1);
  if (cudaMalloc((void**)&d_in, nb) != cudaSuccess || cudaMalloc((void**)&d_out, nb * c->nranks) != cudaSuccess) {
    cudaFree(d_in);
    return fail(SEM_ENOMEM, "allgather buffers");
  }
  std::vector<int64_t> pad((size_t)std::max<int64_t>(per_rank, 1), -2);
  std::copy(mine.begin(), mine.end(), pad.begin());
  cudaMemcpy(d_in, pad.data(), nb, cudaMemcpyHostToDevice);
  ncclResult_t r = ncclAllGather(d_in, d_out, (size_t)std::max<int64_t>(per_rank, 1), ncclInt64, c->nccl, 0);
  all->resize((size_t)std::max<int64_t>(per_rank, 1) * c->nranks);
  cudaError_t ce = cudaMemcpy(all->data(), d_out, nb * c->nranks, cudaMemcpyDeviceToHost);
  cudaFree(d_in);
  cudaFree(d_out);
  if (r != ncclSuccess) return fail(SEM_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
  if (ce != cudaSuccess) return fail(SEM_ECUDA, "allgather copy");
  return SEM_OK;
}

static sem_status allreduce_i64(sem_comm* c, int64_t* v, int n) {
  int64_t* d = nullptr;
  if (cudaMalloc((void**)&d, sizeof(int64_t) * n) != cudaSuccess) return fail(SEM_ENOMEM, "allreduce buffer");
  cudaMemcpy(d, v, sizeof(int64_t) * n, cudaMemcpyHostToDevice);
  ncclResult_t r = ncclAllReduce(d, d, n, ncclInt64, ncclSum, c->nccl, 0);
  cudaMemcpy(v, d, sizeof(int64_t) * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (r != ncclSuccess) return fail(SEM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  return SEM_OK;
}

// per-peer exchange of one int64 value per shared interface entity
// (entity order = each peer's list order, identical on both sides)
static sem_status exchange_entity_i64(sem_mesh* m, const std::vector<int64_t>& val,
                                      std::vector<std::vector<int64_t>>* recv) {
  const IfacePlan& P = m->iface;
  int64_t tot = 0;
  for (auto& l : P.peer_list) tot += (int64_t)l.size();
  std::vector<int64_t> send;
  send.reserve(tot);
  for (auto& l : P.peer_list)
    for (int32_t q : l) send.push_back(val[q]);
  int64_t *d_s = nullptr, *d_r = nullptr;
  const size_t nb = sizeof(int64_t) * (size_t)std::max<int64_t>(tot, 1);
  if (cudaMalloc((void**)&d_s, nb) != cudaSuccess || cudaMalloc((void**)&d_r, nb) != cudaSuccess) {
    cudaFree(d_s);
    return fail(SEM_ENOMEM, "exchange buffers");
  }
  if (tot) cudaMemcpy(d_s, send.data(), sizeof(int64_t) * tot, cudaMemcpyHostToDevice);
  ncclResult_t r = ncclGroupStart();
  int64_t off = 0;
  for (size_t p = 0; p < P.peers.size() && r == ncclSuccess; ++p) {
    const size_t n = P.peer_list[p].size();
    r = ncclSend(d_s + off, n, ncclInt64, P.peers[p], m->comm->nccl, 0);
    if (r == ncclSuccess) r = ncclRecv(d_r + off, n, ncclInt64, P.peers[p], m->comm->nccl, 0);
    off += (int64_t)n;
  }
  ncclResult_t r2 = ncclGroupEnd();
  std::vector<int64_t> got(tot);
  if (tot) cudaMemcpy(got.data(), d_r, sizeof(int64_t) * tot, cudaMemcpyDeviceToHost);
  cudaFree(d_s);
  cudaFree(d_r);
  if (r != ncclSuccess || r2 != ncclSuccess) return fail(SEM_ENCCL, "exchange_entity_i64: NCCL send/recv");
  recv->assign(P.peers.size(), {});
  off = 0;
  for (size_t p = 0; p < P.peers.size(); ++p) {
    (*recv)[p].assign(got.begin() + off, got.begin() + off + P.peer_list[p].size());
    off += (int64_t)P.peer_list[p].size();
  }
  return SEM_OK;
}
#endif

// Called after build_topology, before any upload: find the interface
// entities (marks kEntInterface) and the processing order (elements that
// touch the interface first, so the exchange can start while the interior is
// still being computed).
sem_status comm_plan_interface(sem_mesh* m, std::vector<int64_t>* pos) {
#ifdef SEM_WITH_NCCL
  sem_comm* c = m->comm;
  Topology& T = m->topo;
  std::vector<int64_t> keys;
  std::vector<int32_t> ents;
  iface_candidates(T, &keys, &ents);
  std::vector<int64_t> counts_all;
  SEM_TRY_ST(allgather_i64(c, {(int64_t)ents.size()}, 1, &counts_all));
  int64_t maxc = 0;
  for (int r = 0; r < c->nranks; ++r) maxc = std::max(maxc, counts_all[r]);
  std::vector<int64_t> gathered;
  SEM_TRY_ST(allgather_i64(c, keys, maxc * 4, &gathered));
  std::vector<int64_t> all_keys;
  all_keys.reserve(gathered.size());
  for (int r = 0; r < c->nranks; ++r)
    all_keys.insert(all_keys.end(), gathered.begin() + (size_t)r * std::max<int64_t>(maxc * 4, 1),
                    gathered.begin() + (size_t)r * std::max<int64_t>(maxc * 4, 1) + counts_all[r] * 4);
  std::string err = iface_plan(T, c->rank, c->nranks, std::vector<int64_t>(counts_all.begin(), counts_all.end()),
                               all_keys, &m->iface);
  if (!err.empty()) return fail(SEM_EINVAL, err);
  for (int32_t x : m->iface.ents) T.ent_flags[x] |= kEntInterface;
  // boundary elements first
  std::vector<uint8_t> bnd(m->E, 0);
  for (int32_t x : m->iface.ents)
    for (int cc = T.ent_ptr[x]; cc < T.ent_ptr[x + 1]; ++cc) bnd[T.ent_copy[cc] >> 8] = 1;
  pos->assign(m->E, 0);
  int64_t q = 0;
  for (int64_t e = 0; e < m->E; ++e)
    if (bnd[e]) (*pos)[e] = q++;
  m->n_boundary = q;
  for (int64_t e = 0; e < m->E; ++e)
    if (!bnd[e]) (*pos)[e] = q++;
  int64_t nn = 0;
  for (int32_t x : m->iface.ents) nn += T.ent_nodes(x);
  m->n_interface = nn;
  return SEM_OK;
#else
  (void)m; (void)pos;
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

// Called after the uploads: global multiplicity and masks of interface
// entities, device exchange tables, global unique / masked counts.
sem_status comm_setup_device(sem_mesh* m) {
#ifdef SEM_WITH_NCCL
  sem_comm* c = m->comm;
  Topology& T = m->topo;
  const IfacePlan& P = m->iface;
  const int64_t ni = (int64_t)P.ents.size();
  const int mm = m->lx - 2;
  // exchange local copy counts and Dirichlet flags of interface entities
  std::vector<int64_t> cnt(ni), msk(ni);
  for (int64_t q = 0; q < ni; ++q) {
    const int32_t x = P.ents[q];
    cnt[q] = T.ent_ptr[x + 1] - T.ent_ptr[x];
    msk[q] = (T.ent_flags[x] & kEntMasked) ? 1 : 0;
  }
  std::vector<std::vector<int64_t>> rc, rm;
  SEM_TRY_ST(exchange_entity_i64(m, cnt, &rc));
  SEM_TRY_ST(exchange_entity_i64(m, msk, &rm));
  std::vector<int32_t> gcount(T.nEnt());
  for (int64_t x = 0; x < T.nEnt(); ++x) gcount[x] = T.ent_ptr[x + 1] - T.ent_ptr[x];
  std::vector<int64_t> gc(cnt), gm(msk);
  for (size_t p = 0; p < P.peers.size(); ++p)
    for (size_t k = 0; k < P.peer_list[p].size(); ++k) {
      gc[P.peer_list[p][k]] += rc[p][k];
      gm[P.peer_list[p][k]] |= rm[p][k];
    }
  for (int64_t q = 0; q < ni; ++q) {
    gcount[P.ents[q]] = (int32_t)gc[q];
    if (gm[q]) T.ent_flags[P.ents[q]] |= kEntMasked;
  }
  // unique / masked counts: an interface entity is counted by its lowest rank
  int64_t uniq = 0, masked = 0;
  {
    const int64_t interior = m->E * (int64_t)mm * mm * mm;
    uniq = interior;
    std::vector<uint8_t> isif(T.nEnt(), 0);
    for (int64_t q = 0; q < ni; ++q) isif[P.ents[q]] = (P.ranks[q][0] == c->rank) ? 2 : 1;
    for (int64_t x = 0; x < T.nEnt(); ++x) {
      if (isif[x] == 1) continue;
      uniq += T.ent_nodes(x);
    }
    for (int64_t x = 0; x < T.nEnt(); ++x)
      if (T.ent_flags[x] & kEntMasked) masked += (int64_t)T.ent_nodes(x) * (T.ent_ptr[x + 1] - T.ent_ptr[x]);
  }
  m->n_masked = masked;
  int64_t red[2] = {uniq, masked};
  SEM_TRY_ST(allreduce_i64(c, red, 2));
  m->n_unique = red[0];
  m->n_masked_glob = red[1];
  // device tables
  std::vector<int32_t> if_ent(P.ents.begin(), P.ents.end()), node_ent;
  std::vector<int64_t> noff(ni + 1, 0);
  for (int64_t q = 0; q < ni; ++q) {
    noff[q + 1] = noff[q] + T.ent_nodes(P.ents[q]);
    for (int n = 0; n < T.ent_nodes(P.ents[q]); ++n) node_ent.push_back((int32_t)q);
  }
  const int64_t nn = noff[ni];
  m->peer_cnt.assign(P.peers.size(), 0);
  m->peer_off.assign(P.peers.size() + 1, 0);
  std::vector<int32_t> send_idx;
  for (size_t p = 0; p < P.peers.size(); ++p) {
    for (int32_t q : P.peer_list[p])
      for (int64_t n = noff[q]; n < noff[q + 1]; ++n) send_idx.push_back((int32_t)n);
    m->peer_off[p + 1] = (int64_t)send_idx.size();
    m->peer_cnt[p] = m->peer_off[p + 1] - m->peer_off[p];
  }
  // contributions of each interface entity, by rank: offsets into U =
  // [own partials (nn) | received from peer 0 | peer 1 | ...]
  std::vector<int32_t> src_ptr(ni + 1, 0);
  std::vector<int64_t> src;
  {
    std::vector<std::vector<int64_t>> pos_in_peer(ni);  // per entity: (peer index, node offset in recv)
    std::vector<int64_t> recv_at(P.peers.size(), 0);
    for (size_t p = 0; p < P.peers.size(); ++p) {
      int64_t off = nn + m->peer_off[p];
      for (int32_t q : P.peer_list[p]) {
        pos_in_peer[q].push_back((int64_t)p);
        pos_in_peer[q].push_back(off);
        off += noff[q + 1] - noff[q];
      }
    }
    for (int64_t q = 0; q < ni; ++q) {
      for (int r : P.ranks[q]) {
        if (r == c->rank) {
          src.push_back(noff[q]);
        } else {
          const int pi = (int)(std::lower_bound(P.peers.begin(), P.peers.end(), r) - P.peers.begin());
          int64_t o = -1;
          for (size_t k = 0; k + 1 < pos_in_peer[q].size(); k += 2)
            if (pos_in_peer[q][k] == pi) o = pos_in_peer[q][k + 1];
          if (o < 0) return fail(SEM_EINVAL, "interface plan: missing peer contribution");
          src.push_back(o);
        }
      }
      src_ptr[q + 1] = (int32_t)src.size();
    }
  }
  m->n_if_nodes = nn;
  auto up = [&](auto** d, const auto& h) -> sem_status {
    using V = typename std::remove_reference<decltype(h)>::type::value_type;
    if (*d) cudaFree(*d);
    *d = nullptr;
    if (h.empty()) return SEM_OK;
    if (cudaMalloc((void**)d, sizeof(V) * h.size()) != cudaSuccess) return fail(SEM_ENOMEM, "cudaMalloc(iface)");
    if (cudaMemcpy(*d, h.data(), sizeof(V) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SEM_ECUDA, "upload iface");
    return SEM_OK;
  };
  SEM_TRY_ST(up(&m->d_if_ent, if_ent));
  SEM_TRY_ST(up(&m->d_if_node_ent, node_ent));
  SEM_TRY_ST(up(&m->d_if_noff, noff));
  SEM_TRY_ST(up(&m->d_if_src_ptr, src_ptr));
  SEM_TRY_ST(up(&m->d_if_src, src));
  SEM_TRY_ST(up(&m->d_send_idx, send_idx));
  SEM_TRY_ST(up(&m->d_ent_gcount, gcount));
  // U: own partials, two receive regions (P2P parity; NCCL uses the first),
  // one P2P flag per source rank
  const int64_t nU = nn + 2 * m->peer_off.back() + c->nranks;
  if (cudaMalloc((void**)&m->d_U, sizeof(double) * std::max<int64_t>(nU, 1)) != cudaSuccess ||
      cudaMalloc((void**)&m->d_sendbuf, sizeof(double) * std::max<int64_t>(m->peer_off.back(), 1)) != cudaSuccess)
    return fail(SEM_ENOMEM, "cudaMalloc(exchange buffers)");
  cudaMemset(m->d_U, 0, sizeof(double) * std::max<int64_t>(nU, 1));
  p2p_xchg_setup(m);  // collective; m->xp2p stays false without peer mappings
  if (cudaMemcpy(m->d_ent_flags, T.ent_flags.data(), T.ent_flags.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(SEM_ECUDA, "upload flags");
  cudaError_t ce = launch_mult_mask(m, 0);
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) return fail(SEM_ECUDA, std::string("mult/mask: ") + cudaGetErrorString(ce));
  if (!m->comm_stream && cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SEM_ECUDA, "comm stream");
  for (cudaEvent_t* ev : {&m->ev_pack, &m->ev_comm})
    if (!*ev && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) return fail(SEM_ECUDA, "event");
  return SEM_OK;
#else
  (void)m;
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

sem_status comm_allreduce_sum(sem_mesh* m, double* d, int n, cudaStream_t s) {
#ifdef SEM_WITH_NCCL
  if (m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  if (m->comm->p2p && n <= 4) {
    SEM_CUDA_TRY(launch_p2p_allreduce(m, d, n, s));
    return SEM_OK;
  }
  SEM_NCCL_TRY(ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclSum, m->comm->nccl, s));
  return SEM_OK;
#else
  (void)m; (void)d; (void)n; (void)s;
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

// Interface part of the gather-scatter.  Phase 1 (after every element that
// touches the interface is done): own partials + pack, then the grouped
// send/recv on comm_stream.  Phase 2: per-node sum of all ranks' partials
// in rank order, written to the local copies (0 where masked).
sem_status comm_exchange_begin(sem_mesh* m, const double* u, cudaStream_t s) {
#ifdef SEM_WITH_NCCL
  if (!m->comm || m->iface.peers.empty()) return SEM_OK;
  if (m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  SEM_CUDA_TRY(launch_if_partial(m, u, s));
  if (m->xp2p) {  // partials stored straight into the peers' receive regions
    SEM_CUDA_TRY(launch_if_pack_p2p(m, s));
    return SEM_OK;
  }
  SEM_CUDA_TRY(launch_if_pack(m, s));
  SEM_CUDA_TRY(cudaEventRecord(m->ev_pack, s));
  SEM_CUDA_TRY(cudaStreamWaitEvent(m->comm_stream, m->ev_pack, 0));
  const IfacePlan& P = m->iface;
  SEM_NCCL_TRY(ncclGroupStart());
  for (size_t p = 0; p < P.peers.size(); ++p) {
    SEM_NCCL_TRY(ncclSend(m->d_sendbuf + m->peer_off[p], (size_t)m->peer_cnt[p], ncclDouble, P.peers[p],
                          m->comm->nccl, m->comm_stream));
    SEM_NCCL_TRY(ncclRecv(m->d_U + m->n_if_nodes + m->peer_off[p], (size_t)m->peer_cnt[p], ncclDouble, P.peers[p],
                          m->comm->nccl, m->comm_stream));
  }
  SEM_NCCL_TRY(ncclGroupEnd());
  SEM_CUDA_TRY(cudaEventRecord(m->ev_comm, m->comm_stream));
  return SEM_OK;
#else
  (void)m; (void)u; (void)s;
  return SEM_OK;
#endif
}

sem_status comm_exchange_end(sem_mesh* m, double* u, int mode, cudaStream_t s) {
  if (!m->comm || m->n_if_nodes == 0) return SEM_OK;
  if (m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  if (m->xp2p) {
    if (mode & 1) SEM_CUDA_TRY(launch_if_wait_p2p(m, s));
  } else if ((mode & 1) && !m->iface.peers.empty()) {
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_comm, 0));
  }
  SEM_CUDA_TRY(launch_if_unpack(m, u, mode, s));
  return SEM_OK;
}

sem_status comm_gs_exchange(sem_mesh* m, double* u, int mode, cudaStream_t s) {
  if (mode & 1) SEM_TRY_ST(comm_exchange_begin(m, u, s));
  return comm_exchange_end(m, u, mode, s);
}

// Synchronise and read the communicator's sticky error word (SEM_ENCCL and
// retire the communicator if a peer wait timed out).
sem_status comm_check(sem_comm* c) {
  if (!c) return SEM_OK;
  if (c->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  if (!c->d_err) return SEM_OK;
  unsigned e = 0;
  cudaError_t ce = cudaMemcpy(&e, c->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return fail(SEM_ECUDA, std::string("comm status: ") + cudaGetErrorString(ce));
  if (e) {
    c->broken = true;
    return fail(SEM_ENCCL, "a peer did not arrive within ~2 s (peer-memory wait timed out); communicator retired");
  }
  return SEM_OK;
}

void comm_mesh_free(sem_mesh* m) {
  p2p_xchg_free(m);
  void* ptrs[] = {m->d_if_ent, m->d_if_node_ent, m->d_if_noff, m->d_if_src_ptr, m->d_if_src,
                  m->d_send_idx, m->d_U, m->d_sendbuf, m->d_ent_gcount};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (m->ev_pack) cudaEventDestroy(m->ev_pack);
  if (m->ev_comm) cudaEventDestroy(m->ev_comm);
  if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
}

}  // namespace sem

using namespace sem;

extern "C" {

sem_status sem_comm_unique_id(void* id128) {
  if (!id128) return fail(SEM_EINVAL, "sem_comm_unique_id: NULL buffer");
#ifdef SEM_WITH_NCCL
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  SEM_NCCL_TRY(ncclGetUniqueId((ncclUniqueId*)id128));
  return SEM_OK;
#else
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

sem_status sem_comm_create(const void* id128, int rank, int nranks, int device, sem_comm_t* out) {
  return sem_comm_create_ex(id128, rank, nranks, device, 1, out);
}

sem_status sem_comm_create_ex(const void* id128, int rank, int nranks, int device, int p2p, sem_comm_t* out) {
  if (!id128 || !out) return fail(SEM_EINVAL, "sem_comm_create: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SEM_EINVAL, "sem_comm_create: bad rank/nranks");
  *out = nullptr;
#ifdef SEM_WITH_NCCL
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) return fail(SEM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce));
  sem_comm* c = new sem_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  // the sticky error word of the peer-memory paths; without it this rank
  // asks for the NCCL path (all ranks agree in p2p_setup)
  c->want_p2p = p2p != 0;
  if (cudaMalloc((void**)&c->d_err, sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(c->d_err, 0, sizeof(unsigned)) != cudaSuccess) {
    cudaGetLastError();
    if (c->d_err) cudaFree(c->d_err);
    c->d_err = nullptr;
    c->want_p2p = false;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    if (c->d_err) cudaFree(c->d_err);
    delete c;
    return fail(SEM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  p2p_setup(c);  // collective; c->p2p stays false if peer mappings are unavailable
  *out = c;
  return SEM_OK;
#else
  (void)device;
  (void)p2p;
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

sem_status sem_comm_status(sem_comm_t c, int* p2p_out) {
  if (!c) return fail(SEM_EINVAL, "sem_comm_status: NULL communicator");
  if (p2p_out) *p2p_out = c->p2p ? 1 : 0;
  return comm_check(c);
}

void sem_comm_destroy(sem_comm_t c) {
  if (!c) return;
#ifdef SEM_WITH_NCCL
  p2p_free(c);
  if (c->nccl) ncclCommDestroy(c->nccl);
#endif
  if (c->d_err) cudaFree(c->d_err);
  delete c;
}

// Host-only planning entry points (no CUDA, no NCCL): the pieces of the
// multi-GPU set-up that the CPU tests drive with torch.distributed (gloo).
sem_status sem_iface_candidates(int64_t E, int N, const int64_t* conn, int64_t* count, int64_t* keys) {
  if (!count || (E > 0 && !conn)) return fail(SEM_EINVAL, "sem_iface_candidates: NULL argument");
  if (N < 1 || N > kMaxN || E < 0) return fail(SEM_EINVAL, "sem_iface_candidates: bad E or N");
  Topology T;
  std::string err = build_topology(E, N, conn, nullptr, &T);
  if (!err.empty()) return fail(SEM_EINVAL, err);
  std::vector<int64_t> k;
  std::vector<int32_t> ents;
  iface_candidates(T, &k, &ents);
  *count = (int64_t)ents.size();
  if (keys) std::copy(k.begin(), k.end(), keys);
  return SEM_OK;
}

sem_status sem_iface_plan(int64_t E, int N, const int64_t* conn, int rank, int nranks, const int64_t* counts,
                          const int64_t* all_keys, int64_t* peer_nodes, int64_t* n_iface_entities,
                          int64_t* n_iface_nodes) {
  if (!counts || !all_keys || !peer_nodes || (E > 0 && !conn))
    return fail(SEM_EINVAL, "sem_iface_plan: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SEM_EINVAL, "sem_iface_plan: bad rank");
  Topology T;
  std::string err = build_topology(E, N, conn, nullptr, &T);
  if (!err.empty()) return fail(SEM_EINVAL, err);
  std::vector<int64_t> cnt(counts, counts + nranks);
  int64_t tot = 0;
  for (int64_t v : cnt) tot += v;
  std::vector<int64_t> keys(all_keys, all_keys + tot * 4);
  IfacePlan P;
  err = iface_plan(T, rank, nranks, cnt, keys, &P);
  if (!err.empty()) return fail(SEM_EINVAL, err);
  for (int r = 0; r < nranks; ++r) peer_nodes[r] = 0;
  int64_t nn = 0;
  for (int32_t x : P.ents) nn += T.ent_nodes(x);
  for (size_t p = 0; p < P.peers.size(); ++p)
    for (int32_t q : P.peer_list[p]) peer_nodes[P.peers[p]] += T.ent_nodes(P.ents[q]);
  if (n_iface_entities) *n_iface_entities = (int64_t)P.ents.size();
  if (n_iface_nodes) *n_iface_nodes = nn;
  return SEM_OK;
}

}  // extern "C"
