// C ABI of libsem_b200 (include/sem.h).  Argument checking, allocation and
// the orchestration of the kernels in kernels.cu; no arithmetic of the method
// runs here except the host-side basis and topology set-up.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "internal.h"

namespace sem {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
sem_status fail(sem_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
cudaError_t launch_sub_mean(sem_mesh* m, double* x, int slot, cudaStream_t s);
// comm.cpp
sem_status comm_plan_interface(sem_mesh* m, std::vector<int64_t>* pos);
sem_status comm_setup_device(sem_mesh* m);
sem_status comm_allreduce_sum(sem_mesh* m, double* d, int n, cudaStream_t s);
sem_status comm_exchange_begin(sem_mesh* m, const double* u, cudaStream_t s);
sem_status comm_exchange_end(sem_mesh* m, double* u, int mode, cudaStream_t s);
sem_status comm_gs_exchange(sem_mesh* m, double* u, int mode, cudaStream_t s);
void comm_mesh_free(sem_mesh* m);
sem_status comm_exchange_begin_u(sem_mesh* m, cudaStream_t s);
sem_status comm_exchange_end_u(sem_mesh* m, cudaStream_t s);
// ulayout.cpp
sem_status build_ulayout(sem_mesh* m, const std::vector<int64_t>& pos);
void ulayout_free(sem_mesh* m);
}  // namespace sem

using namespace sem;

#define SEM_TRY(expr)                 \
  do {                                \
    sem_status _st = (expr);          \
    if (_st != SEM_OK) return _st;    \
  } while (0)

template <class T>
static sem_status dalloc(T** p, int64_t count, const char* what) {
  *p = nullptr;
  if (count <= 0) return SEM_OK;
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (size_t)count);
  if (e != cudaSuccess) {
    *p = nullptr;
    cudaGetLastError();
    return fail(SEM_ENOMEM, std::string("cudaMalloc(") + what + ", " +
                                std::to_string(sizeof(T) * (size_t)count) + " B): " + cudaGetErrorString(e));
  }
  return SEM_OK;
}

// Gather-scatter plan.  Every shared entity (a face,
// edge or vertex needing a sum or a mask) that is not on the rank interface
// is finished in the chunk of its LAST copy (pos[e] = processing position),
// once every chunk holding one of its copies is done.
static sem_status build_gs_lists(sem_mesh* m, const std::vector<int64_t>& pos) {
  const Topology& T = m->topo;
  const int64_t E = m->E;
  const int mm = m->lx - 2;
  // Schedule: by default the operator runs in stream
  // order and one gather-scatter pass follows it (measured faster than
  // overlapping the two: the concurrent gs costs the bandwidth-bound
  // operator more than it hides).  Chunks then only serve the interface
  // exchange: the boundary elements (processed first) form chunk 0, so the
  // exchange starts while the interior is computed; one rank: one chunk.
  // SEM_GS_OVERLAP=1: the older pipeline of ~4M-double chunks (operator on
  // two lanes, each chunk's gs on a high-priority stream).
  m->gs_overlap = false;
  if (const char* env = getenv("SEM_GS_OVERLAP")) m->gs_overlap = atoi(env) != 0;  // tuning knob
  int shift = 4;
  if (m->gs_overlap) {
    while ((int64_t(1) << (shift + 1)) * m->n3 <= (int64_t(1) << 22) && shift < 20) ++shift;
  } else {
    const int64_t span = (m->comm && m->n_boundary > 0) ? m->n_boundary : E;
    while ((int64_t(1) << shift) < span && shift < 30) ++shift;
  }
  if (const char* env = getenv("SEM_CHUNK_SHIFT")) shift = std::max(4, std::min(30, atoi(env)));  // tuning knob
  m->chunk_shift = shift;
  m->lanes = 2;
  if (const char* env = getenv("SEM_LANES")) m->lanes = std::max(1, std::min(2, atoi(env)));  // tuning knob
  m->nchunk = E > 0 ? ((E - 1) >> shift) + 1 : 0;
  const int64_t nEnt = T.nEnt();
  std::vector<int64_t> cnt(E + 1, 0);
  std::vector<int64_t> fpos(nEnt, -1), fmin(nEnt, 0);
  for (int64_t x = 0; x < nEnt; ++x) {
    const int c0 = T.ent_ptr[x], c1 = T.ent_ptr[x + 1];
    if (!(c1 - c0 > 1 || (T.ent_flags[x] & kEntMasked))) continue;
    if (T.ent_flags[x] & kEntInterface) continue;  // finished by the interface exchange
    int64_t last = -1, first = INT64_MAX;
    for (int c = c0; c < c1; ++c) {
      const int64_t p = pos[T.ent_copy[c] >> 8];
      last = std::max(last, p);
      first = std::min(first, p);
    }
    fpos[x] = last;
    fmin[x] = first >> shift;
    cnt[last + 1]++;
  }
  for (int64_t f = 0; f < E; ++f) cnt[f + 1] += cnt[f];
  // chunk of each entity = chunk of its last copy; lowest chunk holding a copy
  m->chunk_c0.assign(m->nchunk, 0);
  for (int64_t c = 0; c < m->nchunk; ++c) m->chunk_c0[c] = c;
  std::vector<int64_t> nfc(m->nchunk + 1, 0), nec(m->nchunk + 1, 0), nvc(m->nchunk + 1, 0);
  for (int64_t x = 0; x < nEnt; ++x) {
    if (fpos[x] < 0) continue;
    const int64_t c = fpos[x] >> shift;
    m->chunk_c0[c] = std::min(m->chunk_c0[c], fmin[x]);
    (x < T.nF ? nfc : (x < T.nF + T.nEd ? nec : nvc))[c + 1]++;
  }
  for (int64_t c = 0; c < m->nchunk; ++c) {
    nfc[c + 1] += nfc[c];
    nec[c + 1] += nec[c];
    nvc[c + 1] += nvc[c];
  }
  m->chunk_f = nfc;
  m->chunk_e = nec;
  m->chunk_v = nvc;
  std::vector<int64_t> fdesc(2 * (size_t)nfc[m->nchunk]);
  std::vector<int32_t> eents(nec[m->nchunk]), vents(nvc[m->nchunk]);
  {
    std::vector<int64_t> ff(nfc.begin(), nfc.end() - 1), fe(nec.begin(), nec.end() - 1),
        fv(nvc.begin(), nvc.end() - 1);
    for (int64_t x = 0; x < nEnt; ++x) {  // ascending x keeps entities in creation (element) order
      if (fpos[x] < 0) continue;
      const int64_t c = fpos[x] >> shift;
      if (x < T.nF) {
        const int c0c = T.ent_ptr[x], mult = T.ent_ptr[x + 1] - c0c;
        const int64_t q = ff[c]++;
        fdesc[2 * q] = T.ent_copy[c0c] | ((T.ent_flags[x] & kEntMasked) ? kFaceMasked : 0);
        fdesc[2 * q + 1] = mult > 1 ? T.ent_copy[c0c + 1] : -1;
      } else if (x < T.nF + T.nEd) {
        eents[fe[c]++] = (int32_t)x;
      } else {
        vents[fv[c]++] = (int32_t)x;
      }
    }
  }
  auto up = [&](auto** d, const auto& h) -> sem_status {
    using V = typename std::remove_reference<decltype(h)>::type::value_type;
    if (*d) cudaFree(*d);
    *d = nullptr;
    if (h.empty()) return SEM_OK;
    if (cudaMalloc((void**)d, sizeof(V) * h.size()) != cudaSuccess) return fail(SEM_ENOMEM, "cudaMalloc(gs plan)");
    if (cudaMemcpy(*d, h.data(), sizeof(V) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SEM_ECUDA, "upload gs plan");
    return SEM_OK;
  };
  SEM_TRY(up(&m->d_fdesc, fdesc));
  SEM_TRY(up(&m->d_eents, eents));
  SEM_TRY(up(&m->d_vents, vents));
  // nodal plan: the same entities, one group per node, offsets precomputed
  m->gs_nodal = true;
  if (const char* env = getenv("SEM_GS_NODAL")) m->gs_nodal = atoi(env) != 0;  // tuning knob
  if ((uint64_t)E * (uint64_t)m->n3 >= (uint64_t(1) << 32)) m->gs_nodal = false;  // uint32 offsets
  m->gs_cls.assign(m->nchunk, {});
  if (m->gs_nodal) {
    int maxm = 1;
    for (int64_t x = 0; x < nEnt; ++x)
      if (fpos[x] >= 0) maxm = std::max(maxm, T.ent_ptr[x + 1] - T.ent_ptr[x]);
    const int ncls = 2 * maxm;  // class (m, masked) -> 2 (m - 1) + masked
    std::vector<int64_t> gcount((size_t)m->nchunk * ncls, 0);
    for (int64_t x = 0; x < nEnt; ++x) {
      if (fpos[x] < 0) continue;
      const int mult = T.ent_ptr[x + 1] - T.ent_ptr[x];
      const int cl = 2 * (mult - 1) + ((T.ent_flags[x] & kEntMasked) ? 1 : 0);
      gcount[(size_t)(fpos[x] >> shift) * ncls + cl] += T.ent_nodes(x);
    }
    std::vector<int64_t> cbase(gcount.size(), 0), cfill(gcount.size(), 0);
    int64_t total = 0;
    for (int64_t c = 0; c < m->nchunk; ++c)
      for (int cl = 0; cl < ncls; ++cl) {
        const size_t k = (size_t)c * ncls + cl;
        if (gcount[k] == 0) continue;
        if (cl / 2 + 1 == 2) total = (total + 1) & ~int64_t(1);  // pair classes: 8-byte aligned
        cbase[k] = total;
        GsClass g;
        g.base = total;
        g.count = gcount[k];
        g.m = cl / 2 + 1;
        g.masked = cl & 1;
        m->gs_cls[c].push_back(g);
        total += g.count * g.m;
      }
    std::vector<uint32_t> gidx((size_t)total);
    for (int64_t x = 0; x < nEnt; ++x) {  // ascending x: creation (element) order
      if (fpos[x] < 0) continue;
      const int c0c = T.ent_ptr[x], mult = T.ent_ptr[x + 1] - c0c;
      const size_t k = (size_t)(fpos[x] >> shift) * ncls + 2 * (mult - 1) + ((T.ent_flags[x] & kEntMasked) ? 1 : 0);
      for (int n = 0; n < T.ent_nodes(x); ++n) {
        const int64_t g = cfill[k]++;
        for (int cc = 0; cc < mult; ++cc) {
          const int64_t cp = T.ent_copy[c0c + cc];
          gidx[(size_t)(cbase[k] + cc * gcount[k] + g)] =
              (uint32_t)((cp >> 8) * m->n3 + copy_node_offset(m->lx, (int)((cp >> 3) & 31), (int)(cp & 7), n));
        }
      }
    }
    // groups of a class in the order of their first copy's offset, so the
    // lanes of a warp touch few sectors
    for (int64_t c = 0; c < m->nchunk; ++c)
      for (const GsClass& g : m->gs_cls[c]) {
        std::vector<int64_t> ord((size_t)g.count);
        for (int64_t q = 0; q < g.count; ++q) ord[(size_t)q] = q;
        const uint32_t* first = gidx.data() + g.base;
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return first[a] < first[b]; });
        // m = 2 (faces): the pair interleaved, one 8-byte load per group;
        // else struct of arrays (coalesced per copy)
        std::vector<uint32_t> tmp((size_t)(g.count * g.m));
        for (int k = 0; k < g.m; ++k)
          for (int64_t q = 0; q < g.count; ++q)
            tmp[(size_t)(g.m == 2 ? 2 * q + k : k * g.count + q)] =
                gidx[(size_t)(g.base + k * g.count + ord[(size_t)q])];
        std::copy(tmp.begin(), tmp.end(), gidx.begin() + g.base);
      }
    SEM_TRY(up(&m->d_gidx, gidx));
  }
  if (!m->aux_stream && cudaStreamCreateWithFlags(&m->aux_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SEM_ECUDA, "cudaStreamCreate(aux)");
  // the gather-scatter stream gets the highest priority: its CTAs take the
  // first free SM slots, so a chunk is summed while its w is still in L2
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char* env = getenv("SEM_GS_PRIO")) if (atoi(env) == 0) prio_hi = prio_lo;  // tuning knob
  if (!m->gs_stream && cudaStreamCreateWithPriority(&m->gs_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess)
    return fail(SEM_ECUDA, "cudaStreamCreate(gs)");
  if (m->comm && !m->bnd_stream) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&m->bnd_stream, cudaStreamNonBlocking, hi) != cudaSuccess)
      return fail(SEM_ECUDA, "cudaStreamCreate(boundary)");
  }
  for (auto ev : m->ev_ax) cudaEventDestroy(ev);
  m->ev_ax.assign(m->nchunk, nullptr);
  for (auto& ev : m->ev_ax)
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return fail(SEM_ECUDA, "event");
  for (cudaEvent_t* ev : {&m->ev_start, &m->ev_aux, &m->ev_gs, &m->ev_cap, &m->ev_bnd, &m->ev_input})
    if (!*ev && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) return fail(SEM_ECUDA, "event");
  if (!m->cap_stream && cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SEM_ECUDA, "cudaStreamCreate(cap)");
  return SEM_OK;
}

// mask . dssum(A_e u) (cg: the CG-fused operator) over all positions.
// Default schedule: the operator over all elements, then one gather-scatter
// pass (fuse_pap: which also reduces the CG's pAp partials); with several
// ranks the boundary elements and the exchange start run on a high-priority
// stream beside the interior launch.  SEM_GS_OVERLAP=1: the chunk pipeline
// (chunk c's operator on lane c % 2, its gather-scatter on gs_stream once
// every chunk holding a copy is done).
template <class ChunkFn>
static sem_status ax_dssum_chunks(sem_mesh* m, double* w, ChunkFn launch_chunk, cudaStream_t s,
                                  bool* fuse_pap = nullptr);

static sem_status ax_dssum_all(sem_mesh* m, const AxArgs& a, bool cg, cudaStream_t s) {
  return ax_dssum_chunks(
      m, a.w, [&](int64_t q0, int64_t n, cudaStream_t lane) { return launch_ax_range(m, a, cg, q0, n, lane); },
      s, cg ? a.pap_fused : nullptr);
}

// the schedules for any element-local operator kernel writing w
template <class ChunkFn>
static sem_status ax_dssum_chunks(sem_mesh* m, double* w, ChunkFn launch_chunk, cudaStream_t s, bool* fuse_pap) {
  AxArgs a{};
  a.w = w;
  const int64_t K = m->nchunk;
  if (K == 0) {  // an empty rank still takes part in the collective exchange
    if (m->comm) {
      SEM_TRY(comm_exchange_begin(m, a.w, s));
      SEM_TRY(comm_exchange_end(m, a.w, 3, s));
    }
    return SEM_OK;
  }
  const int64_t cb = (std::max<int64_t>(m->n_boundary, 1) - 1) >> m->chunk_shift;  // boundary chunk
  if (!m->gs_overlap && m->comm && m->xp2p && m->n_boundary < m->E && m->bnd_stream) {
    // several ranks over peer memory: the boundary elements, then their
    // interface partials and the stores into the peers, run on a
    // high-priority stream while the interior launch fills the rest of the
    // GPU on `s` (no tail bubble between the two launches, and the small
    // exchange kernels off the critical path); the local gather-scatter
    // waits for the boundary launch, the unpack for the stores
    const int64_t qb = std::min(m->E, (cb + 1) << m->chunk_shift);
    SEM_CUDA_TRY(cudaEventRecord(m->ev_start, s));
    SEM_CUDA_TRY(cudaStreamWaitEvent(m->bnd_stream, m->ev_start, 0));
    SEM_CUDA_TRY(launch_chunk(0, qb, m->bnd_stream));
    SEM_CUDA_TRY(cudaEventRecord(m->ev_bnd, m->bnd_stream));
    SEM_TRY(comm_exchange_begin(m, a.w, m->bnd_stream));
    SEM_CUDA_TRY(cudaEventRecord(m->ev_pack, m->bnd_stream));
    SEM_CUDA_TRY(launch_chunk(qb, m->E - qb, s));
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_bnd, 0));
    SEM_CUDA_TRY(launch_gs_flat(m, a.w, 0, K, 3, s, fuse_pap));
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_pack, 0));
    SEM_TRY(comm_exchange_end(m, a.w, 3, s));
    return SEM_OK;
  }
  if (!m->gs_overlap) {
    // one launch up to the end of the boundary chunk, one for the rest
    const int64_t qb = m->comm ? std::min(m->E, (cb + 1) << m->chunk_shift) : m->E;
    SEM_CUDA_TRY(launch_chunk(0, qb, s));
    if (m->comm) SEM_TRY(comm_exchange_begin(m, a.w, s));
    if (qb < m->E) SEM_CUDA_TRY(launch_chunk(qb, m->E - qb, s));
    SEM_CUDA_TRY(launch_gs_flat(m, a.w, 0, K, 3, s, fuse_pap));
    if (m->comm) SEM_TRY(comm_exchange_end(m, a.w, 3, s));
    return SEM_OK;
  }
  SEM_CUDA_TRY(cudaEventRecord(m->ev_start, s));
  SEM_CUDA_TRY(cudaStreamWaitEvent(m->aux_stream, m->ev_start, 0));
  SEM_CUDA_TRY(cudaStreamWaitEvent(m->gs_stream, m->ev_start, 0));
  for (int64_t c = 0; c < K; ++c) {
    cudaStream_t lane = (m->lanes == 2 && (c & 1)) ? m->aux_stream : s;
    const int64_t q0 = c << m->chunk_shift, q1 = std::min(m->E, (c + 1) << m->chunk_shift);
    SEM_CUDA_TRY(launch_chunk(q0, q1 - q0, lane));
    SEM_CUDA_TRY(cudaEventRecord(m->ev_ax[c], lane));
    for (int64_t d = m->chunk_c0[c]; d <= c; ++d) SEM_CUDA_TRY(cudaStreamWaitEvent(m->gs_stream, m->ev_ax[d], 0));
    SEM_CUDA_TRY(launch_gs_flat(m, a.w, c, c + 1, 3, m->gs_stream));
    // every element touching the interface is done: partial sums of the
    // interface entities go out over NVLink while the interior is computed
    if (m->comm && c == cb) {
      for (int64_t d = 0; d < c; ++d) SEM_CUDA_TRY(cudaStreamWaitEvent(lane, m->ev_ax[d], 0));
      SEM_TRY(comm_exchange_begin(m, a.w, lane));
    }
  }
  SEM_CUDA_TRY(cudaEventRecord(m->ev_aux, m->aux_stream));
  SEM_CUDA_TRY(cudaEventRecord(m->ev_gs, m->gs_stream));
  SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_aux, 0));
  SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_gs, 0));
  if (m->comm) SEM_TRY(comm_exchange_end(m, a.w, 3, s));
  return SEM_OK;
}

extern "C" {

const char* sem_version(void) { return "semb200 0.1 sm_100a"; }

const char* sem_last_error(void) { return g_err.c_str(); }

sem_status sem_gll(int N, double* xi, double* w) {
  if (!xi || !w) return fail(SEM_EINVAL, "sem_gll: NULL output");
  if (N < 1 || N > 15) return fail(SEM_EINVAL, "sem_gll: N must be in [1, 15]");
  if (!gll_golub_welsch(N, xi, w)) return fail(SEM_EINVAL, "sem_gll: eigen-solver failed");
  return SEM_OK;
}

static void mesh_free(sem_mesh* m) {
  if (!m) return;
  comm_mesh_free(m);
  ulayout_free(m);
  void* ptrs[] = {m->d_gaff, m->coords, m->G, m->B, m->mult, m->mask, m->m8, m->d_elem_ent, m->d_ent_ptr, m->d_ent_copy,
                  m->d_ent_flags, m->d_ent_cnt, m->d_elist_all, m->r, m->p, m->w, m->dinv, m->xw, m->bw,
                  m->part, m->ticket, m->sc, m->s_cg};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (m->sc_host) cudaFreeHost(m->sc_host);
  void* fp[] = {m->d_fdesc, m->d_eents, m->d_vents, m->d_gidx};
  for (void* p : fp)
    if (p) cudaFree(p);
  for (auto ev : m->ev_ax) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {m->ev_start, m->ev_aux, m->ev_gs, m->ev_cap, m->ev_bnd, m->ev_input})
    if (ev) cudaEventDestroy(ev);
  if (m->bnd_stream) cudaStreamDestroy(m->bnd_stream);
  if (m->aux_stream) cudaStreamDestroy(m->aux_stream);
  if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
  if (m->gs_stream) cudaStreamDestroy(m->gs_stream);
  for (auto ev : m->prof_ev) cudaEventDestroy(ev);
  delete m;
}

void sem_mesh_destroy(sem_mesh_t m) { mesh_free(m); }

sem_status sem_mesh_create(int64_t E, int N, const double* coords, const int64_t* conn, const int8_t* bc,
                           sem_comm_t comm, sem_mesh_t* out) {
  if (!out) return fail(SEM_EINVAL, "sem_mesh_create: out is NULL");
  *out = nullptr;
  if (E < 0) return fail(SEM_EINVAL, "sem_mesh_create: E < 0");
  if (N < 1 || N > kMaxN) return fail(SEM_EINVAL, "sem_mesh_create: N must be in [1, 11]");
  if (E > 0 && (!coords || !conn)) return fail(SEM_EINVAL, "sem_mesh_create: NULL coords or conn");
  if (E >= (int64_t(1) << 31)) return fail(SEM_EINVAL, "sem_mesh_create: too many elements");
  sem_mesh* m = new (std::nothrow) sem_mesh();
  if (!m) return fail(SEM_ENOMEM, "sem_mesh_create: host allocation");
  m->E = E;
  m->N = N;
  m->lx = N + 1;
  m->n3 = m->lx * m->lx * m->lx;
  m->n3p = (m->n3 + 1) & ~1;
  m->nloc = E * m->n3;
  m->comm = comm;
  cudaGetDevice(&m->device);
  // basis
  double xi[kMaxN + 1], w[kMaxN + 1], D[(kMaxN + 1) * (kMaxN + 1)];
  gll_golub_welsch(N, xi, w);
  deriv_matrix(N, xi, D);
  cudaError_t ce = upload_basis(N, D, w);
  if (ce != cudaSuccess) {
    mesh_free(m);
    return fail(SEM_ECUDA, std::string("upload_basis: ") + cudaGetErrorString(ce));
  }
  // topology
  std::string err = build_topology(E, N, conn, bc, &m->topo);
  if (!err.empty()) {
    mesh_free(m);
    return fail(SEM_EINVAL, "sem_mesh_create: " + err);
  }
  std::vector<int64_t> pos(E);
  for (int64_t e = 0; e < E; ++e) pos[e] = e;
  if (comm) {
    sem_status stc = comm_plan_interface(m, &pos);
    if (stc != SEM_OK) {
      mesh_free(m);
      return stc;
    }
  }
  const Topology& T = m->topo;
  const int64_t mm = m->lx - 2;
  m->n_unique = T.nV + T.nEd * mm + T.nF * mm * mm + E * mm * mm * mm;
  m->n_masked = 0;
  for (int64_t x = 0; x < T.nEnt(); ++x)
    if (T.ent_flags[x] & kEntMasked) m->n_masked += (int64_t)T.ent_nodes(x) * (T.ent_ptr[x + 1] - T.ent_ptr[x]);
  m->n_masked_glob = m->n_masked;
  // device arrays
  sem_status st;
#define ALLOC(p, n, what)                  \
  if ((st = dalloc(&(p), (n), what)) != SEM_OK) { \
    mesh_free(m);                          \
    return st;                             \
  }
  ALLOC(m->coords, 3 * m->nloc, "coords");
  ALLOC(m->G, E * 6 * m->n3p, "G");
  ALLOC(m->B, m->nloc, "B");
  ALLOC(m->mult, m->nloc, "mult");
  ALLOC(m->mask, m->nloc, "mask");
  {
    int maxm = 1;  // byte multiplicities only when every count fits (global counts <= 8 ranks x local)
    for (int64_t x = 0; x < T.nEnt(); ++x) maxm = std::max(maxm, T.ent_ptr[x + 1] - T.ent_ptr[x]);
    if (maxm * (comm ? comm->nranks : 1) < 255) ALLOC(m->m8, m->nloc, "multiplicity bytes");
  }
  ALLOC(m->d_elem_ent, E * kSlots, "elem_ent");
  ALLOC(m->d_ent_ptr, T.nEnt() + 1, "ent_ptr");
  ALLOC(m->d_ent_copy, (int64_t)T.ent_copy.size(), "ent_copy");
  ALLOC(m->d_ent_flags, T.nEnt(), "ent_flags");
  ALLOC(m->d_ent_cnt, T.nEnt(), "ent_cnt");
  m->npart = part_capacity(E);
  ALLOC(m->part, m->npart, "partials");
  ALLOC(m->ticket, 4, "ticket");
  ALLOC(m->sc, 1, "scalars");
  if (comm) ALLOC(m->d_elist_all, E, "element order");
#undef ALLOC
  if (cudaMallocHost((void**)&m->sc_host, sizeof(CGScalars)) != cudaSuccess) {
    mesh_free(m);
    return fail(SEM_ENOMEM, "cudaMallocHost(scalars)");
  }
  auto up = [&](void* d, const void* h, size_t bytes) -> cudaError_t {
    return bytes ? cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  cudaError_t e1 = up(m->coords, coords, sizeof(double) * 3 * m->nloc);
  if (e1 == cudaSuccess) e1 = up(m->d_elem_ent, T.elem_ent.data(), sizeof(int32_t) * T.elem_ent.size());
  if (e1 == cudaSuccess) e1 = up(m->d_ent_ptr, T.ent_ptr.data(), sizeof(int32_t) * T.ent_ptr.size());
  if (e1 == cudaSuccess) e1 = up(m->d_ent_copy, T.ent_copy.data(), sizeof(int64_t) * T.ent_copy.size());
  if (e1 == cudaSuccess) e1 = up(m->d_ent_flags, T.ent_flags.data(), T.ent_flags.size());
  if (e1 == cudaSuccess && m->d_elist_all) {
    std::vector<int32_t> order(E);
    for (int64_t e = 0; e < E; ++e) order[pos[e]] = (int32_t)e;
    e1 = up(m->d_elist_all, order.data(), sizeof(int32_t) * E);
  }
  if (e1 == cudaSuccess && T.nEnt() > 0) e1 = cudaMemset(m->d_ent_cnt, 0, sizeof(uint32_t) * T.nEnt());
  if (e1 == cudaSuccess) e1 = cudaMemset(m->ticket, 0, sizeof(unsigned) * 4);
  if (e1 == cudaSuccess) e1 = cudaMemset(m->sc, 0, sizeof(CGScalars));
  if (e1 == cudaSuccess && m->nloc > 0) e1 = launch_mult_mask(m, 0);
  if (e1 == cudaSuccess) e1 = cudaDeviceSynchronize();
  if (e1 != cudaSuccess) {
    mesh_free(m);
    return fail(SEM_ECUDA, std::string("sem_mesh_create upload: ") + cudaGetErrorString(e1));
  }
  st = build_gs_lists(m, pos);
  if (st != SEM_OK) {
    mesh_free(m);
    return st;
  }
  m->cg_unique = false;  // local layout measured faster
  if (const char* env = getenv("SEM_CG_LAYOUT")) m->cg_unique = std::string(env) == "unique";  // tuning knob
  m->cg_pipelined = false;
  if (const char* env = getenv("SEM_CG_VARIANT")) m->cg_pipelined = std::string(env) == "pipelined";
  if (comm) {
    st = comm_setup_device(m);
    if (st != SEM_OK) {
      mesh_free(m);
      return st;
    }
  }
  st = build_ulayout(m, pos);
  if (st != SEM_OK) {
    mesh_free(m);
    return st;
  }
  *out = m;
  return SEM_OK;
}

sem_status sem_mesh_info(sem_mesh_t m, sem_mesh_info_t* info) {
  if (!m || !info) return fail(SEM_EINVAL, "sem_mesh_info: NULL argument");
  info->E = m->E;
  info->N = m->N;
  info->lx = m->lx;
  info->n_local = m->nloc;
  info->n_unique = m->n_unique;
  info->n_entities = m->topo.nEnt();
  info->n_masked = m->n_masked;
  info->n_interface = m->n_interface;
  info->n_boundary_elements = m->n_boundary;
  info->rank = m->comm ? m->comm->rank : 0;
  info->nranks = m->comm ? m->comm->nranks : 1;
  info->n_peers = (int)m->iface.peers.size();
  info->affine = m->affine ? 1 : 0;
  return SEM_OK;
}

sem_status sem_mesh_global_ids(sem_mesh_t m, int64_t* ids) {
  if (!m || (!ids && m->E > 0)) return fail(SEM_EINVAL, "sem_mesh_global_ids: NULL argument");
  const Topology& T = m->topo;
  const int lx = m->lx, mm = lx - 2, n3 = m->n3;
  const int64_t baseE = T.nV, baseF = baseE + T.nEd * mm, baseI = baseF + T.nF * mm * mm;
  for (int64_t e = 0; e < m->E; ++e) {
    int64_t* o = ids + e * n3;
    for (int k = 1; k < lx - 1; ++k)
      for (int j = 1; j < lx - 1; ++j)
        for (int i = 1; i < lx - 1; ++i)
          o[i + lx * (j + lx * k)] = baseI + e * (int64_t)mm * mm * mm + (i - 1) + mm * ((j - 1) + mm * (k - 1));
    for (int s = 0; s < kSlots; ++s) {
      const int32_t ent = T.elem_ent[e * kSlots + s];
      // find this copy's orientation
      int orient = 0;
      for (int c = T.ent_ptr[ent]; c < T.ent_ptr[ent + 1]; ++c) {
        const int64_t cp = T.ent_copy[c];
        if ((cp >> 8) == e && (int)((cp >> 3) & 31) == s) orient = (int)(cp & 7);
      }
      const int nn = T.ent_nodes(ent);
      for (int n = 0; n < nn; ++n) {
        const int off = copy_node_offset(lx, s, orient, n);
        int64_t gid;
        if (ent < T.nF) gid = baseF + (int64_t)ent * mm * mm + n;
        else if (ent < T.nF + T.nEd) gid = baseE + (int64_t)(ent - T.nF) * mm + n;
        else gid = ent - T.nF - T.nEd;
        o[off] = gid;
      }
    }
  }
  return SEM_OK;
}

sem_status sem_geom_factors(sem_mesh_t m) {
  if (!m) return fail(SEM_EINVAL, "sem_geom_factors: NULL mesh");
  if (m->E == 0) {
    m->has_geom = true;
    return SEM_OK;
  }
  unsigned long long* bad = nullptr;
  SEM_CUDA_TRY(cudaMalloc((void**)&bad, sizeof(unsigned long long)));
  unsigned long long init = ~0ull, hb = 0;
  cudaMemcpy(bad, &init, sizeof(init), cudaMemcpyHostToDevice);
  cudaError_t e = launch_geom_bad(m, bad, 0);
  if (e == cudaSuccess) e = cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  if (e != cudaSuccess) return fail(SEM_ECUDA, std::string("sem_geom_factors: ") + cudaGetErrorString(e));
  if (hb != ~0ull) return fail(SEM_EINVAL, "sem_geom_factors: J <= 0 in element " + std::to_string(hb));
  m->has_geom = true;
  // affine-element variant (opt-in): all elements affine ->
  // the operator uses six constants per element instead of G per node
  m->affine = false;
  if (const char* env = getenv("SEM_AFFINE")) {
    if (atoi(env) != 0) {
      if (!m->d_gaff) SEM_TRY(dalloc(&m->d_gaff, m->E * 6, "affine constants"));
      int* flag = nullptr;
      SEM_CUDA_TRY(cudaMalloc((void**)&flag, sizeof(int)));
      int hf = 0;
      cudaMemcpy(flag, &hf, sizeof(int), cudaMemcpyHostToDevice);
      e = launch_affine_detect(m, m->d_gaff, flag, 0);
      if (e == cudaSuccess) e = cudaMemcpy(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost);
      cudaFree(flag);
      if (e != cudaSuccess) return fail(SEM_ECUDA, std::string("affine detection: ") + cudaGetErrorString(e));
      m->affine = (hf == 0);
    }
  }
  return SEM_OK;
}

sem_status sem_geom_get(sem_mesh_t m, double* G, double* B) {
  if (!m) return fail(SEM_EINVAL, "sem_geom_get: NULL mesh");
  if (!m->has_geom) return fail(SEM_EINVAL, "sem_geom_get: call sem_geom_factors first");
  if (m->E == 0) return SEM_OK;
  if (G)
    SEM_CUDA_TRY(cudaMemcpy2D(G, sizeof(double) * m->n3, m->G, sizeof(double) * m->n3p, sizeof(double) * m->n3,
                              (size_t)m->E * 6, cudaMemcpyDeviceToDevice));
  if (B) SEM_CUDA_TRY(cudaMemcpy(B, m->B, sizeof(double) * m->nloc, cudaMemcpyDeviceToDevice));
  return SEM_OK;
}

sem_status sem_mult_mask_get(sem_mesh_t m, double* mult, double* mask) {
  if (!m) return fail(SEM_EINVAL, "sem_mult_mask_get: NULL mesh");
  if (m->nloc == 0) return SEM_OK;
  if (mult) SEM_CUDA_TRY(cudaMemcpy(mult, m->mult, sizeof(double) * m->nloc, cudaMemcpyDeviceToDevice));
  if (mask) SEM_CUDA_TRY(cudaMemcpy(mask, m->mask, sizeof(double) * m->nloc, cudaMemcpyDeviceToDevice));
  return SEM_OK;
}

static sem_status check_op(sem_mesh_t m, const void* u, const void* w, const char* who) {
  if (!m) return fail(SEM_EINVAL, std::string(who) + ": NULL mesh");
  if (!m->has_geom) return fail(SEM_EINVAL, std::string(who) + ": call sem_geom_factors first");
  if (m->nloc > 0 && (!u || !w)) return fail(SEM_EINVAL, std::string(who) + ": NULL field");
  if (u && u == w) return fail(SEM_EINVAL, std::string(who) + ": u and w must not alias");
  return SEM_OK;
}

static void prof_begin(sem_mesh* m, cudaStream_t s, cudaEvent_t* ev) {
  ev[0] = ev[1] = nullptr;
  if (!m->prof) return;
  cudaEventCreate(&ev[0]);
  cudaEventCreate(&ev[1]);
  cudaEventRecord(ev[0], s);
}
static void prof_end(sem_mesh* m, cudaStream_t s, cudaEvent_t* ev) {
  if (!m->prof || !ev[0]) return;
  cudaEventRecord(ev[1], s);
  m->prof_ev.push_back(ev[0]);
  m->prof_ev.push_back(ev[1]);
}

sem_status sem_ax(sem_mesh_t m, const double* u, double* w, const double* h1, const double* h2, double h1c,
                  double h2c, sem_stream_t stream) {
  SEM_TRY(check_op(m, u, w, "sem_ax"));
  AxArgs a{};
  a.u = u;
  a.w = w;
  a.h1 = h1;
  a.h2 = h2;
  a.h1c = h1c;
  a.h2c = h2c;
  SEM_CUDA_TRY(launch_ax_range(m, a, false, 0, m->E, (cudaStream_t)stream));
  return SEM_OK;
}

sem_status sem_gs_op(sem_mesh_t m, double* u, int op, sem_stream_t stream) {
  if (!m) return fail(SEM_EINVAL, "sem_gs_op: NULL mesh");
  if (op != SEM_GS_ADD && op != SEM_GS_MASK) return fail(SEM_EINVAL, "sem_gs_op: unknown op");
  if (m->nloc > 0 && !u) return fail(SEM_EINVAL, "sem_gs_op: NULL field");
  cudaStream_t s = (cudaStream_t)stream;
  if (m->nchunk > 0)
    SEM_CUDA_TRY(launch_gs_flat(m, u, 0, m->nchunk, op == SEM_GS_ADD ? 1 : 2, s));
  if (m->comm) SEM_TRY(comm_gs_exchange(m, u, op == SEM_GS_ADD ? 1 : 2, s));
  return SEM_OK;
}

sem_status sem_ax_dssum(sem_mesh_t m, const double* u, double* w, const double* h1, const double* h2,
                        double h1c, double h2c, sem_stream_t stream) {
  SEM_TRY(check_op(m, u, w, "sem_ax_dssum"));
  cudaStream_t s = (cudaStream_t)stream;
  AxArgs a{};
  a.u = u;
  a.w = w;
  a.h1 = h1;
  a.h2 = h2;
  a.h1c = h1c;
  a.h2c = h2c;
  cudaEvent_t ev[2];
  prof_begin(m, s, ev);
  SEM_TRY(ax_dssum_all(m, a, false, s));
  prof_end(m, s, ev);
  return SEM_OK;
}

sem_status sem_rhs(sem_mesh_t m, const double* f, double* b, sem_stream_t stream) {
  if (!m) return fail(SEM_EINVAL, "sem_rhs: NULL mesh");
  if (!m->has_geom) return fail(SEM_EINVAL, "sem_rhs: call sem_geom_factors first");
  if (m->nloc > 0 && (!f || !b)) return fail(SEM_EINVAL, "sem_rhs: NULL field");
  cudaStream_t s = (cudaStream_t)stream;
  SEM_CUDA_TRY(launch_rhs_local(m, f, b, s));
  SEM_TRY(sem_gs_op(m, b, SEM_GS_ADD, stream));
  SEM_TRY(sem_gs_op(m, b, SEM_GS_MASK, stream));
  return SEM_OK;
}

sem_status sem_jacobi(sem_mesh_t m, const double* h1, const double* h2, double h1c, double h2c, double* dinv,
                      sem_stream_t stream) {
  if (!m) return fail(SEM_EINVAL, "sem_jacobi: NULL mesh");
  if (!m->has_geom) return fail(SEM_EINVAL, "sem_jacobi: call sem_geom_factors first");
  if (m->nloc > 0 && !dinv) return fail(SEM_EINVAL, "sem_jacobi: NULL output");
  cudaStream_t s = (cudaStream_t)stream;
  SEM_CUDA_TRY(launch_diag(m, h1, h2, h1c, h2c, dinv, s));
  SEM_TRY(sem_gs_op(m, dinv, SEM_GS_ADD, stream));
  SEM_CUDA_TRY(launch_invert_diag(m, dinv, s));
  return SEM_OK;
}

static sem_status ensure_cg(sem_mesh* m) {
  sem_status st;
  if (!m->r && (st = dalloc(&m->r, m->nloc, "cg r")) != SEM_OK) return st;
  if (!m->p && (st = dalloc(&m->p, m->nloc, "cg p")) != SEM_OK) return st;
  if (!m->w && (st = dalloc(&m->w, m->nloc, "cg w")) != SEM_OK) return st;
  if (!m->dinv && (st = dalloc(&m->dinv, m->nloc, "cg dinv")) != SEM_OK) return st;
  return SEM_OK;
}

static sem_status allreduce(sem_mesh* m, double* d, int n, cudaStream_t s) {
  if (!m->comm) return SEM_OK;
  return comm_allreduce_sum(m, d, n, s);
}

// U-layout operator for the CG (ax_u.cu): chunk c's operator on lane c % 2,
// the segmented sum of the entities finished in chunk c on gs_stream, and
// the interface exchange started as soon as every boundary element is done.
static sem_status ax_dssum_u(sem_mesh* m, const AxArgs& a, cudaStream_t s) {
  const int64_t K = m->nchunk;
  if (K == 0) {
    if (m->comm) {
      SEM_TRY(comm_exchange_begin_u(m, s));
      SEM_TRY(comm_exchange_end_u(m, s));
    }
    return SEM_OK;
  }
  SEM_CUDA_TRY(cudaEventRecord(m->ev_start, s));
  SEM_CUDA_TRY(cudaStreamWaitEvent(m->aux_stream, m->ev_start, 0));
  SEM_CUDA_TRY(cudaStreamWaitEvent(m->gs_stream, m->ev_start, 0));
  const int64_t cb = (std::max<int64_t>(m->n_boundary, 1) - 1) >> m->chunk_shift;
  for (int64_t c = 0; c < K; ++c) {
    cudaStream_t lane = (m->lanes == 2 && (c & 1)) ? m->aux_stream : s;
    const int64_t q0 = c << m->chunk_shift, q1 = std::min(m->E, (c + 1) << m->chunk_shift);
    SEM_CUDA_TRY(launch_ax_u(m, a, q0, q1 - q0, lane));
    SEM_CUDA_TRY(cudaEventRecord(m->ev_ax[c], lane));
    for (int64_t d = m->chunk_c0[c]; d <= c; ++d) SEM_CUDA_TRY(cudaStreamWaitEvent(m->gs_stream, m->ev_ax[d], 0));
    SEM_CUDA_TRY(launch_segsum(m, c, c + 1, m->gs_stream));
    if (m->comm && c == cb) {
      for (int64_t d = 0; d < c; ++d) SEM_CUDA_TRY(cudaStreamWaitEvent(lane, m->ev_ax[d], 0));
      SEM_TRY(comm_exchange_begin_u(m, lane));
    }
  }
  SEM_CUDA_TRY(cudaEventRecord(m->ev_aux, m->aux_stream));
  SEM_CUDA_TRY(cudaEventRecord(m->ev_gs, m->gs_stream));
  SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_aux, 0));
  SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_gs, 0));
  if (m->comm) SEM_TRY(comm_exchange_end_u(m, s));
  return SEM_OK;
}

static sem_status ensure_cg_u(sem_mesh* m) {
  sem_status st;
  double** vs[] = {&m->ux, &m->ur, &m->up, &m->uw, &m->udinv};
  for (double** v : vs)
    if (!*v) {
      if ((st = dalloc(v, std::max<int64_t>(m->n_u, 1), "cg U vector")) != SEM_OK) return st;
      SEM_CUDA_TRY(cudaMemset(*v, 0, sizeof(double) * std::max<int64_t>(m->n_u, 1)));  // pads stay 0
    }
  return SEM_OK;
}

static sem_status cg_solve_u(sem_mesh* m, const double* b, double* x, const double* h1, const double* h2,
                             double h1c, double h2c, double tol, int maxit, int* iters, double* rel_res,
                             int* converged, cudaStream_t s) {
  SEM_TRY(ensure_cg(m));
  SEM_TRY(ensure_cg_u(m));
  double nz_h2 = (h2 == nullptr) ? (h2c != 0.0 ? 1.0 : 0.0) : 0.0;
  SEM_CUDA_TRY(cudaMemsetAsync(m->sc, 0, sizeof(CGScalars), s));
  if (h2) {
    SEM_CUDA_TRY(launch_count_nonzero(h2, m->nloc, m, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
    nz_h2 = m->sc_host->red[3];
  }
  const int singular = (m->n_masked_glob == 0) && (nz_h2 == 0.0);
  // Jacobi (local layout, then to U), r = mask b, x = p = 0
  SEM_TRY(sem_jacobi(m, h1, h2, h1c, h2c, m->dinv, (sem_stream_t)s));
  SEM_CUDA_TRY(launch_l2u(m, m->dinv, nullptr, m->udinv, s));
  SEM_CUDA_TRY(launch_l2u(m, b, m->mask, m->ur, s));
  SEM_CUDA_TRY(launch_zero2(m, m->ux, m->up, m->n_u, s));
  if (singular) {
    SEM_CUDA_TRY(launch_dot_u(m, m->ur, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean_u(m, m->ur, 3, s));
  }
  CGScalars init{};
  init.tol = tol;
  init.maxit = maxit;
  SEM_CUDA_TRY(cudaMemcpyAsync(&m->sc->tol, &init.tol, sizeof(double), cudaMemcpyHostToDevice, s));
  SEM_CUDA_TRY(cudaMemcpyAsync(&m->sc->maxit, &init.maxit, sizeof(int), cudaMemcpyHostToDevice, s));
  SEM_CUDA_TRY(launch_cg_start_u(m, s));
  SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
  SEM_CUDA_TRY(launch_cg_scalar_step(m, 0, s));
  AxArgs a{};
  a.h1 = h1;
  a.h2 = h2;
  a.h1c = h1c;
  a.h2c = h2c;
  a.part = m->part + pap_part_offset();
  a.x = x;
  m->pap_nparts = m->E;
  const int poll = 8;
  for (int it = 0; it < maxit; ++it) {
    cudaEvent_t ev[2];
    prof_begin(m, s, ev);
    SEM_TRY(ax_dssum_u(m, a, s));
    prof_end(m, s, ev);
    SEM_CUDA_TRY(launch_cg_pap_reduce(m, s));
    SEM_TRY(allreduce(m, &m->sc->red[0], 1, s));
    SEM_CUDA_TRY(launch_cg_update_u(m, s));
    SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
    SEM_CUDA_TRY(launch_cg_scalar_step(m, 1, s));
    if (tol > 0.0 && ((it + 1) % poll == 0)) {
      SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
      SEM_CUDA_TRY(cudaStreamSynchronize(s));
      if (m->sc_host->done) break;
    }
  }
  SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
  SEM_CUDA_TRY(cudaStreamSynchronize(s));
  const CGScalars h = *m->sc_host;
  if (singular && !h.breakdown) {
    SEM_CUDA_TRY(launch_dot_u(m, m->ux, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean_u(m, m->ux, 3, s));
  }
  SEM_CUDA_TRY(launch_u2l(m, m->ux, x, s));
  SEM_CUDA_TRY(cudaStreamSynchronize(s));
  if (iters) *iters = h.iter + (h.breakdown ? 1 : 0);
  if (rel_res) *rel_res = h.bn > 0 ? sqrt(h.rtr) / h.bn : 0.0;
  if (converged) *converged = h.converged;
  if (h.breakdown) return fail(SEM_EBREAKDOWN, "sem_cg_solve: breakdown (pAp <= 0 or NaN)");
  return SEM_OK;
}

// Single-reduction (Chronopoulos-Gear) PCG, ax_p.cu: one fused pass and one
// reduction per iteration.  Same set-up, masking,
// projection and stopping rule as reading R10.
static sem_status cg_solve_pipelined(sem_mesh* m, const double* b, double* x, const double* h1, const double* h2,
                                     double h1c, double h2c, double tol, int maxit, int* iters, double* rel_res,
                                     int* converged, cudaStream_t s) {
  SEM_TRY(ensure_cg(m));
  if (!m->s_cg) {
    sem_status st = dalloc(&m->s_cg, std::max<int64_t>(m->nloc, 1), "cg s");
    if (st != SEM_OK) return st;
  }
  double nz_h2 = (h2 == nullptr) ? (h2c != 0.0 ? 1.0 : 0.0) : 0.0;
  SEM_CUDA_TRY(cudaMemsetAsync(m->sc, 0, sizeof(CGScalars), s));
  if (h2) {
    SEM_CUDA_TRY(launch_count_nonzero(h2, m->nloc, m, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
    nz_h2 = m->sc_host->red[3];
  }
  const int singular = (m->n_masked_glob == 0) && (nz_h2 == 0.0);
  SEM_TRY(sem_jacobi(m, h1, h2, h1c, h2c, m->dinv, (sem_stream_t)s));
  SEM_CUDA_TRY(launch_cg_init(m, b, x, tol, maxit, singular, s));  // r = mask b, x = 0, p = 0
  if (m->nloc > 0) SEM_CUDA_TRY(cudaMemsetAsync(m->s_cg, 0, sizeof(double) * m->nloc, s));
  if (singular) {
    SEM_CUDA_TRY(launch_wdot(m, m->r, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, m->r, 3, s));
  }
  CGScalars init{};
  init.tol = tol;
  init.maxit = maxit;
  SEM_CUDA_TRY(cudaMemcpyAsync(&m->sc->tol, &init.tol, sizeof(double), cudaMemcpyHostToDevice, s));
  SEM_CUDA_TRY(cudaMemcpyAsync(&m->sc->maxit, &init.maxit, sizeof(int), cudaMemcpyHostToDevice, s));
  AxArgs a{};
  a.h1 = h1;
  a.h2 = h2;
  a.h1c = h1c;
  a.h2c = h2c;
  a.part = m->part + pap_part_offset();
  auto pass = [&](int first) -> sem_status {
    cudaEvent_t ev[2];
    prof_begin(m, s, ev);
    SEM_TRY(ax_dssum_chunks(
        m, m->w,
        [&](int64_t q0, int64_t n, cudaStream_t lane) {
          return launch_ax_pcg(m, a, x, m->w, m->w, first, q0, n, lane);
        },
        s));
    prof_end(m, s, ev);
    SEM_CUDA_TRY(launch_reduce3(m, a.part, s));
    SEM_TRY(allreduce(m, &m->sc->red[0], 3, s));
    SEM_CUDA_TRY(launch_pcg_scalar(m, first ? 0 : 1, s));
    return SEM_OK;
  };
  SEM_TRY(pass(1));  // u0 = dinv r0, w0 = A u0, gamma0, delta0, |r0|
  const int poll = 8;
  for (int it = 0; it < maxit; ++it) {
    SEM_TRY(pass(0));
    if (tol > 0.0 && ((it + 1) % poll == 0)) {
      SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
      SEM_CUDA_TRY(cudaStreamSynchronize(s));
      if (m->sc_host->done) break;
    }
  }
  SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
  SEM_CUDA_TRY(cudaStreamSynchronize(s));
  const CGScalars h = *m->sc_host;
  if (singular && !h.breakdown) {
    SEM_CUDA_TRY(launch_wdot(m, x, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, x, 3, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  if (iters) *iters = h.iter + (h.breakdown ? 1 : 0);
  if (rel_res) *rel_res = h.bn > 0 ? sqrt(h.rtr) / h.bn : 0.0;
  if (converged) *converged = h.converged;
  if (h.breakdown) return fail(SEM_EBREAKDOWN, "sem_cg_solve: breakdown (pAp <= 0 or NaN)");
  return SEM_OK;
}

static sem_status cg_solve_impl(sem_mesh* m, const double* b, double* x, const double* h1, const double* h2,
                                double h1c, double h2c, double tol, int maxit, int* iters, double* rel_res,
                                int* converged, cudaStream_t s) {
  SEM_TRY(ensure_cg(m));
  // singular := no masked node anywhere and h2 == 0 everywhere (reading R10)
  int64_t masked = m->n_masked;
  double nz_h2 = (h2 == nullptr) ? (h2c != 0.0 ? 1.0 : 0.0) : 0.0;
  SEM_CUDA_TRY(cudaMemsetAsync(m->sc, 0, sizeof(CGScalars), s));
  if (h2) {
    SEM_CUDA_TRY(launch_count_nonzero(h2, m->nloc, m, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
    nz_h2 = m->sc_host->red[3];
  }
  const int singular = (m->n_masked_glob == 0) && (nz_h2 == 0.0);
  (void)masked;
  // Jacobi preconditioner
  SEM_TRY(sem_jacobi(m, h1, h2, h1c, h2c, m->dinv, (sem_stream_t)s));
  // r = mask b (+ projection), x = 0, p = 0
  if (m->input_pending) {  // sem_cg_solve_host's upload of b
    m->input_pending = false;
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_input, 0));
  }
  SEM_CUDA_TRY(launch_cg_init(m, b, x, tol, maxit, singular, s));
  if (singular) {
    SEM_CUDA_TRY(launch_wdot(m, m->r, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, m->r, 3, s));
  }
  CGScalars init{};
  init.tol = tol;
  init.maxit = maxit;
  init.singular = singular;
  SEM_CUDA_TRY(cudaMemcpyAsync(&m->sc->tol, &init.tol, sizeof(double), cudaMemcpyHostToDevice, s));
  SEM_CUDA_TRY(cudaMemcpyAsync(&m->sc->maxit, &init.maxit, sizeof(int), cudaMemcpyHostToDevice, s));
  SEM_CUDA_TRY(launch_cg_start(m, s));
  SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
  SEM_CUDA_TRY(launch_cg_scalar_step(m, 0, s));
  AxArgs a{};
  a.u = nullptr;
  a.w = m->w;
  a.h1 = h1;
  a.h2 = h2;
  a.h1c = h1c;
  a.h2c = h2c;
  a.r = m->r;
  a.dinv = m->dinv;
  a.p = m->p;
  a.sc = m->sc;
  a.part = m->part + pap_part_offset();
  a.x = x;
  m->pap_nparts = m->E;
  const int poll = 8;
  // one iteration: fused operator (events around it when profiling), pAp,
  // update, scalars -- captured once into a CUDA graph (all streams joined
  // by events, NCCL included) and replayed, unless SEM_GRAPH=0
  // one rank, or several over NVLink peer memory: the pAp reduction (and its
  // allreduce) rides in the gs launch and the rtr/rtz allreduce plus the
  // scalar step in the update's last block (no separate reduce, allreduce or
  // scalar launches)
  const bool fuse = !m->comm || m->comm->p2p;
  bool pap_fused = false;
  a.pap_fused = fuse ? &pap_fused : nullptr;
  auto iteration = [&](cudaStream_t s, cudaEvent_t e0, cudaEvent_t e1, unsigned rec_flags) -> sem_status {
    if (e0) SEM_CUDA_TRY(cudaEventRecordWithFlags(e0, s, rec_flags));
    pap_fused = false;
    SEM_TRY(ax_dssum_all(m, a, true, s));
    if (e1) SEM_CUDA_TRY(cudaEventRecordWithFlags(e1, s, rec_flags));
    if (!pap_fused) {
      SEM_CUDA_TRY(launch_cg_pap_reduce(m, s));
      SEM_TRY(allreduce(m, &m->sc->red[0], 1, s));
    }
    SEM_CUDA_TRY(launch_cg_update(m, s, fuse));
    if (!fuse) {
      SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
      SEM_CUDA_TRY(launch_cg_scalar_step(m, 1, s));
    }
    return SEM_OK;
  };
  // default: graph (measured ~1-2% faster on c2 at 1 and 2 GPUs with the
  // stream-order schedule), except with NCCL on the data path (the NCCL
  // fallback measured up to 3x slower captured than in stream order)
  bool use_graph = maxit > 1 && (!m->comm || m->xp2p);
  if (const char* env = getenv("SEM_GRAPH")) use_graph = maxit > 1 && atoi(env) != 0;  // tuning knob
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cs = s;
  cudaGraphNode_t ev_node[2] = {nullptr, nullptr};
  cudaEvent_t ph[2] = {nullptr, nullptr};
  if (use_graph) {
    const long nl0 = (long)m->nlaunch;
    if (m->prof) {
      SEM_CUDA_TRY(cudaEventCreate(&ph[0]));
      SEM_CUDA_TRY(cudaEventCreate(&ph[1]));
    }
    // captured on an owned stream (the caller's may be the legacy default
    // stream, which cannot be captured), joined to s by events
    cs = m->cap_stream;
    SEM_CUDA_TRY(cudaEventRecord(m->ev_cap, s));
    SEM_CUDA_TRY(cudaStreamWaitEvent(cs, m->ev_cap, 0));
    SEM_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    sem_status st = iteration(cs, ph[0], ph[1], cudaEventRecordExternal);
    cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    if (st != SEM_OK || ce != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      for (cudaEvent_t e : ph)
        if (e) cudaEventDestroy(e);
      if (st != SEM_OK) return st;
      return fail(SEM_ECUDA, std::string("CG graph capture: ") + cudaGetErrorString(ce));
    }
    const long per_iter = (long)m->nlaunch - nl0;
    m->nlaunch = nl0;
    SEM_CUDA_TRY(cudaGraphInstantiateWithFlags(&gexec, graph, cudaGraphInstantiateFlagUseNodePriority));
    if (m->prof) {
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(graph, nodes.data(), &nn);
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev;
        cudaGraphEventRecordNodeGetEvent(nd, &ev);
        if (ev == ph[0]) ev_node[0] = nd;
        if (ev == ph[1]) ev_node[1] = nd;
      }
    }
    for (int it = 0; it < maxit; ++it) {
      if (m->prof && ev_node[0] && ev_node[1]) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaGraphExecEventRecordNodeSetEvent(gexec, ev_node[0], e0);
        cudaGraphExecEventRecordNodeSetEvent(gexec, ev_node[1], e1);
        m->prof_ev.push_back(e0);
        m->prof_ev.push_back(e1);
      }
      SEM_CUDA_TRY(cudaGraphLaunch(gexec, cs));
      m->nlaunch += per_iter;
      if (tol > 0.0 && ((it + 1) % poll == 0)) {
        SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, cs));
        SEM_CUDA_TRY(cudaStreamSynchronize(cs));
        if (m->sc_host->done) break;
      }
    }
  } else {
    for (int it = 0; it < maxit; ++it) {
      cudaEvent_t ev[2] = {nullptr, nullptr};
      if (m->prof) {
        cudaEventCreate(&ev[0]);
        cudaEventCreate(&ev[1]);
        m->prof_ev.push_back(ev[0]);
        m->prof_ev.push_back(ev[1]);
      }
      SEM_TRY(iteration(s, ev[0], ev[1], cudaEventRecordDefault));
      if (tol > 0.0 && ((it + 1) % poll == 0)) {
        SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
        SEM_CUDA_TRY(cudaStreamSynchronize(s));
        if (m->sc_host->done) break;
      }
    }
  }
  if (gexec) {
    SEM_CUDA_TRY(cudaEventRecord(m->ev_cap, cs));
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_cap, 0));
    SEM_CUDA_TRY(cudaStreamSynchronize(cs));
    cudaGraphExecDestroy(gexec);
    cudaGraphDestroy(graph);
    for (cudaEvent_t e : ph)
      if (e) cudaEventDestroy(e);
  }
  SEM_CUDA_TRY(launch_cg_x_final(m, x, s));  // the last deferred x += alpha p
  SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, s));
  SEM_CUDA_TRY(cudaStreamSynchronize(s));
  const CGScalars h = *m->sc_host;
  if (singular && !h.breakdown) {
    SEM_CUDA_TRY(launch_wdot(m, x, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, x, 3, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  if (iters) *iters = h.iter + (h.breakdown ? 1 : 0);
  if (rel_res) *rel_res = h.bn > 0 ? sqrt(h.rtr) / h.bn : 0.0;
  if (converged) *converged = h.converged;
  if (h.breakdown) return fail(SEM_EBREAKDOWN, "sem_cg_solve: breakdown (pAp <= 0 or NaN)");
  return SEM_OK;
}

sem_status sem_cg_solve(sem_mesh_t m, const double* b, double* x, const double* h1, const double* h2, double h1c,
                        double h2c, double tol, int maxit, int* iters, double* rel_res, int* converged,
                        sem_stream_t stream) {
  SEM_TRY(check_op(m, b, x, "sem_cg_solve"));
  if (maxit < 0 || !(tol >= 0.0)) return fail(SEM_EINVAL, "sem_cg_solve: maxit < 0 or tol < 0");
  if (m->cg_pipelined)
    return cg_solve_pipelined(m, b, x, h1, h2, h1c, h2c, tol, maxit, iters, rel_res, converged,
                              (cudaStream_t)stream);
  if (m->cg_unique)
    return cg_solve_u(m, b, x, h1, h2, h1c, h2c, tol, maxit, iters, rel_res, converged, (cudaStream_t)stream);
  return cg_solve_impl(m, b, x, h1, h2, h1c, h2c, tol, maxit, iters, rel_res, converged, (cudaStream_t)stream);
}

sem_status sem_cg_solve_host(sem_mesh_t m, const double* b_host, double* x_host, const double* h1, const double* h2,
                             double h1c, double h2c, double tol, int maxit, int* iters, double* rel_res,
                             int* converged, sem_stream_t stream) {
  if (!m) return fail(SEM_EINVAL, "sem_cg_solve_host: NULL mesh");
  if (m->nloc > 0 && (!b_host || !x_host)) return fail(SEM_EINVAL, "sem_cg_solve_host: NULL field");
  sem_status st;
  if (!m->bw && (st = dalloc(&m->bw, m->nloc, "e2e b")) != SEM_OK) return st;
  if (!m->xw && (st = dalloc(&m->xw, m->nloc, "e2e x")) != SEM_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  // the upload of b runs on the aux stream, overlapping the Jacobi set-up of
  // the standard solver, which waits for it right before r = mask b
  SEM_CUDA_TRY(cudaEventRecord(m->ev_start, s));
  SEM_CUDA_TRY(cudaStreamWaitEvent(m->aux_stream, m->ev_start, 0));
  SEM_CUDA_TRY(cudaMemcpyAsync(m->bw, b_host, sizeof(double) * m->nloc, cudaMemcpyHostToDevice, m->aux_stream));
  SEM_CUDA_TRY(cudaEventRecord(m->ev_input, m->aux_stream));
  if (m->cg_pipelined || m->cg_unique) SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_input, 0));
  else m->input_pending = true;
  st = sem_cg_solve(m, m->bw, m->xw, h1, h2, h1c, h2c, tol, maxit, iters, rel_res, converged, stream);
  if (m->input_pending) {  // (an early error return before the init)
    m->input_pending = false;
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_input, 0));
  }
  if (st != SEM_OK && st != SEM_EBREAKDOWN) return st;
  SEM_CUDA_TRY(cudaMemcpyAsync(x_host, m->xw, sizeof(double) * m->nloc, cudaMemcpyDeviceToHost, s));
  SEM_CUDA_TRY(cudaStreamSynchronize(s));
  return st;
}

sem_status sem_profile_enable(sem_mesh_t m, int on) {
  if (!m) return fail(SEM_EINVAL, "sem_profile_enable: NULL mesh");
  m->prof = on != 0;
  for (auto ev : m->prof_ev) cudaEventDestroy(ev);
  m->prof_ev.clear();
  m->prof_launches = 0;
  m->prof_ms = 0.0;
  return SEM_OK;
}

sem_status sem_profile_get(sem_mesh_t m, int64_t* launches, double* ms, int64_t* kernel_launches) {
  if (!m) return fail(SEM_EINVAL, "sem_profile_get: NULL mesh");
  for (size_t q = 0; q + 1 < m->prof_ev.size(); q += 2) {
    cudaEventSynchronize(m->prof_ev[q + 1]);
    float t = 0.f;
    cudaEventElapsedTime(&t, m->prof_ev[q], m->prof_ev[q + 1]);
    m->prof_ms += t;
    m->prof_launches += 1;
    cudaEventDestroy(m->prof_ev[q]);
    cudaEventDestroy(m->prof_ev[q + 1]);
  }
  m->prof_ev.clear();
  if (launches) *launches = m->prof_launches;
  if (ms) *ms = m->prof_ms;
  if (kernel_launches) *kernel_launches = m->nlaunch;
  return SEM_OK;
}

}  // extern "C"
