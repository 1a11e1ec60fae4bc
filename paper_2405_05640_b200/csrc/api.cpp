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

#include "gmres.h"
#include "hsmg.h"
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
cudaError_t launch_affine_detect(const sem_mesh* m, double* C, int* nonaffine, cudaStream_t s);
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

// mask . dssum(A_e u) over all positions (cg: the CG-fused operator): one
// operator launch per launch segment (one rank: one launch), then one
// gather-scatter pass over the shared nodes (DESIGN.md "Gather-scatter":
// the in-launch alternatives were measured slower).  Several ranks: the boundary segment first (on a high-priority
// stream beside the interior launch when the exchange goes over peer
// memory), the interface exchange started right after it and finished last.
static sem_status ax_dssum_all(sem_mesh* m, const AxArgs& a, bool cg, cudaStream_t s) {
  if (m->comm && m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  if (m->E == 0) {  // an empty rank still takes part in the collective exchange
    if (m->comm) {
      SEM_TRY(comm_exchange_begin(m, a.w, s));
      SEM_TRY(comm_exchange_end(m, a.w, 3, s));
    }
    return SEM_OK;
  }
  const int nseg = (int)m->seg.size() - 1;
  auto launch = [&](int k, cudaStream_t st) -> cudaError_t {
    return launch_ax_range(m, a, cg, m->seg[k], m->seg[k + 1] - m->seg[k], st);
  };
  // the CG vectors in the x-planes-last layout use the plan built for it
  const bool xl = cg && m->xl_active;
  const uint32_t* gidx = xl ? m->d_gidx_xl : m->d_gidx;
  const std::vector<GsClass>& gcls = xl ? m->gs_cls_xl : m->gs_cls;
  bool* pap = cg ? a.pap_fused : nullptr;
  const bool pdl = a.pdl && !m->comm;
  if (m->comm && m->xp2p && nseg == 2 && m->bnd_stream) {
    // several ranks over peer memory: the boundary elements, their interface
    // partials and the stores into the peers on a high-priority stream while
    // the interior launch fills the rest of the GPU; the gather-scatter pass
    // waits for the boundary launch, the unpack for the stores
    SEM_CUDA_TRY(cudaEventRecord(m->ev_start, s));
    SEM_CUDA_TRY(cudaStreamWaitEvent(m->bnd_stream, m->ev_start, 0));
    SEM_CUDA_TRY(launch(0, m->bnd_stream));
    SEM_CUDA_TRY(cudaEventRecord(m->ev_bnd, m->bnd_stream));
    SEM_TRY(comm_exchange_begin(m, a.w, m->bnd_stream));
    SEM_CUDA_TRY(cudaEventRecord(m->ev_pack, m->bnd_stream));
    SEM_CUDA_TRY(launch(1, s));
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_bnd, 0));
    SEM_CUDA_TRY(launch_gs_nodal(m, a.w, gidx, gcls, 3, s, pap, pdl));
    SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_pack, 0));
    SEM_TRY(comm_exchange_end(m, a.w, 3, s));
    return SEM_OK;
  }
  // stream order: the launches, the exchange started after the boundary
  // segment, the gather-scatter pass, the exchange finished
  for (int k = 0; k < nseg; ++k) {
    SEM_CUDA_TRY(launch(k, s));
    if (m->comm && k == 0) SEM_TRY(comm_exchange_begin(m, a.w, s));
  }
  SEM_CUDA_TRY(launch_gs_nodal(m, a.w, gidx, gcls, 3, s, pap, pdl));
  if (m->comm) SEM_TRY(comm_exchange_end(m, a.w, 3, s));
  return SEM_OK;
}

// streams and events of a mesh
static sem_status create_streams(sem_mesh* m) {
  if (!m->aux_stream && cudaStreamCreateWithFlags(&m->aux_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SEM_ECUDA, "cudaStreamCreate(aux)");
  if (m->comm && !m->bnd_stream) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&m->bnd_stream, cudaStreamNonBlocking, hi) != cudaSuccess)
      return fail(SEM_ECUDA, "cudaStreamCreate(boundary)");
  }
  for (cudaEvent_t* ev : {&m->ev_start, &m->ev_cap, &m->ev_bnd, &m->ev_input})
    if (!*ev && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) return fail(SEM_ECUDA, "event");
  if (!m->cap_stream && cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SEM_ECUDA, "cudaStreamCreate(cap)");
  return SEM_OK;
}

// affine-element detection (option affine)
static sem_status detect_affine(sem_mesh* m) {
  m->affine = false;
  if (!m->opt.affine || !m->has_geom || m->E == 0) return SEM_OK;
  if (!m->d_gaff) SEM_TRY(dalloc(&m->d_gaff, m->E * 6, "affine constants"));
  int* flag = nullptr;
  SEM_CUDA_TRY(cudaMalloc((void**)&flag, sizeof(int)));
  int hf = 0;
  cudaMemcpy(flag, &hf, sizeof(int), cudaMemcpyHostToDevice);
  cudaError_t e = launch_affine_detect(m, m->d_gaff, flag, 0);
  if (e == cudaSuccess) e = cudaMemcpy(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(flag);
  if (e != cudaSuccess) return fail(SEM_ECUDA, std::string("affine detection: ") + cudaGetErrorString(e));
  m->affine = (hf == 0);
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

static void hsmg_free(sem::HsmgState* H);

static void mesh_free(sem_mesh* m) {
  if (!m) return;
  if (m->hs) {
    hsmg_free(m->hs);
    m->hs = nullptr;
  }
  comm_mesh_free(m);
  gs_plans_free(m);
  for (double* q : {m->MJ, m->Bg, m->pn_t, m->pn_c, m->pn_r})
    if (q) cudaFree(q);
  if (m->gm) {
    m->gm->drop_graphs();
    void* gp[] = {m->gm->V, m->gm->z, m->gm->Z, m->gm->part, m->gm->ticket, m->gm->red, m->gm->gs};
    for (void* p : gp)
      if (p) cudaFree(p);
    if (m->gm->gs_host) cudaFreeHost(m->gm->gs_host);
    delete m->gm;
    m->gm = nullptr;
  }
  void* ptrs[] = {m->d_gaff, m->coords, m->G, m->B, m->mult, m->mask, m->m8, m->d_elem_ent, m->d_ent_ptr, m->d_ent_copy,
                  m->d_ent_flags, m->d_elist_all, m->r, m->p, m->w, m->dinv, m->xw, m->bw,
                  m->part, m->ticket, m->sc, m->s_cg};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (m->sc_host) cudaFreeHost(m->sc_host);
  for (cudaEvent_t ev : {m->ev_start, m->ev_cap, m->ev_bnd, m->ev_input})
    if (ev) cudaEventDestroy(ev);
  if (m->bnd_stream) cudaStreamDestroy(m->bnd_stream);
  if (m->aux_stream) cudaStreamDestroy(m->aux_stream);
  if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
  for (auto ev : m->prof_ev) cudaEventDestroy(ev);
  delete m;
}

void sem_mesh_destroy(sem_mesh_t m) { mesh_free(m); }

sem_status sem_mesh_create(int64_t E, int N, const double* coords, const int64_t* conn, const int8_t* bc,
                           sem_comm_t comm, sem_mesh_t* out) {
  SEM_NVTX("sem_mesh_create");
  if (!out) return fail(SEM_EINVAL, "sem_mesh_create: out is NULL");
  *out = nullptr;
  if (E < 0) return fail(SEM_EINVAL, "sem_mesh_create: E < 0");
  if (N < 1 || N > kMaxN) return fail(SEM_EINVAL, "sem_mesh_create: N must be in [1, 11]");
  if (E > 0 && (!coords || !conn)) return fail(SEM_EINVAL, "sem_mesh_create: NULL coords or conn");
  if (E * (int64_t)((N + 1) * (N + 1) * (N + 1)) >= (int64_t(1) << 31))
    return fail(SEM_EINVAL, "sem_mesh_create: E * (N+1)^3 must be < 2^31 local nodes per GPU");
  sem_mesh* m = new (std::nothrow) sem_mesh();
  if (!m) return fail(SEM_ENOMEM, "sem_mesh_create: host allocation");
  m->E = E;
  m->N = N;
  m->lx = N + 1;
  m->n3 = m->lx * m->lx * m->lx;
  m->n3p = (m->n3 + 1) & ~1;
  m->nloc = E * m->n3;
  m->comm = comm;
  sem_options_default(&m->opt);
  if (E > 0) {
    m->conn_h.assign(conn, conn + 8 * E);
    if (bc) m->bc_h.assign(bc, bc + 6 * E);
  }
  cudaGetDevice(&m->device);
  if (cudaDeviceGetAttribute(&m->nsm, cudaDevAttrMultiProcessorCount, m->device) != cudaSuccess || m->nsm < 1) {
    cudaGetLastError();
    m->nsm = 1;
  }
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
  if (e1 == cudaSuccess) e1 = cudaMemset(m->ticket, 0, sizeof(unsigned) * 4);
  if (e1 == cudaSuccess) e1 = cudaMemset(m->sc, 0, sizeof(CGScalars));
  if (e1 == cudaSuccess && m->nloc > 0) e1 = launch_mult_mask(m, 0);
  if (e1 == cudaSuccess) e1 = cudaDeviceSynchronize();
  if (e1 != cudaSuccess) {
    mesh_free(m);
    return fail(SEM_ECUDA, std::string("sem_mesh_create upload: ") + cudaGetErrorString(e1));
  }
  st = create_streams(m);
  if (st == SEM_OK && comm) st = comm_setup_device(m);
  m->pos = pos;
  if (st == SEM_OK) st = build_gs_plans(m, pos);
  if (st != SEM_OK) {
    mesh_free(m);
    return st;
  }
  *out = m;
  return SEM_OK;
}

void sem_options_default(sem_options_t* opt) {
  if (!opt) return;
  opt->cg_variant = SEM_CG_STANDARD;
  opt->affine = 0;
  opt->graph = 1;
  opt->pdl = 0;
  opt->gmres_precond = SEM_PC_JACOBI;
  opt->hsmg_coarse_iters = 5;
  opt->pnpn_pressure = SEM_PRESSURE_CG;
  opt->cg_layout = 1;

}

sem_status sem_mesh_get_options(sem_mesh_t m, sem_options_t* opt) {
  if (!m || !opt) return fail(SEM_EINVAL, "sem_mesh_get_options: NULL argument");
  *opt = m->opt;
  return SEM_OK;
}

sem_status sem_mesh_set_options(sem_mesh_t m, const sem_options_t* opt) {
  SEM_NVTX("sem_mesh_set_options");
  if (!m || !opt) return fail(SEM_EINVAL, "sem_mesh_set_options: NULL argument");
  if (opt->cg_variant != SEM_CG_STANDARD && opt->cg_variant != SEM_CG_PIPELINED)
    return fail(SEM_EINVAL, "sem_mesh_set_options: unknown cg_variant");
  if (opt->gmres_precond != SEM_PC_JACOBI && opt->gmres_precond != SEM_PC_HSMG)
    return fail(SEM_EINVAL, "sem_mesh_set_options: unknown gmres_precond");
  if (opt->hsmg_coarse_iters < 1 || opt->hsmg_coarse_iters > 1000)
    return fail(SEM_EINVAL, "sem_mesh_set_options: hsmg_coarse_iters must be in [1, 1000]");
  if (opt->pnpn_pressure != SEM_PRESSURE_CG && opt->pnpn_pressure != SEM_PRESSURE_GMRES)
    return fail(SEM_EINVAL, "sem_mesh_set_options: unknown pnpn_pressure");
  const sem_options_t old = m->opt;
  m->opt = *opt;
  m->opt.affine = opt->affine ? 1 : 0;
  m->opt.graph = opt->graph ? 1 : 0;
  m->opt.pdl = opt->pdl ? 1 : 0;
  m->opt.cg_layout = opt->cg_layout ? 1 : 0;
  if (old.affine != m->opt.affine) SEM_TRY(detect_affine(m));
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
  SEM_NVTX("sem_geom_factors");
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
  // affine-element variant (option affine)
  return detect_affine(m);
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
  SEM_NVTX("sem_ax");
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
  SEM_NVTX("sem_gs_op");
  if (!m) return fail(SEM_EINVAL, "sem_gs_op: NULL mesh");
  if (op != SEM_GS_ADD && op != SEM_GS_MASK) return fail(SEM_EINVAL, "sem_gs_op: unknown op");
  if (m->nloc > 0 && !u) return fail(SEM_EINVAL, "sem_gs_op: NULL field");
  cudaStream_t s = (cudaStream_t)stream;
  SEM_CUDA_TRY(launch_gs_nodal(m, u, m->d_gidx, m->gs_cls, op == SEM_GS_ADD ? 1 : 2, s));
  if (m->comm) SEM_TRY(comm_gs_exchange(m, u, op == SEM_GS_ADD ? 1 : 2, s));
  return SEM_OK;
}

sem_status sem_ax_dssum(sem_mesh_t m, const double* u, double* w, const double* h1, const double* h2,
                        double h1c, double h2c, sem_stream_t stream) {
  SEM_NVTX("sem_ax_dssum");
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
  SEM_NVTX("sem_rhs");
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
  SEM_NVTX("sem_jacobi");
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

// xl_active for the duration of a CG iteration loop (reset on every exit)
struct XlScope {
  sem_mesh* m;
  XlScope(sem_mesh* mm, bool on) : m(mm) { m->xl_active = on; }
  ~XlScope() { m->xl_active = false; }
};

static sem_status allreduce(sem_mesh* m, double* d, int n, cudaStream_t s) {
  if (!m->comm) return SEM_OK;
  return comm_allreduce_sum(m, d, n, s);
}

}  // extern "C"

// The single-reduction CG's pass (ax_p.cu) in the unfused schedule: one
// launch per segment, the exchange started after the boundary segment, one
// gather-scatter pass over the full nodal plan, the exchange finished.
template <class LaunchFn>
static sem_status ax_dssum_unfused(sem_mesh* m, double* w, LaunchFn launch, cudaStream_t s) {
  if (m->comm && m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  const int nseg = (int)m->seg.size() - 1;
  for (int k = 0; k < nseg && m->E > 0; ++k) {
    SEM_CUDA_TRY(launch(m->seg[k], m->seg[k + 1] - m->seg[k], s));
    if (m->comm && k == 0) SEM_TRY(comm_exchange_begin(m, w, s));
  }
  if (m->comm && m->E == 0) SEM_TRY(comm_exchange_begin(m, w, s));
  SEM_CUDA_TRY(launch_gs_nodal(m, w, m->d_gidx, m->gs_cls, 3, s));
  if (m->comm) SEM_TRY(comm_exchange_end(m, w, 3, s));
  return SEM_OK;
}

extern "C" {

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
    SEM_TRY(ax_dssum_unfused(
        m, m->w, [&](int64_t q0, int64_t n, cudaStream_t st) { return launch_ax_pcg(m, a, x, m->w, m->w, first, q0, n, st); },
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
  // Jacobi preconditioner (kept when the caller set reuse_dinv: the same
  // operator was just solved with, sem_pnpn_step's velocity components)
  if (!m->reuse_dinv) SEM_TRY(sem_jacobi(m, h1, h2, h1c, h2c, m->dinv, (sem_stream_t)s));
  m->reuse_dinv = false;
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
  // option cg_layout: the operator output A_e p (w) is kept per element in
  // the x-planes-last layout during the iteration loop
  const bool use_xl = m->opt.cg_layout != 0;
  XlScope xl_scope(m, use_xl);
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
  a.pdl = m->opt.pdl && !m->comm;
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
  auto iteration = [&](cudaStream_t s, cudaEvent_t e0, cudaEvent_t e1, unsigned rec_flags,
                       cudaGraphConditionalHandle loop) -> sem_status {
    if (e0) SEM_CUDA_TRY(cudaEventRecordWithFlags(e0, s, rec_flags));
    pap_fused = false;
    SEM_TRY(ax_dssum_all(m, a, true, s));
    if (e1) SEM_CUDA_TRY(cudaEventRecordWithFlags(e1, s, rec_flags));
    if (!pap_fused) {
      SEM_CUDA_TRY(launch_cg_pap_reduce(m, s));
      SEM_TRY(allreduce(m, &m->sc->red[0], 1, s));
    }
    SEM_CUDA_TRY(launch_cg_update(m, s, fuse, loop, a.pdl));
    if (!fuse) {
      SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
      SEM_CUDA_TRY(launch_cg_scalar_step(m, 1, s));
    }
    return SEM_OK;
  };
  // default: graph (measured ~1-2% faster on c2 at 1 and 2 GPUs with the
  // stream-order schedule), except with NCCL on the data path (the NCCL
  // fallback measured up to 3x slower captured than in stream order)
  const bool use_graph = m->opt.graph && maxit > 1 && (!m->comm || m->xp2p);
  // the whole loop as ONE graph: a conditional WHILE node whose body is the
  // captured iteration and whose condition the update kernel sets to !done
  // (no host polls, no per-iteration launches); per-iteration
  // graph launches instead while profiling (event nodes time each operator)
  const bool use_cond = use_graph && fuse && !m->prof;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cs = s;
  cudaGraphNode_t ev_node[2] = {nullptr, nullptr};
  cudaEvent_t ph[2] = {nullptr, nullptr};
  if (use_cond) {
    const long nl0 = (long)m->nlaunch;
    SEM_CUDA_TRY(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle loop = 0;
    cudaError_t ce = cudaGraphConditionalHandleCreate(&loop, graph, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = loop;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode = nullptr;
    if (ce == cudaSuccess) ce = cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp);
    if (ce != cudaSuccess) {
      cudaGraphDestroy(graph);
      return fail(SEM_ECUDA, std::string("CG conditional graph: ") + cudaGetErrorString(ce));
    }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cs = m->cap_stream;
    SEM_CUDA_TRY(cudaEventRecord(m->ev_cap, s));
    SEM_CUDA_TRY(cudaStreamWaitEvent(cs, m->ev_cap, 0));
    SEM_CUDA_TRY(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    sem_status st = iteration(cs, nullptr, nullptr, 0, loop);
    cudaGraph_t captured = nullptr;
    ce = cudaStreamEndCapture(cs, &captured);
    if (st != SEM_OK || ce != cudaSuccess) {
      cudaGraphDestroy(graph);
      if (st != SEM_OK) return st;
      return fail(SEM_ECUDA, std::string("CG loop-body capture: ") + cudaGetErrorString(ce));
    }
    const long per_iter = (long)m->nlaunch - nl0;
    m->nlaunch = nl0;
    ce = cudaGraphInstantiateWithFlags(&gexec, graph, cudaGraphInstantiateFlagUseNodePriority);
    if (ce != cudaSuccess) {
      cudaGraphDestroy(graph);
      return fail(SEM_ECUDA, std::string("CG conditional graph instantiate: ") + cudaGetErrorString(ce));
    }
    SEM_CUDA_TRY(cudaGraphLaunch(gexec, cs));
    SEM_CUDA_TRY(cudaMemcpyAsync(m->sc_host, m->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, cs));
    SEM_CUDA_TRY(cudaStreamSynchronize(cs));
    m->nlaunch += per_iter * std::max(1, m->sc_host->iter + (m->sc_host->breakdown ? 1 : 0));
  } else if (use_graph) {
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
    sem_status st = iteration(cs, ph[0], ph[1], cudaEventRecordExternal, 0);
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
      SEM_TRY(iteration(s, ev[0], ev[1], cudaEventRecordDefault, 0));
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
  m->xl_active = false;
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
  SEM_NVTX("sem_cg_solve");
  SEM_TRY(check_op(m, b, x, "sem_cg_solve"));
  if (maxit < 0 || !(tol >= 0.0)) return fail(SEM_EINVAL, "sem_cg_solve: maxit < 0 or tol < 0");
  if (m->comm && m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  sem_status st;
  if (m->opt.cg_variant == SEM_CG_PIPELINED)
    st = cg_solve_pipelined(m, b, x, h1, h2, h1c, h2c, tol, maxit, iters, rel_res, converged, (cudaStream_t)stream);
  else
    st = cg_solve_impl(m, b, x, h1, h2, h1c, h2c, tol, maxit, iters, rel_res, converged, (cudaStream_t)stream);
  // a peer wait that timed out (multi-GPU) outranks the numerical outcome
  if (m->comm && (st == SEM_OK || st == SEM_EBREAKDOWN)) SEM_TRY(comm_check(m->comm));
  return st;
}

// ---------------------------------------------------------------------------
// Hybrid-Schwarz multigrid (reading R16; kernels in hsmg.cu,
// host set-up in hsmg_setup.cpp, the oracle's oracle/hsmg.py in the same
// order).  Levels are ordinary meshes of this library (same elements, order
// N_l, the fine element map evaluated at the level's GLL nodes): their
// operator, gather-scatter, multi-GPU exchange and CG are the ones above.
// ---------------------------------------------------------------------------
static constexpr double kHsmgCoarseTol = 1e-12;

// u <- mask . dssum(u) (one pass; the interface exchange with a communicator)
static sem_status gs_dssum_mask(sem_mesh* m, double* u, cudaStream_t s, int extra = 0) {
  SEM_CUDA_TRY(launch_gs_nodal(m, u, m->d_gidx, m->gs_cls, 3 | extra, s, nullptr, false));
  if (m->comm) SEM_TRY(comm_gs_exchange(m, u, 3 | extra, s));
  return SEM_OK;
}

static void hsmg_free(sem::HsmgState* H) {
  if (!H) return;
  for (int l = 0; l < kHsmgMaxLevels; ++l) {
    for (double* q : {H->r[l], H->z[l], H->t[l], H->fdm[l], H->J[l]})
      if (q) cudaFree(q);
    if (H->owned[l] && H->lev[l]) mesh_free(H->lev[l]);
  }
  if (H->L) cudaFree(H->L);
  delete H;
}

static sem_status hsmg_ensure(sem_mesh* m) {
  if (m->hs) return SEM_OK;
  if (!m->has_geom) return fail(SEM_EINVAL, "hybrid-Schwarz multigrid: call sem_geom_factors first");
  HsmgState* H = new (std::nothrow) HsmgState();
  if (!H) return fail(SEM_ENOMEM, "hsmg: host allocation");
  auto bail = [&](sem_status st) {
    hsmg_free(H);
    return st;
  };
  int orders[kHsmgMaxLevels];
  H->nlev = hsmg_level_orders(m->N, orders);
  for (int l = 0; l < H->nlev; ++l) H->N[l] = orders[l];
  const int64_t E = m->E;
  std::vector<double> cf((size_t)3 * m->nloc);
  if (m->nloc > 0 &&
      cudaMemcpy(cf.data(), m->coords, sizeof(double) * cf.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    return bail(fail(SEM_ECUDA, "hsmg: coordinates download"));
  // element lengths (the same corners at every level)
  std::vector<double> L((size_t)3 * std::max<int64_t>(E, 1), 0.0);
  hsmg_element_lengths(E, m->lx, cf.data(), L.data());
  sem_status st = dalloc(&H->L, 3 * std::max<int64_t>(E, 1), "hsmg lengths");
  if (st != SEM_OK) return bail(st);
  if (cudaMemcpy(H->L, L.data(), sizeof(double) * L.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(SEM_ECUDA, "hsmg: lengths upload"));
  std::vector<double> xf(m->lx), wf(m->lx);
  gll_golub_welsch(m->N, xf.data(), wf.data());
  // level meshes: level 0 is this mesh when it smooths; the order-1 level is
  // always a mesh of its own
  const int first_owned = H->nlev > 1 ? 1 : 0;
  if (H->nlev > 1) H->lev[0] = m;
  for (int l = first_owned; l < H->nlev; ++l) {
    const int Nl = H->N[l], lxl = Nl + 1;
    std::vector<double> xl(lxl), wl(lxl), K((size_t)lxl * m->lx);
    gll_golub_welsch(Nl, xl.data(), wl.data());
    hsmg_lagrange(m->lx, xf.data(), lxl, xl.data(), K.data());
    const int64_t n3l = (int64_t)lxl * lxl * lxl;
    std::vector<double> cl((size_t)3 * E * n3l);
    hsmg_interp_coords(E, m->lx, lxl, K.data(), cf.data(), cl.data());
    sem_mesh* lev = nullptr;
    st = sem_mesh_create(E, Nl, cl.data(), m->conn_h.data(), m->bc_h.empty() ? nullptr : m->bc_h.data(), m->comm,
                         &lev);
    if (st != SEM_OK) return bail(st);
    H->lev[l] = lev;
    H->owned[l] = true;
    if ((st = sem_geom_factors(lev)) != SEM_OK) return bail(st);
    if ((st = ensure_cg(lev)) != SEM_OK) return bail(st);
  }
  // work vectors, smoother factors, transfer matrices
  for (int l = 0; l < H->nlev; ++l) {
    sem_mesh* ml = H->lev[l];
    const int64_t n = std::max<int64_t>(ml->nloc, 1);
    if (l > 0 && ((st = dalloc(&H->r[l], n, "hsmg r")) != SEM_OK || (st = dalloc(&H->z[l], n, "hsmg z")) != SEM_OK))
      return bail(st);
    if (l + 1 < H->nlev) {
      if ((st = dalloc(&H->t[l], n, "hsmg t")) != SEM_OK) return bail(st);
      const int lx = ml->lx, lxc = H->N[l + 1] + 1;
      std::vector<double> f((size_t)lx * lx + lx);
      if (!hsmg_fdm_1d(ml->N, f.data(), f.data() + lx * lx)) return bail(fail(SEM_EINVAL, "hsmg: eigen-solver"));
      if ((st = dalloc(&H->fdm[l], (int64_t)f.size(), "hsmg fdm")) != SEM_OK) return bail(st);
      std::vector<double> xa(lx), wa(lx), xb(lxc), wb(lxc), J((size_t)lx * lxc);
      gll_golub_welsch(ml->N, xa.data(), wa.data());
      gll_golub_welsch(H->N[l + 1], xb.data(), wb.data());
      hsmg_lagrange(lxc, xb.data(), lx, xa.data(), J.data());  // J[a*lxc + b]
      if ((st = dalloc(&H->J[l], (int64_t)J.size(), "hsmg J")) != SEM_OK) return bail(st);
      if (cudaMemcpy(H->fdm[l], f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(H->J[l], J.data(), sizeof(double) * J.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(SEM_ECUDA, "hsmg: factor upload"));
    }
  }
  m->hs = H;
  return SEM_OK;
}

// Jacobi-PCG (R10) driven entirely on the device: no host read, so it can sit
// inside a preconditioner; at most maxit steps, stopping at tol (k_cg_update
// turns every later launch into a no-op).  m->dinv must hold the Jacobi
// inverse of (h1c, h2c).
static sem_status cg_device(sem_mesh* m, const double* b, double* x, double h1c, double h2c, double tol, int maxit,
                            cudaStream_t s) {
  const int singular = (m->n_masked_glob == 0) && (h2c == 0.0);
  SEM_CUDA_TRY(cudaMemsetAsync(m->sc, 0, sizeof(CGScalars), s));
  SEM_CUDA_TRY(launch_cg_config(m, tol, maxit, singular, s));
  SEM_CUDA_TRY(launch_cg_init(m, b, x, tol, maxit, singular, s));
  if (singular) {
    SEM_CUDA_TRY(launch_wdot(m, m->r, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, m->r, 3, s));
  }
  SEM_CUDA_TRY(launch_cg_start(m, s));
  SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
  SEM_CUDA_TRY(launch_cg_scalar_step(m, 0, s));
  AxArgs a{};
  a.w = m->w;
  a.h1c = h1c;
  a.h2c = h2c;
  a.r = m->r;
  a.dinv = m->dinv;
  a.p = m->p;
  a.sc = m->sc;
  a.part = m->part + pap_part_offset();
  a.x = x;
  m->pap_nparts = m->E;
  const bool fuse = !m->comm || m->comm->p2p;
  bool pap_fused = false;
  a.pap_fused = fuse ? &pap_fused : nullptr;
  for (int it = 0; it < maxit; ++it) {
    pap_fused = false;
    SEM_TRY(ax_dssum_all(m, a, true, s));
    if (!pap_fused) {
      SEM_CUDA_TRY(launch_cg_pap_reduce(m, s));
      SEM_TRY(allreduce(m, &m->sc->red[0], 1, s));
    }
    SEM_CUDA_TRY(launch_cg_update(m, s, fuse));
    if (!fuse) {
      SEM_TRY(allreduce(m, &m->sc->red[1], 2, s));
      SEM_CUDA_TRY(launch_cg_scalar_step(m, 1, s));
    }
  }
  SEM_CUDA_TRY(launch_cg_x_final(m, x, s));
  if (singular) {
    SEM_CUDA_TRY(launch_wdot(m, x, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, x, 3, s));
  }
  return SEM_OK;
}

// the coarse level's Jacobi inverse for (h1c, h2c), recomputed when they change
// (outside any graph capture)
static sem_status hsmg_prepare(sem_mesh* m, double h1c, double h2c, cudaStream_t s) {
  HsmgState* H = m->hs;
  sem_mesh* C = H->lev[H->nlev - 1];
  if (H->h1c != h1c || H->h2c != h2c) {
    SEM_TRY(sem_jacobi(C, nullptr, nullptr, h1c, h2c, C->dinv, (sem_stream_t)s));
    H->h1c = h1c;
    H->h2c = h2c;
  }
  return SEM_OK;
}

// z = M r, one V(1,0) cycle (R16); `skip` (may be NULL): a device flag that
// turns the fine-level kernels into no-ops (a GMRES cycle that has stopped)
static sem_status hsmg_vcycle(sem_mesh* m, const double* r, double* z, double h1c, double h2c, const int* skip,
                              cudaStream_t s) {
  HsmgState* H = m->hs;
  const int nl = H->nlev;
  sem_mesh* C = H->lev[nl - 1];
  const int K = m->opt.hsmg_coarse_iters;
  if (nl == 1) return cg_device(C, r, z, h1c, h2c, kHsmgCoarseTol, K, s);
  const double* rl = r;
  for (int l = 0; l + 1 < nl; ++l) {
    sem_mesh* M = H->lev[l];
    double* zl = l == 0 ? z : H->z[l];
    // smoother: z_l = mask (1/m) dssum(A~_e^-1 r_l)
    SEM_CUDA_TRY(launch_fdm(M, rl, zl, H->L, H->fdm[l], h1c, h2c, skip, s));
    SEM_TRY(gs_dssum_mask(M, zl, s, 4));  // the 1/m average rides in the pass (interior nodes: m = 1)
    // restricted residual r_{l+1} = mask dssum(J^T (r_l / m - mask A_e z_l))
    // = R_l (r_l - A_l z_l) (hsmg.cu k_restrict)
    AxArgs a{};
    a.u = zl;
    a.w = H->t[l];
    a.h1c = h1c;
    a.h2c = h2c;
    a.skip = skip;
    // A_e z_l unassembled: the restriction's coarse dssum assembles it
    SEM_CUDA_TRY(launch_ax_range(M, a, false, 0, M->E, s));
    SEM_CUDA_TRY(launch_restrict(M, H->N[l + 1] + 1, rl, H->t[l], H->J[l], H->r[l + 1], skip, s));
    SEM_TRY(gs_dssum_mask(H->lev[l + 1], H->r[l + 1], s));
    rl = H->r[l + 1];
  }
  SEM_TRY(cg_device(C, rl, H->z[nl - 1], h1c, h2c, kHsmgCoarseTol, K, s));
  for (int l = nl - 2; l >= 0; --l)
    SEM_CUDA_TRY(launch_prolong_add(H->lev[l], H->N[l + 1] + 1, H->z[l + 1], H->J[l], l == 0 ? z : H->z[l], skip, s));
  return SEM_OK;
}

sem_status sem_hsmg_apply(sem_mesh_t m, const double* r, double* z, double h1c, double h2c, sem_stream_t stream) {
  SEM_NVTX("sem_hsmg_apply");
  SEM_TRY(check_op(m, r, z, "sem_hsmg_apply"));
  if (r == z && m->nloc > 0) return fail(SEM_EINVAL, "sem_hsmg_apply: z must not alias r");
  if (m->comm && m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  SEM_TRY(hsmg_ensure(m));
  SEM_TRY(hsmg_prepare(m, h1c, h2c, (cudaStream_t)stream));
  SEM_TRY(hsmg_vcycle(m, r, z, h1c, h2c, nullptr, (cudaStream_t)stream));
  return SEM_OK;
}

// Restarted GMRES(m) for A x = b (reading R14; kernels and
// algorithm in gmres.cu).  Host loop: one cycle of up to `restart` Arnoldi
// steps is issued without any host synchronisation (the device stops a cycle
// early through GmScalars::cycle_stop, which also makes the operator launch a
// no-op), then the cycle end (y, x update, true residual, next v_0); the host
// reads the scalars once per cycle.
static sem_status gm_ensure(sem_mesh* m, int restart, bool flex) {
  GmState*& G = m->gm;
  if (G && G->restart >= restart) {
    if (flex && !G->Z) SEM_TRY(dalloc(&G->Z, (int64_t)G->restart * std::max<int64_t>(m->nloc, 1), "FGMRES Z"));
    return SEM_OK;
  }
  if (G) {
    G->drop_graphs();
    void* gp[] = {G->V, G->z, G->Z, G->part, G->ticket, G->red, G->gs};
    for (void* p : gp)
      if (p) cudaFree(p);
    if (G->gs_host) cudaFreeHost(G->gs_host);
    if (G->stop_host) cudaFreeHost(G->stop_host);
    for (cudaEvent_t e : G->ev_stop)
      if (e) cudaEventDestroy(e);
    delete G;
    G = nullptr;
  }
  G = new (std::nothrow) GmState();
  if (!G) return fail(SEM_ENOMEM, "sem_gmres_solve: host allocation");
  G->restart = restart;
  G->ld = std::max<int64_t>((m->nloc + 31) / 32 * 32, 32);
  SEM_TRY(dalloc(&G->V, (int64_t)(restart + 1) * G->ld, "GMRES basis"));
  SEM_TRY(dalloc(&G->z, std::max<int64_t>(m->nloc, 1), "GMRES z"));
  if (flex) SEM_TRY(dalloc(&G->Z, (int64_t)restart * std::max<int64_t>(m->nloc, 1), "FGMRES Z"));
  SEM_TRY(dalloc(&G->part, kGmMaxBlocks * 34, "GMRES partials"));
  SEM_TRY(dalloc(&G->ticket, 4, "GMRES ticket"));
  SEM_TRY(dalloc(&G->red, 40, "GMRES sums"));
  SEM_TRY(dalloc(&G->gs, 1, "GMRES scalars"));
  SEM_CUDA_TRY(cudaMemset(G->ticket, 0, sizeof(unsigned) * 4));
  if (cudaMallocHost((void**)&G->gs_host, sizeof(GmScalars)) != cudaSuccess)
    return fail(SEM_ENOMEM, "cudaMallocHost(GMRES scalars)");
  if (cudaMallocHost((void**)&G->stop_host, 2 * sizeof(int)) != cudaSuccess)
    return fail(SEM_ENOMEM, "cudaMallocHost(GMRES stop flags)");
  for (cudaEvent_t& e : G->ev_stop) SEM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SEM_OK;
}

sem_status sem_gmres_solve(sem_mesh_t m, const double* b, double* x, const double* h1, const double* h2, double h1c,
                           double h2c, double tol, int maxit, int restart, int* iters, double* rel_res,
                           int* converged, sem_stream_t stream) {
  SEM_NVTX("sem_gmres_solve");
  SEM_TRY(check_op(m, b, x, "sem_gmres_solve"));
  if (maxit < 0 || !(tol >= 0.0)) return fail(SEM_EINVAL, "sem_gmres_solve: maxit < 0 or tol < 0");
  if (restart < 1 || restart > kGmMaxRestart)
    return fail(SEM_EINVAL, "sem_gmres_solve: restart must be in [1, " + std::to_string(kGmMaxRestart) + "]");
  if (m->comm && m->comm->broken) return fail(SEM_ENCCL, "communicator retired after a peer timeout");
  cudaStream_t s = (cudaStream_t)stream;
  const bool flex = m->opt.gmres_precond == SEM_PC_HSMG;
  if (flex && (h1 || h2))
    return fail(SEM_EINVAL, "sem_gmres_solve: the multigrid preconditioner takes constant coefficients only");
  SEM_TRY(ensure_cg(m));
  if (flex) SEM_TRY(hsmg_ensure(m));
  SEM_TRY(gm_ensure(m, restart, flex));
  GmState* G = m->gm;
  // singular := no masked node anywhere and h2 == 0 everywhere (reading R10)
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
  SEM_TRY(sem_jacobi(m, h1, h2, h1c, h2c, m->dinv, stream));
  // b_m = mask b (projected when singular) into m->r; x = 0
  SEM_CUDA_TRY(launch_cg_init(m, b, x, tol, maxit, singular, s));
  if (singular) {
    SEM_CUDA_TRY(launch_wdot(m, m->r, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, m->r, 3, s));
  }
  const double* bm = m->r;
  GmScalars init{};
  init.tol = tol;
  init.maxit = maxit;
  init.restart = restart;
  SEM_CUDA_TRY(cudaMemcpyAsync(G->gs, &init, sizeof(GmScalars), cudaMemcpyHostToDevice, s));
  // r_0 = b (x = 0): v_0 = b / |b|
  if (m->nloc > 0) SEM_CUDA_TRY(cudaMemsetAsync(m->w, 0, sizeof(double) * m->nloc, s));
  SEM_CUDA_TRY(gm_launch_resid(m, G, bm, s));
  SEM_TRY(allreduce(m, &G->gs->nn, 1, s));
  SEM_CUDA_TRY(gm_launch_start(m, G, 1, flex, s));
  AxArgs a{};
  a.h1 = h1;
  a.h2 = h2;
  a.h1c = h1c;
  a.h2c = h2c;
  // one Arnoldi step j: (V-cycle), operator, the three vector passes, Givens
  auto arnoldi_step = [&](int j, cudaStream_t st) -> sem_status {
    AxArgs aj = a;
    aj.u = G->z;
    if (flex) {  // Z_j = M v_j (one V-cycle), stored for the solution update
      aj.u = G->Z + (int64_t)j * m->nloc;
      SEM_TRY(hsmg_vcycle(m, G->V + (int64_t)j * G->ld, G->Z + (int64_t)j * m->nloc, h1c, h2c, &G->gs->cycle_stop,
                          st));
    }
    aj.w = m->w;
    aj.skip = &G->gs->cycle_stop;
    SEM_TRY(ax_dssum_all(m, aj, false, st));  // w = A M v_j
    SEM_CUDA_TRY(gm_launch_dots(m, G, j + 1, st));
    SEM_TRY(allreduce(m, G->gs->h, j + 1, st));
    SEM_CUDA_TRY(gm_launch_update(m, G, j + 1, st));
    SEM_TRY(allreduce(m, G->red, 33, st));
    SEM_CUDA_TRY(gm_launch_unpack(m, G, j + 1, st));
    SEM_CUDA_TRY(gm_launch_givens(m, G, st));
    SEM_CUDA_TRY(gm_launch_next(m, G, j, flex, st));
    return SEM_OK;
  };
  // graphs (one rank): everything a step's kernels bake in is the key
  // (buffers are fixed per mesh while G lives); with several ranks the
  // j+1-value allreduces go through NCCL and the steps stay in stream order
  const bool use_graph = m->opt.graph && !m->prof && !m->comm;
  if (use_graph) {
    const int kc = flex ? m->opt.hsmg_coarse_iters : 0;
    if (G->key_flex != (int)flex || G->key_h1c != h1c || G->key_h2c != h2c || G->key_h1 != h1 || G->key_h2 != h2 ||
        G->key_coarse != kc || (int)G->exec.size() != G->restart) {
      G->drop_graphs();
      G->exec.assign(G->restart, nullptr);
      G->key_flex = flex;
      G->key_h1c = h1c;
      G->key_h2c = h2c;
      G->key_h1 = h1;
      G->key_h2 = h2;
      G->key_coarse = kc;
    }
  }
  if (flex) SEM_TRY(hsmg_prepare(m, h1c, h2c, s));
  for (;;) {
    SEM_CUDA_TRY(cudaMemcpyAsync(G->gs_host, G->gs, sizeof(GmScalars), cudaMemcpyDeviceToHost, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (G->gs_host->done) break;
    const int steps = std::min(restart, maxit - G->gs_host->it);
    for (int j = 0; j < steps; ++j) {
      // the cycle ends at the first step that sets cycle_stop: read step j-1's
      // flag while step j is queued (steps after the stop are no-ops)
      if (j >= 2) {
        SEM_CUDA_TRY(cudaEventSynchronize(G->ev_stop[(j - 2) & 1]));
        if (G->stop_host[(j - 2) & 1]) break;
      }
      if (!use_graph) {
        SEM_TRY(arnoldi_step(j, s));
        SEM_CUDA_TRY(cudaMemcpyAsync(&G->stop_host[j & 1], &G->gs->cycle_stop, sizeof(int), cudaMemcpyDeviceToHost, s));
        SEM_CUDA_TRY(cudaEventRecord(G->ev_stop[j & 1], s));
        continue;
      }
      cudaGraphExec_t& ex = G->exec[j];
      if (!ex) {  // capture step j once on the owned stream (joined to s), replay on s
        SEM_CUDA_TRY(cudaEventRecord(m->ev_cap, s));
        SEM_CUDA_TRY(cudaStreamWaitEvent(m->cap_stream, m->ev_cap, 0));
        SEM_CUDA_TRY(cudaStreamBeginCapture(m->cap_stream, cudaStreamCaptureModeThreadLocal));
        const sem_status st = arnoldi_step(j, m->cap_stream);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(m->cap_stream, &g);
        if (st != SEM_OK || ce != cudaSuccess) {
          if (g) cudaGraphDestroy(g);
          if (st != SEM_OK) return st;
          return fail(SEM_ECUDA, std::string("GMRES step capture: ") + cudaGetErrorString(ce));
        }
        const cudaError_t ie = cudaGraphInstantiateWithFlags(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
          ex = nullptr;
          return fail(SEM_ECUDA, std::string("GMRES step graph: ") + cudaGetErrorString(ie));
        }
      }
      SEM_CUDA_TRY(cudaGraphLaunch(ex, s));
      SEM_CUDA_TRY(cudaMemcpyAsync(&G->stop_host[j & 1], &G->gs->cycle_stop, sizeof(int), cudaMemcpyDeviceToHost, s));
      SEM_CUDA_TRY(cudaEventRecord(G->ev_stop[j & 1], s));
    }
    // cycle end: x += M V y, the true residual, the next cycle's v_0
    SEM_CUDA_TRY(gm_launch_cycle_end(m, G, x, flex, s));
    a.u = x;
    a.w = m->w;
    a.skip = nullptr;
    SEM_TRY(ax_dssum_all(m, a, false, s));
    SEM_CUDA_TRY(gm_launch_resid(m, G, bm, s));
    SEM_TRY(allreduce(m, &G->gs->nn, 1, s));
    SEM_CUDA_TRY(gm_launch_start(m, G, 0, flex, s));
  }
  const GmScalars& h = *G->gs_host;
  if (singular && !h.breakdown) {
    SEM_CUDA_TRY(launch_wdot(m, x, nullptr, 3, s));
    SEM_TRY(allreduce(m, &m->sc->red[3], 1, s));
    SEM_CUDA_TRY(launch_sub_mean(m, x, 3, s));
    SEM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  if (iters) *iters = h.it;
  if (rel_res) *rel_res = h.bn > 0 ? h.beta / h.bn : 0.0;
  if (converged) *converged = h.converged || !(h.bn > 0);
  if (m->comm) SEM_TRY(comm_check(m->comm));
  if (h.breakdown) return fail(SEM_EBREAKDOWN, "sem_gmres_solve: breakdown (zero Givens pivot)");
  return SEM_OK;
}

// One first-order velocity-pressure splitting step (reading
// R15; the oracle's O17 in the same order):
//   c_i = dssum(W J (u.grad)u_i);  u~_i = (dssum(B u_i) - dt c_i) / dssum(B)
//   A p = dssum((grad v, u~)) / dt                         (Poisson, CG)
//   (nu A + B / dt) u_i = dssum(B u~_i / dt - W J d p / dx_i)  (Helmholtz, CG x 3)
sem_status sem_pnpn_step(sem_mesh_t m, double* u, double* p, double dt, double nu, double tol, int maxit,
                         int* iters, sem_stream_t stream) {
  SEM_NVTX("sem_pnpn_step");
  SEM_TRY(check_op(m, u, p, "sem_pnpn_step"));
  if (!(dt > 0.0) || !(nu > 0.0) || maxit < 1 || !(tol >= 0.0))
    return fail(SEM_EINVAL, "sem_pnpn_step: dt > 0, nu > 0, maxit >= 1, tol >= 0 required");
  if (m->n_masked_glob != 0)
    return fail(SEM_EINVAL, "sem_pnpn_step: periodic meshes only (no Dirichlet faces; wall boundary conditions "
                            "of the splitting are out of scope)");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = m->nloc;
  SEM_TRY(ensure_cg(m));
  if (!m->MJ) {
    SEM_TRY(dalloc(&m->MJ, 9 * std::max<int64_t>(n, 1), "metric terms"));
    SEM_TRY(dalloc(&m->Bg, std::max<int64_t>(n, 1), "assembled mass"));
    SEM_TRY(dalloc(&m->pn_t, 3 * std::max<int64_t>(n, 1), "step work"));
    SEM_TRY(dalloc(&m->pn_c, 3 * std::max<int64_t>(n, 1), "step work"));
    SEM_TRY(dalloc(&m->pn_r, std::max<int64_t>(n, 1), "step work"));
    SEM_CUDA_TRY(launch_metrics(m, m->MJ, s));
    if (n > 0) SEM_CUDA_TRY(cudaMemcpyAsync(m->Bg, m->B, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    SEM_TRY(sem_gs_op(m, m->Bg, SEM_GS_ADD, stream));
  }
  // 1-2: convection and the predictor u~ (in pn_t)
  SEM_CUDA_TRY(launch_convect(m, u, m->MJ, m->pn_c, s));
  for (int i = 0; i < 3; ++i) {
    double* ti = m->pn_t + i * n;
    SEM_CUDA_TRY(launch_pn_mul(m, m->B, u + i * n, ti, n, s));
    SEM_CUDA_TRY(launch_pn_axpy(m, ti, 1.0, m->pn_c + i * n, -dt, ti, n, s));
    SEM_TRY(sem_gs_op(m, ti, SEM_GS_ADD, stream));
    SEM_CUDA_TRY(launch_pn_div(m, ti, m->Bg, n, s));
  }
  // 3: pressure Poisson
  SEM_CUDA_TRY(launch_wdiv(m, m->pn_t, m->MJ, m->pn_r, s));
  SEM_TRY(sem_gs_op(m, m->pn_r, SEM_GS_ADD, stream));
  SEM_CUDA_TRY(launch_pn_axpy(m, m->pn_r, 1.0 / dt, m->pn_r, 0.0, m->pn_r, n, s));
  int it[4] = {0, 0, 0, 0};
  double rr = 0.0;
  int conv = 0;
  if (m->opt.pnpn_pressure == SEM_PRESSURE_GMRES)
    SEM_TRY(sem_gmres_solve(m, m->pn_r, p, nullptr, nullptr, 1.0, 0.0, tol, maxit, 30, &it[0], &rr, &conv, stream));
  else
    SEM_TRY(sem_cg_solve(m, m->pn_r, p, nullptr, nullptr, 1.0, 0.0, tol, maxit, &it[0], &rr, &conv, stream));
  // 4: velocity Helmholtz with the pressure gradient
  SEM_CUDA_TRY(launch_grad(m, p, m->MJ, m->pn_c, s));
  for (int i = 0; i < 3; ++i) {
    SEM_CUDA_TRY(launch_pn_mul(m, m->B, m->pn_t + i * n, m->pn_r, n, s));
    SEM_CUDA_TRY(launch_pn_axpy(m, m->pn_r, 1.0 / dt, m->pn_c + i * n, -1.0, m->pn_r, n, s));
    SEM_TRY(sem_gs_op(m, m->pn_r, SEM_GS_ADD, stream));
    // the three components share the operator (nu A + B / dt): one Jacobi set-up
    m->reuse_dinv = i > 0 && m->opt.cg_variant == SEM_CG_STANDARD;
    const sem_status stv = sem_cg_solve(m, m->pn_r, u + i * n, nullptr, nullptr, nu, 1.0 / dt, tol, maxit, &it[1 + i],
                                        &rr, &conv, stream);
    m->reuse_dinv = false;
    SEM_TRY(stv);
  }
  if (iters)
    for (int k = 0; k < 4; ++k) iters[k] = it[k];
  return SEM_OK;
}

sem_status sem_cg_solve_host(sem_mesh_t m, const double* b_host, double* x_host, const double* h1, const double* h2,
                             double h1c, double h2c, double tol, int maxit, int* iters, double* rel_res,
                             int* converged, sem_stream_t stream) {
  SEM_NVTX("sem_cg_solve_host");
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
  if (m->opt.cg_variant == SEM_CG_PIPELINED) SEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_input, 0));
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
