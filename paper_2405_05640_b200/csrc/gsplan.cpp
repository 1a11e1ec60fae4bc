// Host-side gather-scatter plans (readings R7, R8).
//
//  * the standalone nodal plan (k_gs_nodal): one group per shared node that
//    needs a sum or a mask, m uint32 copy offsets per group, classes (m,
//    masked); used by sem_gs_op, the set-up passes (RHS, Jacobi), the
//    unfused schedule and the multi-GPU local pass;
// Copies are listed in ascending element order (the entity CSR order), so
// every sum is taken in the oracle's order (bit-exact on one GPU).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

#include "internal.h"

namespace sem {

template <class V>
static sem_status upload(V** d, const std::vector<V>& h, const char* what) {
  if (*d) cudaFree(*d);
  *d = nullptr;
  if (h.empty()) return SEM_OK;
  if (cudaMalloc((void**)d, sizeof(V) * h.size()) != cudaSuccess) {
    cudaGetLastError();
    return fail(SEM_ENOMEM, std::string("cudaMalloc(") + what + ")");
  }
  if (cudaMemcpy(*d, h.data(), sizeof(V) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(SEM_ECUDA, std::string("upload ") + what);
  return SEM_OK;
}

// host twin of xlast_pos (device_common.cuh): the x-planes-last element layout
static inline int xlast_host(int lx, int q) {
  const int nt = lx * lx, i = q % lx, r = q / lx, g = r >> 2, rr = r & 3;
  const int gs = std::min(4, nt - 4 * g), gb = 4 * g * lx;
  return (i >= 1 && i <= lx - 2) ? gb + rr * (lx - 2) + (i - 1) : gb + gs * (lx - 2) + (i == lx - 1 ? gs : 0) + rr;
}
static inline uint32_t copy_offset(const sem_mesh* m, int64_t cp, int n, bool xl) {
  const int lo = copy_node_offset(m->lx, (int)((cp >> 3) & 31), (int)(cp & 7), n);
  return (uint32_t)((cp >> 8) * m->n3 + (xl ? xlast_host(m->lx, lo) : lo));
}

// Nodal plan over the listed entities: classes (m, masked); m = 2 pairs
// interleaved (one 8-byte load per group), else struct of arrays; groups of
// a class in the order of their first copy's offset.
static sem_status build_nodal(sem_mesh* m, const std::vector<int32_t>& ents, uint32_t** d_idx,
                              std::vector<GsClass>* cls_out, const char* what, bool xl) {
  const Topology& T = m->topo;
  cls_out->clear();
  int maxm = 1;
  for (int32_t x : ents) maxm = std::max(maxm, T.ent_ptr[x + 1] - T.ent_ptr[x]);
  const int ncls = 2 * maxm;  // class (m, masked) -> 2 (m - 1) + masked
  auto cls_of = [&](int32_t x) {
    return 2 * (T.ent_ptr[x + 1] - T.ent_ptr[x] - 1) + ((T.ent_flags[x] & kEntMasked) ? 1 : 0);
  };
  std::vector<int64_t> gcount(ncls, 0), cbase(ncls, 0), cfill(ncls, 0);
  for (int32_t x : ents) gcount[cls_of(x)] += T.ent_nodes(x);
  int64_t total = 0;
  for (int cl = 0; cl < ncls; ++cl) {
    if (gcount[cl] == 0) continue;
    if (cl / 2 + 1 == 2) total = (total + 1) & ~int64_t(1);  // pair classes: 8-byte aligned
    cbase[cl] = total;
    GsClass g;
    g.base = total;
    g.count = gcount[cl];
    g.m = cl / 2 + 1;
    g.masked = cl & 1;
    cls_out->push_back(g);
    total += g.count * g.m;
  }
  std::vector<uint32_t> gidx((size_t)total);
  for (int32_t x : ents) {
    const int c0c = T.ent_ptr[x], mult = T.ent_ptr[x + 1] - c0c;
    const int cl = cls_of(x);
    for (int n = 0; n < T.ent_nodes(x); ++n) {
      const int64_t g = cfill[cl]++;
      for (int cc = 0; cc < mult; ++cc)
        gidx[(size_t)(cbase[cl] + cc * gcount[cl] + g)] = copy_offset(m, T.ent_copy[c0c + cc], n, xl);
    }
  }
  for (const GsClass& g : *cls_out) {
    std::vector<int64_t> ord((size_t)g.count);
    for (int64_t q = 0; q < g.count; ++q) ord[(size_t)q] = q;
    const uint32_t* first = gidx.data() + g.base;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return first[a] < first[b]; });
    std::vector<uint32_t> tmp((size_t)(g.count * g.m));
    for (int k = 0; k < g.m; ++k)
      for (int64_t q = 0; q < g.count; ++q)
        tmp[(size_t)(g.m == 2 ? 2 * q + k : k * g.count + q)] = gidx[(size_t)(g.base + k * g.count + ord[(size_t)q])];
    std::copy(tmp.begin(), tmp.end(), gidx.begin() + g.base);
  }
  return upload(d_idx, gidx, what);
}

void gs_plans_free(sem_mesh* m) {
  if (m->d_gidx) cudaFree(m->d_gidx);
  m->d_gidx = nullptr;
  m->gs_cls.clear();
  if (m->d_gidx_xl) cudaFree(m->d_gidx_xl);
  m->d_gidx_xl = nullptr;
  m->gs_cls_xl.clear();
}

// Called at mesh creation (pos = processing position of every element) and
// when the fused-gs options change.
sem_status build_gs_plans(sem_mesh* m, const std::vector<int64_t>& pos) {
  const Topology& T = m->topo;
  gs_plans_free(m);
  // entities needing an action: a sum (several copies) or a mask; the
  // interface entities are finished by the exchange (comm.cpp)
  std::vector<int32_t> act;
  for (int64_t x = 0; x < T.nEnt(); ++x) {
    const int c = T.ent_ptr[x + 1] - T.ent_ptr[x];
    if (!(c > 1 || (T.ent_flags[x] & kEntMasked))) continue;
    if (T.ent_flags[x] & kEntInterface) continue;
    act.push_back((int32_t)x);
  }
  SEM_TRY_ST(build_nodal(m, act, &m->d_gidx, &m->gs_cls, "gs plan", false));
  SEM_TRY_ST(build_nodal(m, act, &m->d_gidx_xl, &m->gs_cls_xl, "gs plan (x-planes-last layout)", true));
  // launch segments: one rank -> one launch; several ranks -> the boundary
  // elements (positions [0, n_boundary)) and the interior
  m->seg.assign(1, 0);
  if (m->comm && m->n_boundary > 0 && m->n_boundary < m->E) m->seg.push_back(m->n_boundary);
  m->seg.push_back(m->E);

  return SEM_OK;
}

}  // namespace sem
