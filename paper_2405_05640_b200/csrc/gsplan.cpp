// Host-side gather-scatter plans (readings R7, R8).
//
//  * the element descriptors of the element-gather schedule (gs_elem.cu):
//    per (element, entity slot) the copy-list pointer, the copy count, the
//    action (own value / masked / sum) and the element's own orientation;
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

static inline uint32_t copy_offset(const sem_mesh* m, int64_t cp, int n) {
  return (uint32_t)((cp >> 8) * m->n3 + copy_node_offset(m->lx, (int)((cp >> 3) & 31), (int)(cp & 7), n));
}

// Nodal plan over the listed entities: classes (m, masked); m = 2 pairs
// interleaved (one 8-byte load per group), else struct of arrays; groups of
// a class in the order of their first copy's offset.
static sem_status build_nodal(sem_mesh* m, const std::vector<int32_t>& ents, uint32_t** d_idx,
                              std::vector<GsClass>* cls_out, const char* what) {
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
        gidx[(size_t)(cbase[cl] + cc * gcount[cl] + g)] = copy_offset(m, T.ent_copy[c0c + cc], n);
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
}

// Partner maps of the element gather (gs_elem.cu): for an own copy (slot s,
// orientation o) and another copy (slot ps, orientation po) of the same
// entity, the other copy's local node holding the own node with loop
// coordinates (a, b) -- face (a, b) = the face-interior position (u - 1,
// v - 1) in the face's own axes, edge (a, 0) = position along the edge,
// vertex (0, 0) -- is o00 + a qa + b qb (orientation maps are affine).
// Tables: faces [6][8][6][8], edges [12][2][12][2], vertices [8][8]; entry
// int2 {o00, qa | qb << 16}.
static int own_node(int lx, int s, int a, int b) {
  const int N = lx - 1;
  int i, j, k;
  if (s < kEdgeSlot0) {
    const int side = (s & 1) ? N : 0, ax = s >> 1;
    i = ax == 0 ? side : 1 + a;
    j = ax == 0 ? 1 + a : (ax == 1 ? side : 1 + b);
    k = ax == 2 ? side : 1 + b;
  } else if (s < kVertSlot0) {
    const int ed = s - kEdgeSlot0, ax = ed >> 2, q = ed & 3;
    const int p = (q & 1) * N, r = (q >> 1) * N;
    i = ax == 0 ? 1 + a : p;
    j = ax == 0 ? p : (ax == 1 ? 1 + a : r);
    k = ax == 2 ? 1 + a : r;
  } else {
    const int c = s - kVertSlot0;
    i = (c & 1) * N;
    j = ((c >> 1) & 1) * N;
    k = (c >> 2) * N;
  }
  return i + lx * (j + lx * k);
}
// canonical index of local node (i, j, k) of copy (s, o): the inverse of
// copy_node_offset
static int canonical_of(int lx, int s, int o, int q) {
  const int M = lx - 2, i = q % lx, j = (q / lx) % lx, k = q / (lx * lx);
  if (s < kEdgeSlot0) {
    const int ax = s >> 1;
    const int u = ax == 0 ? j : i, v = ax == 2 ? j : k;
    const int du = (o & 1) ? M - u : u - 1, dv = (o & 2) ? M - v : v - 1;
    const int a = (o & 4) ? dv : du, b = (o & 4) ? du : dv;
    return a + M * b;
  }
  if (s < kVertSlot0) {
    const int ax = (s - kEdgeSlot0) >> 2;
    const int t = ax == 0 ? i : (ax == 1 ? j : k);
    return (o & 1) ? M - t : t - 1;
  }
  return 0;
}
int gs_qtab_index(int s, int o, int ps, int po) {
  if (s < kEdgeSlot0) return ((s * 8 + o) * 6 + ps) * 8 + po;
  if (s < kVertSlot0) return 2304 + (((s - kEdgeSlot0) * 2 + (o & 1)) * 12 + (ps - kEdgeSlot0)) * 2 + (po & 1);
  return 2304 + 576 + (s - kVertSlot0) * 8 + (ps - kVertSlot0);
}
static std::vector<int32_t> build_qtab(int lx) {
  const int M = lx - 2;
  std::vector<int32_t> tab(2 * (2304 + 576 + 64), 0);
  auto fill = [&](int s, int o, int ps, int po) {
    auto off = [&](int a, int b) { return copy_node_offset(lx, ps, po, canonical_of(lx, s, o, own_node(lx, s, a, b))); };
    const int o00 = off(0, 0);
    int qa = 0, qb = 0;
    if (s < kVertSlot0 && M >= 2) qa = off(1, 0) - o00;
    if (s < kEdgeSlot0 && M >= 2) qb = off(0, 1) - o00;
    const int x = gs_qtab_index(s, o, ps, po);
    tab[2 * x] = o00;
    tab[2 * x + 1] = (qa & 0xffff) | (qb << 16);
  };
  if (M >= 1) {
    for (int s = 0; s < 6; ++s)
      for (int o = 0; o < 8; ++o)
        for (int ps = 0; ps < 6; ++ps)
          for (int po = 0; po < 8; ++po) fill(s, o, ps, po);
    for (int s = kEdgeSlot0; s < kVertSlot0; ++s)
      for (int o = 0; o < 2; ++o)
        for (int ps = kEdgeSlot0; ps < kVertSlot0; ++ps)
          for (int po = 0; po < 2; ++po) fill(s, o, ps, po);
  }
  for (int s = kVertSlot0; s < kSlots; ++s)
    for (int ps = kVertSlot0; ps < kSlots; ++ps) fill(s, 0, ps, 0);
  return tab;
}

// Element descriptors (gs_elem.cu): ptr | m << 32 | action << 40 | orient << 48
// | global multiplicity << 56;
// action 0: own value (one unmasked copy, or an interface entity: the
// exchange writes the rank-summed total, 0 if masked, into every copy
// before the gather reads it), 1: masked, 2: sum over the copies.  Also
// the scratch of the out-of-place sem_ax_dssum and the pAp tickets.
static sem_status build_elem_desc(sem_mesh* m) {
  const Topology& T = m->topo;
  const int64_t E = m->E;
  std::vector<uint64_t> desc((size_t)E * kSlots);
  for (int64_t e = 0; e < E; ++e)
    for (int s = 0; s < kSlots; ++s) {
      const int32_t x = T.elem_ent[(size_t)e * kSlots + s];
      const int c0 = T.ent_ptr[x], c1 = T.ent_ptr[x + 1], mc = c1 - c0;
      if (mc > 255) return fail(SEM_EINVAL, "sem_mesh_create: an entity with more than 255 copies");
      int orient = -1;
      for (int c = c0; c < c1; ++c) {
        const int64_t cp = T.ent_copy[c];
        if ((cp >> 8) == e && (int)((cp >> 3) & 31) == s) orient = (int)(cp & 7);
      }
      if (orient < 0) return fail(SEM_EINVAL, "sem_mesh_create: element missing from its entity's copy list");
      const uint8_t fl = T.ent_flags[x];
      const int gc = m->ent_gcount_h.empty() ? mc : m->ent_gcount_h[x];  // global multiplicity
      if (gc > 255) return fail(SEM_EINVAL, "sem_mesh_create: a node with more than 255 copies");
      const int act = (fl & kEntInterface) ? 0 : ((fl & kEntMasked) ? 1 : (mc > 1 ? 2 : 0));
      desc[(size_t)e * kSlots + s] = (uint64_t)(uint32_t)c0 | ((uint64_t)mc << 32) | ((uint64_t)act << 40) |
                                     ((uint64_t)orient << 48) | ((uint64_t)gc << 56);
    }
  SEM_TRY_ST(upload(&m->d_gs_desc, desc, "element gs descriptors"));
  SEM_TRY_ST(upload(&m->d_gs_qtab, build_qtab(m->lx), "element gs partner maps"));
  if (!m->wt && m->nloc > 0 && cudaMalloc((void**)&m->wt, sizeof(double) * m->nloc) != cudaSuccess) {
    cudaGetLastError();
    return fail(SEM_ENOMEM, "cudaMalloc(gs scratch)");
  }
  const int64_t ntk = (E + kPapGroup - 1) / kPapGroup + 1;
  if (!m->pap_tk) {
    if (cudaMalloc((void**)&m->pap_tk, sizeof(unsigned) * ntk) != cudaSuccess) {
      cudaGetLastError();
      return fail(SEM_ENOMEM, "cudaMalloc(pAp tickets)");
    }
    if (cudaMemset(m->pap_tk, 0, sizeof(unsigned) * ntk) != cudaSuccess) return fail(SEM_ECUDA, "memset tickets");
  }
  return SEM_OK;
}

// Called at mesh creation (pos = processing position of every element) and
// when the fused-gs options change.
sem_status build_gs_plans(sem_mesh* m, const std::vector<int64_t>& pos) {
  const Topology& T = m->topo;
  gs_plans_free(m);
  if (m->E > 0) SEM_TRY_ST(build_elem_desc(m));
  // entities needing an action: a sum (several copies) or a mask; the
  // interface entities are finished by the exchange (comm.cpp)
  std::vector<int32_t> act;
  for (int64_t x = 0; x < T.nEnt(); ++x) {
    const int c = T.ent_ptr[x + 1] - T.ent_ptr[x];
    if (!(c > 1 || (T.ent_flags[x] & kEntMasked))) continue;
    if (T.ent_flags[x] & kEntInterface) continue;
    act.push_back((int32_t)x);
  }
  SEM_TRY_ST(build_nodal(m, act, &m->d_gidx, &m->gs_cls, "gs plan"));
  // launch segments: one rank -> one launch; several ranks -> the boundary
  // elements (positions [0, n_boundary)) and the interior
  m->seg.assign(1, 0);
  if (m->comm && m->n_boundary > 0 && m->n_boundary < m->E) m->seg.push_back(m->n_boundary);
  m->seg.push_back(m->E);

  return SEM_OK;
}

}  // namespace sem
