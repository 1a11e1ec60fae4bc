// Host-side gather-scatter plans (readings R7, R8).
//
//  * the standalone nodal plan (k_gs_nodal): one group per shared node that
//    needs a sum or a mask, m uint32 copy offsets per group, classes (m,
//    masked); used by sem_gs_op, the set-up passes (RHS, Jacobi), the
//    unfused schedule and the multi-GPU local pass;
//  * the fused plan (FinArgs; the finalizer kernel k_gs_fin beside the
//    operator launch): every entity whose copies all lie in one launch
//    segment is listed under its owner, the position of its last copy, with
//    the positions whose completion flags it must wait for; entities
//    spanning two launch segments or with more than kFinMaxM copies form the
//    residual nodal plan run after the launches.
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
  void* ptrs[] = {m->d_gidx, m->d_fin, m->d_fidx, m->d_fdep, m->d_fflag, m->d_ctl,
                  m->d_fbcnt, m->d_fbpart, m->d_fdone, m->d_ridx};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  m->d_gidx = nullptr;
  m->d_fin = nullptr;
  m->d_fidx = nullptr;
  m->d_fdep = nullptr;
  m->d_fflag = nullptr;
  m->d_ctl = nullptr;
  m->d_fbcnt = nullptr;
  m->d_fbpart = nullptr;
  m->d_fdone = nullptr;
  m->d_ridx = nullptr;
  m->gs_cls.clear();
  m->res_cls.clear();
  m->fused = false;
}

// The fused plan (FinArgs) for the launch segments m->seg of positions.
static sem_status build_fused(sem_mesh* m, const std::vector<int64_t>& pos, const std::vector<int32_t>& act) {
  const Topology& T = m->topo;
  const int64_t E = m->E;
  const int nseg = (int)m->seg.size() - 1;
  std::vector<int> seg_of_pos(E);
  for (int s = 0; s < nseg; ++s)
    for (int64_t q = m->seg[s]; q < m->seg[s + 1]; ++q) seg_of_pos[q] = s;
  // per owner position (the entity's last copy) its entities
  std::vector<std::vector<int32_t>> lists(2 * (size_t)E);
  std::vector<int32_t> residual;
  for (int32_t x : act) {
    const int c0 = T.ent_ptr[x], c1 = T.ent_ptr[x + 1];
    int64_t lo = INT64_MAX, hi = -1;
    for (int c = c0; c < c1; ++c) {
      const int64_t p = pos[T.ent_copy[c] >> 8];
      lo = std::min(lo, p);
      hi = std::max(hi, p);
    }
    const int s = seg_of_pos[hi];
    if (c1 - c0 > kFinMaxM || lo < m->seg[s]) {
      residual.push_back(x);
      continue;
    }
    lists[2 * (size_t)hi].push_back(x);
  }
  std::vector<FinDesc> desc(2 * (size_t)E);
  std::vector<uint32_t> idx;
  std::vector<int32_t> dep;
  for (int64_t q = 0; q < E; ++q)
    for (int l = 0; l < 2; ++l) {
      FinDesc& d = desc[2 * (size_t)q + l];
      d = FinDesc{};
      const std::vector<int32_t>& L = lists[2 * (size_t)q + l];
      d.start = (uint32_t)idx.size();
      d.dep_start = (uint32_t)dep.size();
      if (L.empty()) continue;
      std::vector<int64_t> deps;
      for (int mm = 1; mm <= kFinMaxM; ++mm) {
        while (idx.size() & 3) idx.push_back(0);  // each class 16-byte aligned
        int64_t groups = 0;
        for (int32_t x : L) {
          const int c0 = T.ent_ptr[x], c1 = T.ent_ptr[x + 1];
          if (c1 - c0 != mm) continue;
          const bool masked = (T.ent_flags[x] & kEntMasked) != 0;
          for (int n = 0; n < T.ent_nodes(x); ++n) {
            for (int c = c0; c < c1; ++c) {
              uint32_t o = copy_offset(m, T.ent_copy[c], n);
              if (c == c0 && masked) o |= kFinMasked;
              idx.push_back(o);
            }
            ++groups;
          }
          for (int c = c0; c < c1; ++c) deps.push_back(pos[T.ent_copy[c] >> 8]);
        }
        if (groups > 0xffff) return fail(SEM_EINVAL, "fused gather-scatter plan: too many groups per CTA");
        d.cnt[mm - 1] = (uint16_t)groups;
      }
      std::sort(deps.begin(), deps.end());
      deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
      for (int64_t p : deps) dep.push_back((int32_t)p);  // the owner itself included (another kernel)
      if (dep.size() - d.dep_start > 0xffff) return fail(SEM_EINVAL, "fused gather-scatter plan: too many dependencies");
      d.ndep = (uint16_t)(dep.size() - d.dep_start);
    }
  if (idx.size() >= (size_t(1) << 32)) return fail(SEM_EINVAL, "fused gather-scatter plan too large");
  while (idx.size() & 3) idx.push_back(0);
  if (dep.empty()) dep.push_back(0);
  SEM_TRY_ST(upload(&m->d_fin, desc, "fused gs descriptors"));
  SEM_TRY_ST(upload(&m->d_fidx, idx, "fused gs offsets"));
  SEM_TRY_ST(upload(&m->d_fdep, dep, "fused gs dependencies"));
  // completion flags, tickets and the pAp batch counters start at 0
  const int64_t nb = E / kFinBatch + 2 * nseg + 1;
  std::vector<unsigned long long> z64((size_t)std::max<int64_t>(E, 1), 0ull);
  SEM_TRY_ST(upload(&m->d_fflag, z64, "fused gs flags"));
  SEM_TRY_ST(upload(&m->d_fbcnt, std::vector<unsigned>((size_t)nb, 0u), "fused gs batch counters"));
  SEM_TRY_ST(upload(&m->d_fbpart, std::vector<double>((size_t)nb, 0.0), "fused gs batch sums"));
  SEM_TRY_ST(upload(&m->d_fdone, std::vector<unsigned>((size_t)nseg, 0u), "fused gs done counters"));
  SEM_TRY_ST(build_nodal(m, residual, &m->d_ridx, &m->res_cls, "residual gs plan"));
  m->fused = true;
  return SEM_OK;
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
  SEM_TRY_ST(build_nodal(m, act, &m->d_gidx, &m->gs_cls, "gs plan"));
  // launch segments: one rank -> one launch; several ranks -> the boundary
  // elements (positions [0, n_boundary)) and the interior
  m->seg.assign(1, 0);
  if (m->comm && m->n_boundary > 0 && m->n_boundary < m->E) m->seg.push_back(m->n_boundary);
  m->seg.push_back(m->E);
  // launch control blocks (tickets, epochs): the persistent operator per
  // segment, plain sem_ax, the finalizer kernel per segment
  SEM_TRY_ST(upload(&m->d_ctl, std::vector<LaunchCtl>(2 * m->seg.size() - 1, LaunchCtl{}), "launch control"));
  if (m->opt.fused_gs && m->E > 0) SEM_TRY_ST(build_fused(m, pos, act));
  return SEM_OK;
}

}  // namespace sem
