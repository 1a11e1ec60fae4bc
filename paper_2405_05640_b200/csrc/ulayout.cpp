// Host plan of the U layout (unique-node CG vectors; see ax_u.cu and
// DESIGN.md "CG vector layout").  Offsets of every unique node, per-element
// gather/scatter descriptors, the shared-node partial buffer S and the
// segmented-sum lists.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

#include "internal.h"

namespace sem {

sem_status build_ulayout(sem_mesh* m, const std::vector<int64_t>& pos) {
  const Topology& T = m->topo;
  const int64_t E = m->E, nEnt = T.nEnt();
  const int64_t M = m->lx - 2, M3 = M * M * M;
  const int shift = m->chunk_shift;
  const int64_t K = m->nchunk;
  // interface entities: owner = lowest sharing rank
  std::vector<int> ifq(nEnt, -1);
  for (size_t q = 0; q < m->iface.ents.size(); ++q) ifq[m->iface.ents[q]] = (int)q;
  const int me = m->comm ? m->comm->rank : 0;
  auto owned = [&](int64_t x) { return ifq[x] < 0 || m->iface.ranks[ifq[x]][0] == me; };
  // unique offsets: interiors, owned entities, then replicas owned elsewhere
  std::vector<int64_t> uoff(nEnt, -1);
  int64_t off = E * M3;
  for (int pass = 0; pass < 2; ++pass) {
    // faces and edges start 16-byte aligned (bulk copies); entity ids run
    // faces, edges, vertices, so only the start of each pass needs padding
    // (pads are zero in every vector and never written)
    if (off & 1) ++off;
    for (int64_t x = 0; x < nEnt; ++x)
      if (owned(x) == (pass == 0)) {
        uoff[x] = off;
        off += T.ent_nodes(x);
      }
    if (pass == 0) m->n_own = off;  // the dot products run over [0, n_own)
  }
  m->n_u = off;
  // S slots for entities with >= 2 local copies; descriptors per element slot
  std::vector<int64_t> soff(nEnt, -1);
  int64_t S = 0;
  for (int64_t x = 0; x < nEnt; ++x) {
    const int mult = T.ent_ptr[x + 1] - T.ent_ptr[x];
    if (mult >= 2) {
      soff[x] = S;
      S += (int64_t)mult * T.ent_nodes(x);
    }
  }
  std::vector<int64_t> gdesc((size_t)E * kSlots), wdesc((size_t)E * kSlots);
  for (int64_t x = 0; x < nEnt; ++x) {
    const int c0 = T.ent_ptr[x], mult = T.ent_ptr[x + 1] - c0;
    const bool iface = ifq[x] >= 0;
    const bool zero = (T.ent_flags[x] & kEntMasked) && !iface;
    for (int k = 0; k < mult; ++k) {
      const int64_t cp = T.ent_copy[c0 + k];
      const size_t at = (size_t)(cp >> 8) * kSlots + ((cp >> 3) & 31);
      gdesc[at] = (uoff[x] << 4) | (k == 0 ? 8 : 0) | (cp & 7);
      if (mult == 1) wdesc[at] = (uoff[x] << 2) | 2 | (zero ? 1 : 0);
      else wdesc[at] = (soff[x] + (int64_t)k * T.ent_nodes(x)) << 2;
    }
  }
  // segmented sums, grouped by the chunk of the last copy (group K: interface)
  std::vector<int64_t> nf(K + 3, 0), ne(K + 3, 0), nv(K + 3, 0), grp(nEnt, -1);
  for (int64_t x = 0; x < nEnt; ++x) {
    const int c0 = T.ent_ptr[x], mult = T.ent_ptr[x + 1] - c0;
    if (mult < 2) continue;
    int64_t g = K;
    if (ifq[x] < 0) {
      int64_t last = 0;
      for (int c = c0; c < c0 + mult; ++c) last = std::max(last, pos[T.ent_copy[c] >> 8]);
      g = last >> shift;
    }
    grp[x] = g;
    (x < T.nF ? nf : (x < T.nF + T.nEd ? ne : nv))[g + 1]++;
  }
  for (int64_t g = 0; g <= K; ++g) {
    nf[g + 1] += nf[g];
    ne[g + 1] += ne[g];
    nv[g + 1] += nv[g];
  }
  m->useg_f.assign(nf.begin(), nf.begin() + K + 2);
  m->useg_e.assign(ne.begin(), ne.begin() + K + 2);
  m->useg_v.assign(nv.begin(), nv.begin() + K + 2);
  m->nseg_e = ne[K + 1];
  std::vector<int64_t> fseg(2 * (size_t)nf[K + 1]), xseg(3 * (size_t)(ne[K + 1] + nv[K + 1]));
  {
    std::vector<int64_t> ff(nf.begin(), nf.begin() + K + 1), fe(ne.begin(), ne.begin() + K + 1),
        fv(nv.begin(), nv.begin() + K + 1);
    for (int64_t x = 0; x < nEnt; ++x) {
      if (grp[x] < 0) continue;
      const int64_t g = grp[x];
      const int mult = T.ent_ptr[x + 1] - T.ent_ptr[x];
      const int64_t mk = ((T.ent_flags[x] & kEntMasked) && ifq[x] < 0) ? kFaceMasked : 0;
      if (x < T.nF) {
        const int64_t q = ff[g]++;
        fseg[2 * q] = uoff[x];
        fseg[2 * q + 1] = soff[x] | mk;
      } else {
        const int64_t q = (x < T.nF + T.nEd) ? fe[g]++ : ne[K + 1] + fv[g]++;
        xseg[3 * q] = uoff[x];
        xseg[3 * q + 1] = soff[x] | mk;
        xseg[3 * q + 2] = mult;
      }
    }
  }
  std::vector<int64_t> if_uoff(m->iface.ents.size());
  for (size_t q = 0; q < m->iface.ents.size(); ++q) if_uoff[q] = uoff[m->iface.ents[q]];
  auto up = [&](auto** d, const auto& h) -> sem_status {
    using V = typename std::remove_reference<decltype(h)>::type::value_type;
    if (*d) cudaFree(*d);
    *d = nullptr;
    if (h.empty()) return SEM_OK;
    if (cudaMalloc((void**)d, sizeof(V) * h.size()) != cudaSuccess) return fail(SEM_ENOMEM, "cudaMalloc(U plan)");
    if (cudaMemcpy(*d, h.data(), sizeof(V) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SEM_ECUDA, "upload U plan");
    return SEM_OK;
  };
  SEM_TRY_ST(up(&m->d_gdesc, gdesc));
  SEM_TRY_ST(up(&m->d_wdesc, wdesc));
  SEM_TRY_ST(up(&m->d_fseg, fseg));
  SEM_TRY_ST(up(&m->d_xseg, xseg));
  SEM_TRY_ST(up(&m->d_if_uoff, if_uoff));
  if (m->d_Su) cudaFree(m->d_Su);
  m->d_Su = nullptr;
  if (S > 0 && cudaMalloc((void**)&m->d_Su, sizeof(double) * S) != cudaSuccess)
    return fail(SEM_ENOMEM, "cudaMalloc(S)");
  return SEM_OK;
}

void ulayout_free(sem_mesh* m) {
  void* ptrs[] = {m->d_gdesc, m->d_wdesc, m->d_Su, m->d_fseg, m->d_xseg, m->d_if_uoff,
                  m->ux, m->ur, m->up, m->uw, m->udinv};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

}  // namespace sem
