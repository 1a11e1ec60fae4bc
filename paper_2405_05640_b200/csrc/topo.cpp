// Topological numbering and gather-scatter plan (host, once per mesh).
//
// "only unit-depth communication is necessary in a so-called
// gather-scatter phase"; "The only asymmetry that is introduced
// is through the gather-scatter operation".  Reading R7: two
// local nodes are the same global node iff they are the same vertex, or the
// same interior point of the same edge or face, where edges and faces are
// identified by their (sorted) global vertex ids from the connectivity.
//
// Each shared node belongs to exactly one ENTITY (a vertex, an edge interior
// or a face interior).  The node order inside an entity is canonical and
// depends only on global vertex ids:
//   edge: from the smaller to the larger vertex id;
//   face: origin at the corner with the smallest id, first axis toward the
//         adjacent corner with the smaller id, second axis toward the other.
// A copy of an entity in element e is (e, slot, orient); slot is the local
// face (0..5: r-,r+,s-,s+,t-,t+), edge (6..17) or vertex (18..25) index.
#include <algorithm>
#include <array>
#include <string>
#include <unordered_map>

#include "internal.h"

namespace sem {

namespace {

struct KeyHash {
  size_t operator()(const std::array<int64_t, 4>& k) const {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < 4; ++i) {
      h ^= (uint64_t)k[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 1099511628211ull;
    }
    return (size_t)h;
  }
};

// corner slot of the (u,v) corner of local face f
int face_corner(int f, int u, int v) {
  const int ax = f >> 1, side = f & 1;
  int a, b, c;
  if (ax == 0) { a = side; b = u; c = v; }
  else if (ax == 1) { a = u; b = side; c = v; }
  else { a = u; b = v; c = side; }
  return a + 2 * b + 4 * c;
}
// corner slots of the start/end of local edge ed (0..11)
void edge_corners(int ed, int* s0, int* s1) {
  const int ax = ed >> 2, q = ed & 3, lo = q & 1, hi = q >> 1;
  int a0, b0, c0;
  if (ax == 0) { a0 = 0; b0 = lo; c0 = hi; }
  else if (ax == 1) { a0 = lo; b0 = 0; c0 = hi; }
  else { a0 = lo; b0 = hi; c0 = 0; }
  *s0 = a0 + 2 * b0 + 4 * c0;
  *s1 = *s0 + (ax == 0 ? 1 : ax == 1 ? 2 : 4);
}

}  // namespace

int copy_node_offset(int lx, int slot, int orient, int n) {
  const int N = lx - 1, m = lx - 2;
  int i, j, k;
  if (slot < kEdgeSlot0) {  // face interior, canonical n = a + m b
    const int f = slot, a = n % m, b = n / m;
    const int du = (orient & 4) ? b : a, dv = (orient & 4) ? a : b;
    const int u = 1 + ((orient & 1) ? m - 1 - du : du);
    const int v = 1 + ((orient & 2) ? m - 1 - dv : dv);
    const int side = (f & 1) ? N : 0, ax = f >> 1;
    if (ax == 0) { i = side; j = u; k = v; }
    else if (ax == 1) { i = u; j = side; k = v; }
    else { i = u; j = v; k = side; }
  } else if (slot < kVertSlot0) {  // edge interior
    const int ed = slot - kEdgeSlot0, ax = ed >> 2, q = ed & 3;
    const int t = 1 + ((orient & 1) ? m - 1 - n : n);
    const int p = (q & 1) * N, r = (q >> 1) * N;
    if (ax == 0) { i = t; j = p; k = r; }
    else if (ax == 1) { i = p; j = t; k = r; }
    else { i = p; j = r; k = t; }
  } else {  // vertex
    const int c = slot - kVertSlot0;
    i = (c & 1) * N; j = ((c >> 1) & 1) * N; k = (c >> 2) * N;
  }
  return i + lx * (j + lx * k);
}

std::string build_topology(int64_t E, int N, const int64_t* conn, const int8_t* bc,
                           Topology* T) {
  T->E = E; T->N = N; T->lx = N + 1; T->m = N - 1;
  std::unordered_map<std::array<int64_t, 4>, int32_t, KeyHash> fmap, emap, vmap;
  fmap.reserve((size_t)E * 4); emap.reserve((size_t)E * 4); vmap.reserve((size_t)E * 2);
  std::vector<int32_t> elem_ent((size_t)E * kSlots);
  std::vector<uint8_t> elem_orient((size_t)E * kSlots, 0);
  std::vector<std::array<int64_t, 4>> fkeys, ekeys, vkeys;

  for (int64_t e = 0; e < E; ++e) {
    const int64_t* g = conn + e * 8;
    for (int a = 0; a < 8; ++a)
      for (int b = a + 1; b < 8; ++b)
        if (g[a] == g[b])
          return "element " + std::to_string(e) + " has repeated vertex id " + std::to_string(g[a]) +
                 " (a periodic direction needs >= 3 elements)";
    for (int a = 0; a < 8; ++a)
      if (g[a] < 0) return "negative vertex id in element " + std::to_string(e);
    // faces
    for (int f = 0; f < 6; ++f) {
      int64_t c[2][2];
      for (int v = 0; v < 2; ++v)
        for (int u = 0; u < 2; ++u) c[u][v] = g[face_corner(f, u, v)];
      std::array<int64_t, 4> key = {c[0][0], c[1][0], c[0][1], c[1][1]};
      std::sort(key.begin(), key.end());
      auto it = fmap.find(key);
      int32_t id;
      if (it == fmap.end()) {
        id = (int32_t)fkeys.size();
        fmap.emplace(key, id);
        fkeys.push_back(key);
      } else {
        id = it->second;
      }
      // canonical frame
      int u0 = 0, v0 = 0;
      for (int v = 0; v < 2; ++v)
        for (int u = 0; u < 2; ++u)
          if (c[u][v] < c[u0][v0]) { u0 = u; v0 = v; }
      const int64_t nu = c[1 - u0][v0], nv = c[u0][1 - v0];
      const int swap = (nu < nv) ? 0 : 1;
      elem_ent[e * kSlots + f] = id;
      elem_orient[e * kSlots + f] = (uint8_t)(u0 | (v0 << 1) | (swap << 2));
    }
    // edges
    for (int ed = 0; ed < 12; ++ed) {
      int s0, s1;
      edge_corners(ed, &s0, &s1);
      std::array<int64_t, 4> key = {std::min(g[s0], g[s1]), std::max(g[s0], g[s1]), -1, -1};
      auto it = emap.find(key);
      int32_t id;
      if (it == emap.end()) {
        id = (int32_t)ekeys.size();
        emap.emplace(key, id);
        ekeys.push_back(key);
      } else {
        id = it->second;
      }
      elem_ent[e * kSlots + kEdgeSlot0 + ed] = id;
      elem_orient[e * kSlots + kEdgeSlot0 + ed] = (uint8_t)(g[s0] > g[s1] ? 1 : 0);
    }
    // vertices
    for (int c = 0; c < 8; ++c) {
      std::array<int64_t, 4> key = {g[c], -1, -1, -1};
      auto it = vmap.find(key);
      int32_t id;
      if (it == vmap.end()) {
        id = (int32_t)vkeys.size();
        vmap.emplace(key, id);
        vkeys.push_back(key);
      } else {
        id = it->second;
      }
      elem_ent[e * kSlots + kVertSlot0 + c] = id;
    }
  }
  T->nF = (int64_t)fkeys.size();
  T->nEd = (int64_t)ekeys.size();
  T->nV = (int64_t)vkeys.size();
  const int64_t nEnt = T->nEnt();
  if (nEnt >= (int64_t)INT32_MAX) return "too many entities";
  // global entity id: faces [0,nF), edges [nF, nF+nEd), vertices after
  for (int64_t e = 0; e < E; ++e) {
    for (int s = kEdgeSlot0; s < kVertSlot0; ++s) elem_ent[e * kSlots + s] += (int32_t)T->nF;
    for (int s = kVertSlot0; s < kSlots; ++s) elem_ent[e * kSlots + s] += (int32_t)(T->nF + T->nEd);
  }
  // CSR of copies (ascending element, then slot)
  T->ent_ptr.assign(nEnt + 1, 0);
  for (int64_t q = 0; q < E * kSlots; ++q) T->ent_ptr[elem_ent[q] + 1]++;
  for (int64_t x = 0; x < nEnt; ++x) T->ent_ptr[x + 1] += T->ent_ptr[x];
  T->ent_copy.assign(T->ent_ptr[nEnt], 0);
  std::vector<int32_t> fill(T->ent_ptr.begin(), T->ent_ptr.end() - 1);
  for (int64_t e = 0; e < E; ++e)
    for (int s = 0; s < kSlots; ++s) {
      const int32_t x = elem_ent[e * kSlots + s];
      T->ent_copy[fill[x]++] = (e << 8) | ((int64_t)s << 3) | elem_orient[e * kSlots + s];
    }
  for (int64_t x = 0; x < T->nF; ++x)
    if (T->ent_ptr[x + 1] - T->ent_ptr[x] > 2)
      return "non-conforming topology: a face is shared by more than two elements "
             "(a periodic direction needs >= 3 elements)";
  // masks: a Dirichlet face masks its face, its 4 edges and its 4 vertices
  T->ent_flags.assign(nEnt, 0);
  if (bc) {
    for (int64_t e = 0; e < E; ++e)
      for (int f = 0; f < 6; ++f) {
        if (bc[e * 6 + f] != 1) continue;
        T->ent_flags[elem_ent[e * kSlots + f]] |= kEntMasked;
        int cs[4] = {face_corner(f, 0, 0), face_corner(f, 1, 0), face_corner(f, 0, 1),
                     face_corner(f, 1, 1)};
        for (int c = 0; c < 4; ++c) T->ent_flags[elem_ent[e * kSlots + kVertSlot0 + cs[c]]] |= kEntMasked;
        for (int ed = 0; ed < 12; ++ed) {
          int s0, s1;
          edge_corners(ed, &s0, &s1);
          bool in0 = false, in1 = false;
          for (int c = 0; c < 4; ++c) { in0 |= (cs[c] == s0); in1 |= (cs[c] == s1); }
          if (in0 && in1) T->ent_flags[elem_ent[e * kSlots + kEdgeSlot0 + ed]] |= kEntMasked;
        }
      }
  }
  T->ent_key.resize((size_t)nEnt * 4);
  for (int64_t x = 0; x < T->nF; ++x)
    for (int q = 0; q < 4; ++q) T->ent_key[x * 4 + q] = fkeys[x][q];
  for (int64_t x = 0; x < T->nEd; ++x)
    for (int q = 0; q < 4; ++q) T->ent_key[(T->nF + x) * 4 + q] = ekeys[x][q];
  for (int64_t x = 0; x < T->nV; ++x)
    for (int q = 0; q < 4; ++q) T->ent_key[(T->nF + T->nEd + x) * 4 + q] = vkeys[x][q];
  T->elem_ent.swap(elem_ent);
  return "";
}

}  // namespace sem

// ---------------------------------------------------------------------------
// Interface planning for a partitioned mesh (host only; "these
// parts of the domain are then distributed among the MPI ranks"
// "only unit-depth communication is necessary").
// ---------------------------------------------------------------------------
namespace sem {

void iface_candidates(const Topology& T, std::vector<int64_t>* keys, std::vector<int32_t>* ents) {
  // an entity can be shared with another rank only if it lies on a face that
  // has a single local copy (the rank's boundary, physical walls included)
  std::vector<uint8_t> cand(T.nEnt(), 0);
  for (int64_t f = 0; f < T.nF; ++f) {
    if (T.ent_ptr[f + 1] - T.ent_ptr[f] != 1) continue;
    cand[f] = 1;
    const int64_t cp = T.ent_copy[T.ent_ptr[f]];
    const int64_t e = cp >> 8;
    const int slot = (int)((cp >> 3) & 31);
    int cs[4] = {face_corner(slot, 0, 0), face_corner(slot, 1, 0), face_corner(slot, 0, 1), face_corner(slot, 1, 1)};
    for (int c = 0; c < 4; ++c) cand[T.elem_ent[e * kSlots + kVertSlot0 + cs[c]]] = 1;
    for (int ed = 0; ed < 12; ++ed) {
      int s0, s1;
      edge_corners(ed, &s0, &s1);
      bool in0 = false, in1 = false;
      for (int c = 0; c < 4; ++c) { in0 |= (cs[c] == s0); in1 |= (cs[c] == s1); }
      if (in0 && in1) cand[T.elem_ent[e * kSlots + kEdgeSlot0 + ed]] = 1;
    }
  }
  keys->clear();
  ents->clear();
  for (int64_t x = 0; x < T.nEnt(); ++x)
    if (cand[x]) {
      ents->push_back((int32_t)x);
      for (int q = 0; q < 4; ++q) keys->push_back(T.ent_key[x * 4 + q]);
    }
}

std::string iface_plan(const Topology& T, int rank, int nranks, const std::vector<int64_t>& counts,
                       const std::vector<int64_t>& all_keys, IfacePlan* P) {
  P->rank = rank;
  P->nranks = nranks;
  P->ents.clear();
  P->ranks.clear();
  P->peers.clear();
  P->peer_list.clear();
  if ((int)counts.size() != nranks) return "iface_plan: counts size";
  std::unordered_map<std::array<int64_t, 4>, std::vector<int>, KeyHash> owners;
  int64_t off = 0;
  for (int r = 0; r < nranks; ++r) {
    for (int64_t q = 0; q < counts[r]; ++q, ++off) {
      std::array<int64_t, 4> k = {all_keys[off * 4], all_keys[off * 4 + 1], all_keys[off * 4 + 2],
                                  all_keys[off * 4 + 3]};
      auto& v = owners[k];
      if (v.empty() || v.back() != r) v.push_back(r);
    }
  }
  std::vector<int64_t> mykeys;
  std::vector<int32_t> myents;
  iface_candidates(T, &mykeys, &myents);
  struct Item { std::array<int64_t, 4> key; int32_t ent; const std::vector<int>* ranks; };
  std::vector<Item> items;
  for (size_t q = 0; q < myents.size(); ++q) {
    std::array<int64_t, 4> k = {mykeys[q * 4], mykeys[q * 4 + 1], mykeys[q * 4 + 2], mykeys[q * 4 + 3]};
    auto it = owners.find(k);
    if (it == owners.end()) return "iface_plan: own key missing from the gathered keys";
    if (it->second.size() >= 2) items.push_back({k, myents[q], &it->second});
  }
  std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.key < b.key; });
  std::vector<std::vector<int32_t>> per(nranks);
  for (size_t q = 0; q < items.size(); ++q) {
    P->ents.push_back(items[q].ent);
    P->ranks.push_back(*items[q].ranks);
    for (int r : *items[q].ranks)
      if (r != rank) per[r].push_back((int32_t)q);
  }
  for (int r = 0; r < nranks; ++r)
    if (!per[r].empty()) {
      P->peers.push_back(r);
      P->peer_list.push_back(per[r]);
    }
  return "";
}

}  // namespace sem
