// Element-major gather-scatter (readings R7, R8; DESIGN.md §4 "Gather-scatter,
// element gather").  PAPER.md:71: the only coupling of the element-by-element
// operator is the unit-depth gather-scatter over shared element nodes.
//
// The nodal pass (k_gs_nodal) walks the shared-node groups and scatters 8-byte
// loads/stores over w in place: every 32-byte sector of w is touched (the
// r-faces, i = 0 and i = N, sit in every row) and the pass is latency bound.
// Here each WARP owns a sequence of elements.  An element's unassembled
// operator output t (and in the CG its r and dinv) arrives in the warp's
// shared-memory stage by bulk copy (TMA engine, one mbarrier per stage) while
// the warp works on the previous element, so the bytes in flight do not
// depend on registers.  The warp then assembles the element's boundary nodes
// entity by entity -- faces, edges, vertices, lane-parallel -- summing every
// copy in the entity's copy-list order (ascending element: the oracle's and
// k_gs_nodal's order, so the sums are bit-identical), its own copy from the
// stage and the neighbours' from t in global memory (L2: the warps work on a
// sliding window of elements, so a neighbour's lines are read from HBM once),
// 0 where masked, and writes the sums into the stage.  Nothing is written to
// t, so no element waits for another.
//
//   MODE 0  w = mask . dssum(t)                       (sem_ax_dssum, out of place)
//   MODE 1  r -= alpha mask . dssum(t), rtr, rtz      (the CG update, R10; the
//           assembled A p is never stored)
//
// The per-element descriptor (gsplan.cpp, build_elem_desc) is one 64-bit word
// per (element, entity slot): copy-list pointer | m << 32 | action << 40 |
// own orientation << 48 | global multiplicity << 56 (action 0: own value -- a
// single unmasked copy, or an interface entity whose rank-summed total the
// exchange already wrote into every copy; 1: masked; 2: sum of the copies).
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "device_common.cuh"
#include "p2p.cuh"

namespace sem {

namespace {
constexpr int kGeMaxC = 8;  // copies staged per entity (more: read from the global list)

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int LX, int MODE>
struct GeCfg {
  static constexpr int N3 = LX * LX * LX;
  static constexpr int N3P = (N3 + 1) & ~1;
  static constexpr int M = LX - 2;
  static constexpr int MD = M > 0 ? M : 1;  // divisor (lx = 2: no face or edge interiors)
  static constexpr int NARR = MODE == 1 ? 3 : 1;  // t (, r, dinv)
  static constexpr bool BULK = (N3 % 2) == 0;     // element blocks 16-byte aligned -> bulk copies
  // per warp and stage: data, descriptors, 1/multiplicities, partner maps;
  // then the two mbarriers
  static constexpr int STAGE_BYTES = NARR * N3P * 8 + kSlots * 16 + kSlots * kGeMaxC * 8;
  static constexpr int WARP_BYTES = 2 * STAGE_BYTES + 16;
  // warps per CTA: four, fewer when two CTAs of them would not fit an SM
  static constexpr int WPC_RAW = 115000 / WARP_BYTES;
  static constexpr int WPC = WPC_RAW < 1 ? 1 : (WPC_RAW > 4 ? 4 : WPC_RAW);
  static constexpr int SMEM = WPC * WARP_BYTES;
  static constexpr int FACE_IT = (6 * M * M + 31) / 32;
  static constexpr int EDGE_IT = (12 * M + 31) / 32;
  static constexpr int FACE_A = FACE_IT > 0 ? FACE_IT : 1, EDGE_A = EDGE_IT > 0 ? EDGE_IT : 1;
};

// local offset of face-interior node (a, b) of face slot f (the face's own
// (u, v) axes: x-faces (j, k), y-faces (i, k), z-faces (i, j))
template <int LX>
__device__ __forceinline__ int face_node(int f, int a, int b, int& i, int& j, int& k) {
  const int side = (f & 1) ? LX - 1 : 0, ax = f >> 1;
  i = ax == 0 ? side : 1 + a;
  j = ax == 0 ? 1 + a : (ax == 1 ? side : 1 + b);
  k = ax == 2 ? side : 1 + b;
  return i + LX * (j + LX * k);
}
template <int LX>
__device__ __forceinline__ int edge_node(int ed, int t, int& i, int& j, int& k) {
  constexpr int N = LX - 1;
  const int ax = ed >> 2, q = ed & 3;
  const int p = (q & 1) * N, r = (q >> 1) * N;
  i = ax == 0 ? 1 + t : p;
  j = ax == 0 ? p : (ax == 1 ? 1 + t : r);
  k = ax == 2 ? 1 + t : r;
  return i + LX * (j + LX * k);
}
// the entity slot of local node (i, j, k) (-1: element interior)
template <int LX>
__device__ __forceinline__ int node_slot(int i, int j, int k) {
  constexpr int N = LX - 1;
  const int bi = (i == 0 || i == N), bj = (j == 0 || j == N), bk = (k == 0 || k == N);
  const int nb = bi + bj + bk;
  if (nb == 0) return -1;
  if (nb == 1) return bi ? (i == N) : (bj ? 2 + (j == N) : 4 + (k == N));
  if (nb == 2) {
    const int ax = !bi ? 0 : (!bj ? 1 : 2);
    const int p = ax == 0 ? j : i, r = ax == 2 ? j : k;
    return kEdgeSlot0 + ax * 4 + (p != 0) + 2 * (r != 0);
  }
  return kVertSlot0 + (i != 0) + 2 * (j != 0) + 4 * (k != 0);
}
// canonical index within entity `slot` of local node (i, j, k) of a copy with
// orientation o (the inverse of node_offset<LX>)
template <int LX>
__device__ __forceinline__ int node_canonical(int slot, int o, int i, int j, int k) {
  constexpr int M = LX - 2;
  if (slot < kEdgeSlot0) {
    const int ax = slot >> 1;
    const int u = ax == 0 ? j : i, v = ax == 2 ? j : k;
    const int du = (o & 1) ? M - u : u - 1, dv = (o & 2) ? M - v : v - 1;
    const int a = (o & 4) ? dv : du, b = (o & 4) ? du : dv;
    return a + M * b;
  }
  if (slot < kVertSlot0) {
    const int ax = (slot - kEdgeSlot0) >> 2;
    const int t = ax == 0 ? i : (ax == 1 ? j : k);
    return (o & 1) ? M - t : t - 1;
  }
  return 0;
}
}  // namespace

struct GeArgs {
  const double* t;            // unassembled element output [E][n3]
  double* w;                  // MODE 0: assembled output
  const uint64_t* desc;       // [E][26]
  const int64_t* copy;        // entity copy lists (e << 8 | slot << 3 | orient)
  const int32_t* qtab;        // partner maps (gsplan.cpp build_qtab)
  int64_t E;
  const int* skip;            // MODE 0: device flag, set -> the launch does nothing (GMRES cycle end)
  // MODE 1 (CG update)
  double* r;
  const double* dinv;
  double* part;
  unsigned* ticket;
  CGScalars* sc;
  int fuse_scalar;
  P2PArgs p2p;
  cudaGraphConditionalHandle loop;
};

// Partner maps (gsplan.cpp build_qtab): the copy (ps, po) of the entity whose
// own copy is (s, o) holds the own node with loop coordinates (a, b) at local
// offset o00 + a qa + b qb (orientation maps are affine).
__device__ __forceinline__ int qtab_index(int s, int o, int ps, int po) {
  if (s < kEdgeSlot0) return ((s * 8 + o) * 6 + ps) * 8 + po;
  if (s < kVertSlot0) return 2304 + (((s - kEdgeSlot0) * 2 + (o & 1)) * 12 + (ps - kEdgeSlot0)) * 2 + (po & 1);
  return 2304 + 576 + (s - kVertSlot0) * 8 + (ps - kVertSlot0);
}

// The assembled value of the own node (a, b) of an entity: its copies in list
// order (every copy, the own one included, read from t: the stage still
// equals t here), 0 where masked.  Q: the staged maps {offset of (0, 0) in
// t, qa | qb << 16}, padded to MAXC with copies of the first.  Split in two
// so that a lane issues the loads of all its nodes before the first sum.
template <int MAXC>
__device__ __forceinline__ void gather_load(const double* __restrict__ t, int a, int b, int mc, const int2* Q,
                                            double (&v)[MAXC]) {
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int2 qq = Q[c];
    const int qa = (int)(short)(qq.y & 0xffff), qb = qq.y >> 16;
    v[c] = c < mc ? __ldg(t + (qq.x + a * qa + b * qb)) : 0.0;
  }
}
template <int MAXC>
__device__ __forceinline__ double gather_sum(const double (&v)[MAXC], int mc, bool masked) {
  double sum = v[0];
#pragma unroll
  for (int c = 1; c < MAXC; ++c)
    if (c < mc) sum += v[c];
  return masked ? 0.0 : sum;
}

template <int LX, int MODE>
__global__ void __launch_bounds__(32 * GeCfg<LX, MODE>::WPC) k_gs_elem(const GeArgs A) {
  using C = GeCfg<LX, MODE>;
  constexpr int N3 = C::N3, N3P = C::N3P, M = C::M, MD = C::MD;
  constexpr int NF = 6 * M * M, NE = 12 * M;
  extern __shared__ __align__(128) unsigned char ge_smem[];
  __shared__ double s_red[64];
  __shared__ int s_flag;
  // per-CTA node tables: face / edge loop index -> local offset | a << 16 |
  // b << 24 | slot << 8 ... (see below), node -> slot (-1 interior)
  __shared__ uint32_t s_fnode[NF > 0 ? NF : 1];
  __shared__ uint32_t s_enode[NE > 0 ? NE : 1];
  __shared__ int8_t s_slot[N3];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int x = threadIdx.x; x < NF; x += blockDim.x) {
    const int f = x / (MD * MD), ab = x - f * MD * MD, a = ab % MD, b = ab / MD;
    int i, j, k;
    s_fnode[x] = (uint32_t)face_node<LX>(f, a, b, i, j, k) | ((uint32_t)a << 12) | ((uint32_t)b << 18) |
                 ((uint32_t)f << 24);
  }
  for (int x = threadIdx.x; x < NE; x += blockDim.x) {
    const int ed = x / MD, tt = x - ed * MD;
    int i, j, k;
    s_enode[x] = (uint32_t)edge_node<LX>(ed, tt, i, j, k) | ((uint32_t)tt << 12) | ((uint32_t)(kEdgeSlot0 + ed) << 24);
  }
  for (int q = threadIdx.x; q < N3; q += blockDim.x) s_slot[q] = (int8_t)node_slot<LX>(q % LX, (q / LX) % LX, q / (LX * LX));
  __syncthreads();
  unsigned char* wbase = ge_smem + (size_t)wib * C::WARP_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase + 2 * C::STAGE_BYTES);
  auto stage_data = [&](int st) { return reinterpret_cast<double*>(wbase + (size_t)st * C::STAGE_BYTES); };
  auto stage_desc = [&](int st) {
    return reinterpret_cast<uint64_t*>(wbase + (size_t)st * C::STAGE_BYTES + C::NARR * N3P * 8);
  };
  auto stage_w = [&](int st) {
    return reinterpret_cast<double*>(wbase + (size_t)st * C::STAGE_BYTES + C::NARR * N3P * 8 + kSlots * 8);
  };
  auto stage_q = [&](int st) {
    return reinterpret_cast<int2*>(wbase + (size_t)st * C::STAGE_BYTES + C::NARR * N3P * 8 + kSlots * 16);
  };
  double alpha = 0.0;
  if (MODE == 0 && A.skip && *A.skip) return;
  if (MODE == 1) {
    // the same early exits as k_cg_update (loop != 0: body of a WHILE node)
    if (A.sc->done) {
      if (A.loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(A.loop, 0);
      return;
    }
    const double pAp = A.sc->red[0];
    if (!(pAp > 0.0)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.sc->breakdown = 1;
        A.sc->done = 1;
        A.sc->pAp = pAp;
        if (A.loop) cudaGraphSetConditional(A.loop, 0);
      }
      return;
    }
    alpha = A.sc->rtz / pAp;
  }
  const int64_t nw = (int64_t)gridDim.x * C::WPC;
  int64_t e = (int64_t)blockIdx.x * C::WPC + wib;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncwarp();
  // element data of e into stage st (bulk copies issued by lane 0; the odd-n3
  // fallback: plain loads by the warp, completed by a lane-0 arrival)
  auto issue_data = [&](int64_t ee, int st) {
    double* D = stage_data(st);
    const size_t eo = (size_t)ee * N3;
    if constexpr (C::BULK) {
      if (lane == 0) {
        fence_proxy_async_smem();  // the stage was last read/written by the generic proxy
        const uint64_t pol = policy_evict_first();
        mbar_expect_tx(&bar[st], C::NARR * N3 * 8);
        bulk_g2s(D, A.t + eo, N3 * 8, &bar[st], policy_evict_last());
        if (MODE == 1) {
          bulk_g2s(D + N3P, A.r + eo, N3 * 8, &bar[st], pol);
          bulk_g2s(D + 2 * N3P, A.dinv + eo, N3 * 8, &bar[st], pol);
        }
      }
    } else {
      for (int q = lane; q < N3; q += 32) {
        D[q] = __ldg(A.t + eo + q);
        if (MODE == 1) {
          D[N3P + q] = A.r[eo + q];
          D[2 * N3P + q] = __ldg(A.dinv + eo + q);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[st]);
    }
  };
  // the staging lanes (lane = slot < 26): descriptor, 1/multiplicity and the
  // partner maps of element ee (copies cp, list order) into stage st; an
  // entity taking its own value (one copy, or an interface entity the
  // exchange finished) gets the own copy alone
  const int2* __restrict__ qtab = reinterpret_cast<const int2*>(A.qtab);
  auto stage_meta = [&](int st, int64_t ee, uint64_t d, const int64_t* cp) {
    const int act = (int)((d >> 40) & 0xff), o = (int)((d >> 48) & 7);
    const int mc = act == 2 ? (int)((d >> 32) & 0xff) : 1;
    stage_desc(st)[lane] = (d & ~(0xffull << 32)) | ((uint64_t)mc << 32);
    stage_w(st)[lane] = 1.0 / (double)(int)(d >> 56);  // the oracle's mult = 1/m
    int2* Q = stage_q(st) + lane * kGeMaxC;
    int2 first = make_int2(0, 0);
#pragma unroll
    for (int c = 0; c < kGeMaxC; ++c) {
      int2 q = first;
      if (c < mc) {
        const int64_t cpc = act == 2 ? cp[c] : (((int64_t)ee << 8) | (lane << 3) | o);
        const int2 tq = __ldg(qtab + qtab_index(lane, o, (int)((cpc >> 3) & 31), (int)(cpc & 7)));
        q = make_int2((int)((cpc >> 8) * N3) + tq.x, tq.y);
      }
      if (c == 0) first = q;
      Q[c] = q;
    }
  };
  // descriptors two elements ahead, copy lists one ahead (registers), staged
  // after the current element is done
  uint64_t dnext = 0;  // descriptor of the element after e (lane < 26)
  int64_t cpr[kGeMaxC];
  if (e < A.E) {
    issue_data(e, 0);
    if (lane < kSlots) {
      const uint64_t d0 = __ldg(A.desc + e * kSlots + lane);
      const int mc = (int)((d0 >> 32) & 0xff);
#pragma unroll
      for (int c = 0; c < kGeMaxC; ++c) cpr[c] = c < mc ? __ldg(A.copy + (uint32_t)d0 + c) : 0;
      stage_meta(0, e, d0, cpr);
      if (e + nw < A.E) dnext = __ldg(A.desc + (e + nw) * kSlots + lane);
    }
  }
  double acc[2] = {0.0, 0.0};
  uint32_t phase[2] = {0u, 0u};
  int st = 0;
  for (; e < A.E; e += nw, st ^= 1) {
    const int64_t en = e + nw;
    const bool has_next = en < A.E;
    if (has_next) issue_data(en, st ^ 1);
    // copy lists of the next element, descriptor of the one after
    uint64_t dn2 = 0;
    if (has_next && lane < kSlots) {
      const int mc = (int)((dnext >> 32) & 0xff);
#pragma unroll
      for (int c = 0; c < kGeMaxC; ++c) cpr[c] = c < mc ? __ldg(A.copy + (uint32_t)dnext + c) : 0;
      if (en + nw < A.E) dn2 = __ldg(A.desc + (en + nw) * kSlots + lane);
    }
    __syncwarp();
    const uint64_t* SD = stage_desc(st);
    const int2* SQ = stage_q(st);
    // faces (at most two copies: topo.cpp rejects more), edges, vertices:
    // every load of the lane first (from t in global memory; the stage is not
    // needed yet), then the sums in list order
    double fv[C::FACE_A][2];
    int fq[C::FACE_A], fm[C::FACE_A];
#pragma unroll
    for (int it = 0; it < C::FACE_IT; ++it) {
      const int idx = lane + 32 * it;
      fq[it] = -1;
      fm[it] = 0;
      fv[it][0] = fv[it][1] = 0.0;
      if (idx < NF) {
        const uint32_t fn = s_fnode[idx];
        const int f = (int)(fn >> 24);
        const uint64_t d = SD[f];
        fq[it] = (int)(fn & 0xfff);
        fm[it] = ((d >> 40) & 0xff) == 1 ? -1 : (int)((d >> 32) & 0xff);  // -1: masked
        gather_load<2>(A.t, (int)((fn >> 12) & 63), (int)((fn >> 18) & 63), fm[it] < 0 ? 0 : fm[it],
                       SQ + f * kGeMaxC, fv[it]);
      }
    }
    double evv[C::EDGE_A][4];
    int eq[C::EDGE_A], emc[C::EDGE_A], es[C::EDGE_A];
#pragma unroll
    for (int it = 0; it < C::EDGE_IT; ++it) {
      const int idx = lane + 32 * it;
      eq[it] = -1;
      emc[it] = 0;
      es[it] = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) evv[it][c] = 0.0;
      if (idx < NE) {
        const uint32_t en_ = s_enode[idx];
        const int s = (int)(en_ >> 24);
        const uint64_t d = SD[s];
        eq[it] = (int)(en_ & 0xfff);
        es[it] = s | (((int)(en_ >> 12) & 63) << 8);
        emc[it] = ((d >> 40) & 0xff) == 1 ? -1 : (int)((d >> 32) & 0xff);
        gather_load<4>(A.t, (int)((en_ >> 12) & 63), 0, emc[it] < 0 ? 0 : emc[it], SQ + s * kGeMaxC, evv[it]);
      }
    }
    double vvv[kGeMaxC];
    int vq = -1, vmc = 0;
#pragma unroll
    for (int c = 0; c < kGeMaxC; ++c) vvv[c] = 0.0;
    if (lane < 8) {
      const int s = kVertSlot0 + lane;
      const uint64_t d = SD[s];
      vq = (lane & 1) * (LX - 1) + LX * (((lane >> 1) & 1) * (LX - 1) + LX * ((lane >> 2) * (LX - 1)));
      vmc = ((d >> 40) & 0xff) == 1 ? -1 : (int)((d >> 32) & 0xff);
      gather_load<kGeMaxC>(A.t, 0, 0, vmc < 0 ? 0 : vmc, SQ + s * kGeMaxC, vvv);
    }
    double fsum[C::FACE_A], esum[C::EDGE_A], vsum = 0.0;
#pragma unroll
    for (int it = 0; it < C::FACE_IT; ++it) fsum[it] = gather_sum<2>(fv[it], fm[it], fm[it] < 0);
#pragma unroll
    for (int it = 0; it < C::EDGE_IT; ++it) {
      esum[it] = gather_sum<4>(evv[it], emc[it], emc[it] < 0);
      if (emc[it] > 4) {  // an edge of more than four elements (unstructured meshes)
        const int s = es[it] & 0xff;
        double v8[kGeMaxC];
        gather_load<kGeMaxC>(A.t, es[it] >> 8, 0, emc[it], SQ + s * kGeMaxC, v8);
        esum[it] = gather_sum<kGeMaxC>(v8, emc[it], false);
      }
    }
    if (lane < 8) vsum = gather_sum<kGeMaxC>(vvv, vmc, vmc < 0);
    mbar_wait(&bar[st], phase[st]);
    phase[st] ^= 1u;
    double* T = stage_data(st);
#pragma unroll
    for (int it = 0; it < C::FACE_IT; ++it)
      if (fq[it] >= 0) T[fq[it]] = fsum[it];
#pragma unroll
    for (int it = 0; it < C::EDGE_IT; ++it)
      if (eq[it] >= 0) T[eq[it]] = esum[it];
    if (vq >= 0) T[vq] = vsum;
    __syncwarp();
    const size_t eo = (size_t)e * N3;
    if (MODE == 0) {
      for (int q = lane; q < N3; q += 32) A.w[eo + q] = T[q];
    } else {
      const double* R = T + N3P;
      const double* Dv = T + 2 * N3P;
      const double* SW = stage_w(st);
      for (int q = lane; q < N3; q += 32) {
        const int s = s_slot[q];
        const double mw = s < 0 ? 1.0 : SW[s];
        const double rq = R[q] - alpha * T[q];
        A.r[eo + q] = rq;
        acc[0] += mw * rq * rq;
        acc[1] += mw * rq * (Dv[q] * rq);
      }
    }
    __syncwarp();  // the stage's generic-proxy accesses are done before it is refilled
    if (has_next && lane < kSlots) stage_meta(st ^ 1, en, dnext, cpr);
    dnext = dn2;
    __syncwarp();
  }
  if (MODE == 1) {
    grid_sum_last_block<2>(acc, A.part, A.ticket, &A.sc->red[1], s_red, &s_flag);
    // the last block takes the scalar step (after the NVLink allreduce of
    // rtr, rtz when there are several ranks), as k_cg_update does
    if (A.fuse_scalar && s_flag) {
      if (A.p2p.peers) {
        __syncthreads();
        if (threadIdx.x < 32) p2p_allreduce_warp(&A.sc->red[1], 2, A.p2p, threadIdx.x);
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        cg_scalar_step(A.sc);
        if (A.loop) cudaGraphSetConditional(A.loop, A.sc->done ? 0 : 1);
      }
    }
  }
}

P2PArgs p2p_args(const sem_mesh* m);  // p2p.cu

constexpr int kGeMaxDevices = 64;

template <int LX, int MODE>
static cudaError_t launch_ge(const sem_mesh* m, const GeArgs& A, cudaStream_t s) {
  using C = GeCfg<LX, MODE>;
  auto kern = k_gs_elem<LX, MODE>;
  // per device: the dynamic shared memory attribute and the resident CTAs
  static std::atomic<int> ctas[kGeMaxDevices];
  const int dev = m->device;
  if (dev < 0 || dev >= kGeMaxDevices) return cudaErrorInvalidDevice;
  int per_sm = ctas[dev].load(std::memory_order_acquire);
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * C::WPC, C::SMEM);
    if (e != cudaSuccess) return e;
    per_sm = std::max(1, per_sm);
    ctas[dev].store(per_sm, std::memory_order_release);
  }
  const int64_t need = (A.E + C::WPC - 1) / C::WPC;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)m->nsm * per_sm));
  kern<<<grid, 32 * C::WPC, C::SMEM, s>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_gs_elem_dssum(const sem_mesh* m, const double* t, double* w, const int* skip, cudaStream_t s) {
  if (m->E == 0) return cudaSuccess;
  GeArgs A{};
  A.t = t;
  A.w = w;
  A.desc = m->d_gs_desc;
  A.copy = m->d_ent_copy;
  A.qtab = m->d_gs_qtab;
  A.E = m->E;
  A.skip = skip;
  SEM_COUNT_LAUNCH(m);
  cudaError_t e = cudaErrorInvalidValue;
  SEM_LX_DISPATCH_INT(m->lx, e, (launch_ge<LX, 0>(m, A, s)));
  return e;
}

cudaError_t launch_gs_elem_cg_update(sem_mesh* m, const double* t, cudaStream_t s, bool fuse_scalar,
                                     cudaGraphConditionalHandle loop) {
  GeArgs A{};
  A.t = t;
  A.desc = m->d_gs_desc;
  A.copy = m->d_ent_copy;
  A.qtab = m->d_gs_qtab;
  A.E = m->E;
  A.r = m->r;
  A.dinv = m->dinv;
  A.part = m->part;
  A.ticket = m->ticket;
  A.sc = m->sc;
  A.fuse_scalar = fuse_scalar ? 1 : 0;
  A.p2p = p2p_args(m);
  A.loop = loop;
  SEM_COUNT_LAUNCH(m);
  cudaError_t e = cudaErrorInvalidValue;
  SEM_LX_DISPATCH_INT(m->lx, e, (launch_ge<LX, 1>(m, A, s)));
  return e;
}

}  // namespace sem
