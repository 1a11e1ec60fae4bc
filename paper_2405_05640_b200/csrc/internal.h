// Internal declarations of libsem_b200 (not part of the ABI; see include/sem.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sem.h"

#ifdef SEM_WITH_NCCL
#include <nccl.h>
#endif
#include <nvtx3/nvToolsExt.h>

namespace sem {

constexpr int kMaxN = 11;           // lx <= 12
constexpr int kSlots = 26;          // 6 faces + 12 edges + 8 vertices per element
constexpr int kFaceSlot0 = 0, kEdgeSlot0 = 6, kVertSlot0 = 18;

// ---- error plumbing -------------------------------------------------------
void set_error(const std::string& msg);
sem_status fail(sem_status st, const std::string& msg);
#define SEM_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::sem::fail(SEM_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define SEM_TRY_ST(expr)               \
  do {                                 \
    sem_status _st = (expr);           \
    if (_st != SEM_OK) return _st;     \
  } while (0)

// NVTX range over an entry point (visible in Nsight Systems / ncu --nvtx;
// header-only NVTX v3, a no-op without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define SEM_NVTX(name) ::sem::NvtxRange _sem_nvtx_range(name)

// ---- basis (host) ----------------------------------------------------------
// GLL nodes/weights by Golub-Welsch, D by barycentric weights (basis.cpp).
bool gll_golub_welsch(int N, double* xi, double* w);
void deriv_matrix(int N, const double* xi, double* D);  // D[i*lx+l] = l_l'(xi_i)

// ---- topology / gather-scatter plan (host, topo.cpp) ----------------------
// Every shared node belongs to exactly one "entity": a vertex, the interior
// of an edge, or the interior of a face.  An entity has a canonical node
// order defined by GLOBAL vertex ids only, so all copies (in any element, on
// any rank) agree on it.  A copy is encoded as (e << 8) | (slot << 3) | orient.
struct Topology {
  int64_t E = 0;
  int N = 0, lx = 0, m = 0;               // m = lx - 2 interior nodes per edge
  int64_t nF = 0, nEd = 0, nV = 0;        // entity counts; ids: faces, edges, vertices
  std::vector<int32_t> elem_ent;          // [E][26]
  std::vector<int32_t> ent_ptr;           // CSR over copies, size nEnt+1
  std::vector<int64_t> ent_copy;          // copies, ascending element within an entity
  std::vector<uint8_t> ent_flags;         // bit0: masked (Dirichlet), bit1: interface
  // entity keys (sorted global vertex ids; unused slots = -1), for cross-rank matching
  std::vector<int64_t> ent_key;           // [nEnt][4]
  int64_t nEnt() const { return nF + nEd + nV; }
  int ent_nodes(int64_t ent) const {
    return ent < nF ? m * m : (ent < nF + nEd ? m : 1);
  }
};
enum : uint8_t { kEntMasked = 1, kEntInterface = 2 };
// Returns empty string on success, else an error message.
std::string build_topology(int64_t E, int N, const int64_t* conn, const int8_t* bc,
                           Topology* T);
// Local node offset (0..n3-1) of canonical node n of a copy (slot, orient).
int copy_node_offset(int lx, int slot, int orient, int n);

// Interface between ranks (topo.cpp): candidates = entities lying on a face
// with a single local copy (keys: 4 sorted vertex ids, -1 padded); the plan
// lists the local entities also present on another rank, sorted by key
// (the canonical order every rank agrees on), their sharing ranks, and per
// peer the positions (into ents) of the entities shared with it.
struct IfacePlan {
  int rank = 0, nranks = 1;
  std::vector<int32_t> ents;
  std::vector<std::vector<int>> ranks;          // ascending, includes rank
  std::vector<int> peers;                       // ascending
  std::vector<std::vector<int32_t>> peer_list;  // per peer: indices into ents
};
void iface_candidates(const Topology& T, std::vector<int64_t>* keys, std::vector<int32_t>* ents);
std::string iface_plan(const Topology& T, int rank, int nranks, const std::vector<int64_t>& counts,
                       const std::vector<int64_t>& all_keys, IfacePlan* P);

// ---- device-side plan handed to kernels ------------------------------------
struct GsPlan {
  const int32_t* elem_ent;   // [E][26]
  const int32_t* ent_ptr;    // [nEnt+1]
  const int64_t* ent_copy;   // [ncopy]
  const uint8_t* ent_flags;  // [nEnt]
  int64_t nF, nEd, nV;
};

// Nodal gather-scatter plan (standalone gs pass, k_gs_nodal): every shared
// node needing a sum or a mask is a group of m local copies, listed per
// class (m, masked) as uint32 offsets into the local vector: copy k
// (ascending element order) of group g is idx[base + k*count + g] (struct of
// arrays), except for m = 2 classes: idx[base + 2g + k] (pairs, base even).
struct GsClass {
  int64_t base = 0, count = 0;
  int m = 0, masked = 0;
};
constexpr int kGsMaxCls = 16;  // classes per launch (more -> several launches)
struct GsLaunchCls {
  int64_t base;
  int32_t count, item0;
  int32_t m, masked;
};
struct GsLaunch {
  int ncls, nitems, n2;  // n2: items of the leading m <= 2 classes
  int pdl;               // launched as a programmatic dependent (griddepcontrol.wait first)
  int scale;             // mode & 4: every sum times 1/m (the multigrid smoother's average)
  GsLaunchCls c[kGsMaxCls];
};

// CG scalars living in device memory.
struct CGScalars {
  double rtz, rtz_prev, pAp, rtr, bn, tol, alpha, beta;
  double xalpha;        // alpha of the last p not yet added to x (deferred x update)
  double red[4];        // reduction outputs (local sums; allreduced in place)
  int iter, maxit, done, converged, breakdown, singular;
};

struct Comm;  // comm.cpp
struct GmState;  // gmres.h
struct HsmgState;  // hsmg.h

}  // namespace sem

struct sem_comm {
#ifdef SEM_WITH_NCCL
  ncclComm_t nccl = nullptr;
#endif
  int rank = 0, nranks = 1, device = 0;
  // CG scalar allreduce over NVLink peer memory (p2p.cu); NCCL if !p2p
  bool p2p = false;
  void* p2p_local = nullptr;              // own mailbox
  uint8_t** d_p2p_peers = nullptr;        // [nranks] mailbox bases, device array
  unsigned long long* p2p_seq = nullptr;  // call counter (device)
  std::vector<void*> p2p_opened;          // IPC mappings to close
  // sticky device-side failure word of the peer-memory paths: a spin that
  // timed out (lost or desynchronised peer) ORs a bit in; checked by the
  // host after every collective call that synchronises; once set the
  // communicator is broken (every later collective returns SEM_ENCCL)
  unsigned* d_err = nullptr;
  bool broken = false;
  bool want_p2p = true;                   // sem_comm_create_ex option
};

struct sem_mesh {
  int64_t E = 0;
  int N = 0, lx = 0, n3 = 0, n3p = 0;
  int64_t nloc = 0;
  int device = 0;
  sem_comm* comm = nullptr;
  sem::Topology topo;
  int64_t n_unique = 0, n_masked = 0, n_interface = 0;
  int64_t n_masked_glob = 0;  // over all ranks
  bool has_geom = false;
  bool affine = false;        // every element affine and the affine option on: operator reads d_gaff, not G
  double* d_gaff = nullptr;   // [E][6] per-element metric constants (affine variant)
  sem_options_t opt{};        // sem_mesh_set_options
  int nsm = 148;              // SMs of the mesh's device (cudaDevAttrMultiProcessorCount)
  // device arrays
  double* coords = nullptr;   // [3][E][n3]
  double* G = nullptr;        // [E][6][n3p]
  double* B = nullptr;        // [E][n3]
  double* mult = nullptr;     // [E][n3] 1/m
  double* mask = nullptr;     // [E][n3] 0/1
  uint8_t* m8 = nullptr;      // [E][n3] multiplicity m as a byte (vector update pass)
  int32_t* d_elem_ent = nullptr;
  int32_t* d_ent_ptr = nullptr;
  int64_t* d_ent_copy = nullptr;
  uint8_t* d_ent_flags = nullptr;
  int32_t* d_elist_all = nullptr;  // element processing order (NULL = identity)
  // standalone gather-scatter (sem_gs_op, set-up passes): every non-interface entity
  uint32_t* d_gidx = nullptr;
  std::vector<sem::GsClass> gs_cls;
  // the same plan for the CG vectors in the x-planes-last element layout
  // (xlast_pos, device_common.cuh), used while xl_active (cg_solve_impl)
  uint32_t* d_gidx_xl = nullptr;
  std::vector<sem::GsClass> gs_cls_xl;
  bool xl_active = false;
  bool reuse_dinv = false;    // the next standard CG solve keeps m->dinv (sem_pnpn_step's velocity components)

  // launch segments of positions (one rank: one; several: boundary, interior)
  std::vector<int64_t> pos;        // processing position of every element
  std::vector<int64_t> seg;        // segment bounds [0, .., E]
  cudaStream_t aux_stream = nullptr;
  cudaStream_t cap_stream = nullptr;  // the CG graph is captured and replayed here
  cudaStream_t bnd_stream = nullptr;  // several ranks: boundary elements + exchange start (high priority)
  cudaEvent_t ev_bnd = nullptr;
  cudaEvent_t ev_input = nullptr;
  bool input_pending = false;  // sem_cg_solve_host: b still uploading on aux (ev_input)
  cudaEvent_t ev_start = nullptr, ev_cap = nullptr;
  // CG work
  double *r = nullptr, *p = nullptr, *w = nullptr, *dinv = nullptr, *xw = nullptr, *bw = nullptr;
  double* s_cg = nullptr;     // s = A p of the single-reduction CG
  double* part = nullptr;     // reduction partials
  int64_t npart = 0;
  unsigned int* ticket = nullptr;
  sem::CGScalars* sc = nullptr;     // device
  sem::CGScalars* sc_host = nullptr;  // pinned
  double* h_buf = nullptr;    // pinned host staging for e2e
  sem::GmState* gm = nullptr; // restarted GMRES work space (sem_gmres_solve)
  sem::HsmgState* hs = nullptr;  // multigrid levels (sem_hsmg_apply, GMRES with SEM_PC_HSMG)
  std::vector<int64_t> conn_h;   // host copies of the mesh description (level meshes)
  std::vector<int8_t> bc_h;
  // time step (sem_pnpn_step): metric terms, assembled mass, work vectors
  double* MJ = nullptr;       // [E][9][n3] W J dr_a/dx_m
  double* Bg = nullptr;       // [E][n3] dssum(B)
  double* pn_t = nullptr;     // [3][E][n3]
  double* pn_c = nullptr;     // [3][E][n3]
  double* pn_r = nullptr;     // [E][n3]
  // multi-GPU interface (comm.cpp)
  sem::IfacePlan iface;
  int64_t n_boundary = 0, n_if_nodes = 0;
  int32_t* d_if_ent = nullptr;       // [ni] local entity ids, sorted by key
  int32_t* d_if_node_ent = nullptr;  // [nn] interface entity of each node
  int64_t* d_if_noff = nullptr;      // [ni + 1] node offsets (own partials in U)
  int32_t* d_if_src_ptr = nullptr;   // [ni + 1] contributions per entity (by rank)
  int64_t* d_if_src = nullptr;       // offsets into U of each contribution
  int32_t* d_send_idx = nullptr;     // pack: own-partial node index per sent value
  double* d_U = nullptr;             // [own partials | received per peer (x2 parity) | P2P flags]
  // interface exchange over NVLink peer memory (p2p.cu); NCCL send/recv if !xp2p
  bool xp2p = false;
  double** d_x_dst = nullptr;               // [peer] remote receive slot for this rank
  int64_t* d_x_stride = nullptr;            // [peer] its parity stride
  unsigned long long** d_x_flag = nullptr;  // [peer] remote flag for this rank
  int32_t* d_x_prank = nullptr;             // [peer] rank
  int32_t* d_x_peer_of = nullptr;           // [send item] peer index
  int64_t* d_x_peer_off = nullptr;          // [peer + 1] send offsets
  unsigned long long* d_x_seq = nullptr;    // exchange counter (+ pack ticket)
  std::vector<void*> x_opened;
  double* d_sendbuf = nullptr;
  int32_t* d_ent_gcount = nullptr;   // global copies per entity (multiplicity)
  std::vector<int64_t> peer_cnt, peer_off;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
  // profiling
  int64_t nlaunch = 0;          // kernels launched by the library on this mesh
  int64_t pap_nparts = 0;       // pAp partials written by the last fused-operator launch
  bool prof = false;
  int64_t prof_launches = 0;
  double prof_ms = 0.0;
  std::vector<cudaEvent_t> prof_ev;
  sem::GsPlan plan() const {
    return sem::GsPlan{d_elem_ent, d_ent_ptr, d_ent_copy, d_ent_flags, topo.nF, topo.nEd, topo.nV};
  }
};

namespace sem {
// kernels.cu launchers (return cudaError_t of the launch)
cudaError_t upload_basis(int N, const double* D, const double* w);
cudaError_t launch_geom_bad(const sem_mesh* m, unsigned long long* bad, cudaStream_t s);
cudaError_t launch_affine_detect(const sem_mesh* m, double* C, int* nonaffine, cudaStream_t s);
struct AxArgs {
  const double* u; double* w;
  const double* h1; const double* h2; double h1c, h2c;
  // CG prologue (p <- dinv r + beta p) and pAp partials
  const double* r; const double* dinv; double* p; CGScalars* sc; double* part;
  double* x;  // CG: deferred x += xalpha p_old before p is replaced (nullptr: no x update)
  bool* pap_fused;  // CG: set when the pAp reduction was fused into the gs launch
  const int* skip;  // device flag: when set the operator launch does nothing (GMRES)
  bool pdl;         // launch as a programmatic dependent of the previous kernel (option pdl)
};
// operator over processing positions [elem0, elem0 + count) (cg: the CG-fused
// variant: deferred x update, p update, pAp partials)
cudaError_t launch_ax_range(const sem_mesh* m, const AxArgs& a, bool cg, int64_t elem0, int64_t count,
                            cudaStream_t s);
// standalone nodal gather-scatter over a class list (mode: 1 add, 2 mask, 3
// add then mask; | 4: the sums times 1/m, as z *= mult would); pap_fused != nullptr: the last launch also reduces the CG
// operator's pAp partials into sc->red[0] (allreduced) and sets *pap_fused
cudaError_t launch_gs_nodal(const sem_mesh* m, double* w, const uint32_t* idx, const std::vector<GsClass>& cls,
                            int mode, cudaStream_t s, bool* pap_fused = nullptr, bool pdl = false);
cudaError_t launch_diag(const sem_mesh* m, const double* h1, const double* h2, double h1c,
                        double h2c, double* d, cudaStream_t s);
cudaError_t launch_invert_diag(const sem_mesh* m, double* d, cudaStream_t s);
cudaError_t launch_mult_mask(const sem_mesh* m, cudaStream_t s);
cudaError_t launch_rhs_local(const sem_mesh* m, const double* f, double* b, cudaStream_t s);
// CG pieces
cudaError_t launch_cg_init(sem_mesh* m, const double* b, double* x, double tol, int maxit,
                           int singular, cudaStream_t s);
cudaError_t launch_wdot(sem_mesh* m, const double* a, const double* b, int slot, cudaStream_t s);
cudaError_t launch_sub_mean(sem_mesh* m, double* x, int slot, cudaStream_t s);
cudaError_t launch_cg_start(sem_mesh* m, cudaStream_t s);
cudaError_t launch_cg_config(sem_mesh* m, double tol, int maxit, int singular, cudaStream_t s);
cudaError_t launch_cg_pap_reduce(sem_mesh* m, cudaStream_t s);
// loop != 0: the update's last block (or block 0 on an early exit) sets the
// WHILE condition of the enclosing conditional graph node to !done
cudaError_t launch_cg_update(sem_mesh* m, cudaStream_t s, bool fuse_scalar, cudaGraphConditionalHandle loop = 0,
                             bool pdl = false);
// launch `kern` with the programmatic-stream-serialization attribute when pdl
// (the kernel then starts with griddepcontrol.wait)
template <class... KArgs, class... Args>
cudaError_t launch_maybe_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
  if (!pdl) {
    kern<<<grid, block, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
cudaError_t launch_cg_x_final(sem_mesh* m, double* x, cudaStream_t s);

cudaError_t launch_cg_scalar_step(sem_mesh* m, int phase, cudaStream_t s);
cudaError_t launch_count_nonzero(const double* a, int64_t n, sem_mesh* m, int slot, cudaStream_t s);
cudaError_t launch_ax_pcg(const sem_mesh* m, const AxArgs& a, double* x, const double* win, double* wout,
                          int first, int64_t elem0, int64_t count, cudaStream_t s);
cudaError_t launch_reduce3(sem_mesh* m, const double* in, cudaStream_t s);
cudaError_t launch_pcg_scalar(sem_mesh* m, int phase, cudaStream_t s);
// reduction scratch: [kMaxVecBlocks * 4 | per-position partials (3 per position)]
constexpr int64_t kMaxVecBlocks = 256 * 8;
int64_t part_capacity(int64_t E);
int64_t pap_part_offset();
// pnpn.cu: the time-step operators
cudaError_t upload_basis_pnpn(int N, const double* D, const double* w);
cudaError_t launch_metrics(const sem_mesh* m, double* MJ, cudaStream_t s);
cudaError_t launch_grad(const sem_mesh* m, const double* p, const double* MJ, double* g, cudaStream_t s);
cudaError_t launch_wdiv(const sem_mesh* m, const double* f, const double* MJ, double* dv, cudaStream_t s);
cudaError_t launch_convect(const sem_mesh* m, const double* u, const double* MJ, double* c, cudaStream_t s);
cudaError_t launch_pn_axpy(const sem_mesh* m, const double* a, double sa, const double* b, double sb, double* out,
                           int64_t n, cudaStream_t s);
cudaError_t launch_pn_mul(const sem_mesh* m, const double* a, const double* b, double* out, int64_t n,
                          cudaStream_t s);
cudaError_t launch_pn_div(const sem_mesh* m, double* a, const double* b, int64_t n, cudaStream_t s);
// comm.cpp: synchronise and check a communicator's sticky error word
sem_status comm_check(sem_comm* c);
// host: gather-scatter plans (gsplan.cpp)
sem_status build_gs_plans(sem_mesh* m, const std::vector<int64_t>& pos);
void gs_plans_free(sem_mesh* m);
}  // namespace sem
