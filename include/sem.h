/*
 * sem.h -- C ABI of the B200-native SEM hot path (libsem_b200.so).
 *
 * The operation (arXiv 2405.05640, PAPER.md "Neko", lines 71-74): spectral
 * elements -- "E non-overlapping hexahedral elements" with order-N
 * "Gauss-Lobatto-Legendre" bases -- an operator applied
 * "element-by-element or matrix-free" whose only coupling is the
 * "unit-depth" "gather-scatter phase", inside "preconditioned
 * Krylov subspace methods ... for each time step" ("CG together
 * with a block-Jacobi preconditioner").  The paper writes no
 * formula; the standard SEM definitions it cites (Deville, Fischer & Mund
 * 2002) are spelled out in DESIGN.md "Readings" (R1..R12 = SURVEY.md 8(c)
 * O1..O10) and referenced below.
 *
 * Conventions (all entry points):
 *   - lx = N + 1 nodes per direction, n3 = lx^3 nodes per element.
 *   - Local (element) layout of every field: double [E][n3], node (i,j,k) of
 *     element e at e*n3 + i + lx*j + lx*lx*k (i <-> r fastest)  [reading R3].
 *   - "device" pointers are CUDA device pointers on the mesh's device (any
 *     allocator: torch tensors, cudaMalloc); "host" pointers are host memory.
 *   - Ownership: the caller owns every pointer it passes and the library only
 *     borrows it for the duration of the call (stream-ordered for device
 *     pointers passed with a stream).  Host arrays given to sem_mesh_create
 *     are copied.  The mesh owns G, B, the gather-scatter plan and the CG
 *     work vectors; sem_mesh_destroy frees them.
 *   - Errors: every entry point returns a sem_status and never throws across
 *     the ABI.  On failure sem_last_error() returns a thread-local message.
 *     Non-convergence of CG is NOT an error (converged = 0); breakdown
 *     (pAp <= 0 or NaN) is SEM_EBREAKDOWN.
 *   - Collectives: when the mesh was created with a communicator,
 *     sem_gs_op(SEM_GS_ADD), sem_ax_dssum, sem_rhs, sem_jacobi and
 *     sem_cg_solve must be called by every rank in the same order.
 *   - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).
 *     Calls are asynchronous with respect to the host except sem_cg_solve,
 *     which synchronises `stream` before returning (it returns scalars).
 */
#ifndef SEM_B200_H
#define SEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sem_stream_t; /* == cudaStream_t */
typedef struct sem_mesh* sem_mesh_t;
typedef struct sem_comm* sem_comm_t;

typedef enum {
  SEM_OK = 0,
  SEM_EINVAL = 1,     /* bad argument, size, topology, or J <= 0 */
  SEM_ENOMEM = 2,     /* host or device allocation failed */
  SEM_ECUDA = 3,      /* CUDA runtime error (message has the CUDA string) */
  SEM_ENCCL = 4,      /* NCCL error */
  SEM_EBREAKDOWN = 5  /* CG breakdown: pAp <= 0 or NaN */
} sem_status;

enum { SEM_GS_ADD = 0, SEM_GS_MASK = 1 };

/* Library version string, e.g. "semb200 0.1 sm_100a". */
const char* sem_version(void);

/* Thread-local message describing the last failing call on this thread. */
const char* sem_last_error(void);

/* GLL nodes xi[0..N] (ascending, xi[0] = -1, xi[N] = 1) and weights w[0..N]
 * of order N >= 1 (reading R1), computed by the library's own rule
 * (Golub-Welsch on the Jacobi matrix of P^(1,1)_{N-1}).  host outputs, each
 * of N+1 doubles.  Used by callers to place mesh nodes.  EINVAL if N < 1 or
 * N > 15. */
sem_status sem_gll(int N, double* xi, double* w);

/* ---------------------------------------------------------------------- */
/* Multi-GPU bootstrap (optional; comm = NULL means a single GPU).          */
/* Elements are partitioned over ranks ("distributed among the
 * MPI ranks"); interface nodes are exchanged once per gather-scatter
 * ("unit-depth communication") by stores into the peers'
 * memory over NVLink (CUDA IPC mappings made at sem_comm_create /
 * sem_mesh_create), as are the CG scalar sums; NCCL carries the set-up
 * collectives and is the fallback when peer mappings are unavailable
 * (sem_comm_create_ex with p2p = 0 forces it).                             */

/* Rank 0 creates a 128-byte NCCL unique id (host buffer of 128 bytes),
 * which the caller broadcasts to all ranks. */
sem_status sem_comm_unique_id(void* id128);
/* Create the communicator of `rank` in [0, nranks) on CUDA `device`.
 * Collective over all ranks.  *out owned by the caller (sem_comm_destroy).
 * Uses NVLink peer memory for the data path when every rank can map every
 * peer (else NCCL). */
sem_status sem_comm_create(const void* id128, int rank, int nranks, int device,
                           sem_comm_t* out);
/* Same, with p2p = 0 forcing the NCCL data path (send/recv exchange and
 * ncclAllReduce scalars) even when peer mappings are available.  Every rank
 * must pass the same p2p value. */
sem_status sem_comm_create_ex(const void* id128, int rank, int nranks, int device, int p2p,
                              sem_comm_t* out);
/* Health of the communicator's peer-memory data path.  The in-kernel spins
 * that wait for a peer (exchange flags, scalar mailboxes) give up after ~2 s
 * and record the failure in a sticky device word instead of hanging; the
 * library checks it after every synchronising collective call (sem_cg_solve,
 * sem_jacobi's callers) and returns SEM_ENCCL, and from then on every
 * collective on this communicator fails fast with SEM_ENCCL (a lost peer
 * leaves the ranks' sequence counters out of step, so the path cannot be
 * reused; destroy and recreate the communicator).  This call synchronises the
 * device and returns SEM_OK or SEM_ENCCL.  *p2p_out (may be NULL) = 1 when
 * the peer-memory path is in use. */
sem_status sem_comm_status(sem_comm_t comm, int* p2p_out);
void sem_comm_destroy(sem_comm_t comm);

/* Host-only planning of the interface (no CUDA, no NCCL; what
 * sem_mesh_create does internally with a communicator, exposed so the
 * partition logic can be tested on CPU).
 * sem_iface_candidates: keys of the local entities that may be shared with
 *   another rank -- every face with a single local copy and its edges and
 *   vertices.  Key = 4 sorted global vertex ids, -1 padded (vertex: 1 id,
 *   edge: 2, face: 4).  host int64 keys[count][4]; pass keys = NULL to get
 *   the count only.
 * sem_iface_plan: given every rank's candidate counts (counts[nranks]) and
 *   keys (all_keys, concatenated in rank order), the number of interface
 *   NODES this rank exchanges with each rank (peer_nodes[nranks], host), the
 *   number of local interface entities and interface nodes. */
sem_status sem_iface_candidates(int64_t E_local, int N, const int64_t* conn, int64_t* count,
                                int64_t* keys);
sem_status sem_iface_plan(int64_t E_local, int N, const int64_t* conn, int rank, int nranks,
                          const int64_t* counts, const int64_t* all_keys, int64_t* peer_nodes,
                          int64_t* n_iface_entities, int64_t* n_iface_nodes);

/* ---------------------------------------------------------------------- */
/* Mesh.                                                                    */

/* Build a mesh of E_local elements of order N (1 <= N <= 11) on the current
 * CUDA device (E_local * (N+1)^3 < 2^31 local nodes).
 *   coords  host, double [3][E_local][n3]: x, y, z of every local node.
 *   conn    host, int64 [E_local][8]: GLOBAL vertex ids of the 8 corners;
 *           corner (a,b,c) in {0,1}^3 (the node (a*N, b*N, c*N)) at slot
 *           a + 2b + 4c.  Periodic images share ids.  A periodic direction
 *           needs >= 3 elements (else two distinct edges/faces would share a
 *           vertex key): violations -> EINVAL.
 *   bc      host, int8 [E_local][6] for faces r-, r+, s-, s+, t-, t+:
 *           0 = none/interior/periodic, 1 = Dirichlet; NULL = no Dirichlet.
 *           A node is masked if ANY copy lies on a Dirichlet face [R8].
 *   comm    NULL (single GPU) or a communicator; collective if non-NULL.
 * The gather-scatter numbering is built from `conn` alone (topology), never
 * from coordinates [reading R7].  Geometric factors are NOT computed yet
 * (call sem_geom_factors).  EINVAL on bad sizes, N out of range, duplicate
 * vertex ids inside an element, or non-conforming topology. */
sem_status sem_mesh_create(int64_t E_local, int N, const double* coords,
                           const int64_t* conn, const int8_t* bc, sem_comm_t comm,
                           sem_mesh_t* out);
void sem_mesh_destroy(sem_mesh_t m);

/* Per-mesh options (sem_mesh_set_options); defaults from
 * sem_options_default.  They replace environment variables: the library
 * reads no environment. */
enum { SEM_CG_STANDARD = 0, SEM_CG_PIPELINED = 1 };
enum { SEM_PC_JACOBI = 0, SEM_PC_HSMG = 1 };
enum { SEM_PRESSURE_CG = 0, SEM_PRESSURE_GMRES = 1 };
typedef struct {
  int cg_variant;    /* SEM_CG_STANDARD (reading R10, default) or SEM_CG_PIPELINED: the
                        single-reduction Chronopoulos-Gear PCG (same iterates in exact
                        arithmetic; one fused pass and one allreduce per iteration) */
  int affine;        /* 1: at sem_geom_factors (or now, if factors exist) test whether every
                        element is affine (G_ab / (w_i w_j w_k) constant per element to
                        1e-12) and, if so, run the affine-element operator (six metric
                        constants per element instead of G per node); default 0 */
  int graph;         /* 1 (default): the CG loop as one CUDA graph (a conditional WHILE node
                        around the captured iteration); 0: stream order */
  int pdl;           /* 1: one-rank CG iterations launch their kernels as programmatic
                        dependents (the operator's geometric-factor copies start while
                        the previous kernel drains); default 0 */
  int gmres_precond; /* preconditioner of sem_gmres_solve: SEM_PC_JACOBI (default, reading
                        R14) or SEM_PC_HSMG: one hybrid-Schwarz multigrid V-cycle
                        (sem_hsmg_apply, reading R16) per Arnoldi step, the Krylov method
                        then being flexible GMRES (Z_j = M v_j stored) */
  int hsmg_coarse_iters; /* K: at most K Jacobi-PCG steps (tol 1e-12) on the order-1
                        level of the V-cycle; default 5, 1..1000 */
  int pnpn_pressure; /* pressure solve of sem_pnpn_step: SEM_PRESSURE_CG (default, Jacobi-PCG)
                        or SEM_PRESSURE_GMRES: sem_gmres_solve (restart 30) with the mesh's
                        gmres_precond -- with SEM_PC_HSMG the paper's configuration
                        (GMRES + hybrid-Schwarz multigrid for the pressure,
                        CG + Jacobi for the velocity) */
  int cg_layout;     /* 1 (default): inside sem_cg_solve (standard variant) the operator
                        output A_e p is stored per element in the "x-planes last" layout
                        (rows in groups of four: interior nodes, then the i = 0 nodes, then
                        the i = lx-1 nodes), so the gather-scatter pass touches fewer
                        32-byte sectors; every caller-visible array keeps the [E][lx^3]
                        layout and the arithmetic is unchanged.  0: natural layout */
} sem_options_t;
void sem_options_default(sem_options_t* opt);

typedef struct {
  int64_t E;            /* local elements */
  int N, lx;
  int64_t n_local;      /* E * lx^3 */
  int64_t n_unique;     /* unique nodes, GLOBAL over all ranks */
  int64_t n_entities;   /* local faces + edges + vertices (shared-node groups) */
  int64_t n_masked;     /* masked local nodes */
  int64_t n_interface;  /* local interface nodes shared with other ranks */
  int64_t n_boundary_elements; /* local elements touching another rank */
  int rank, nranks;
  int n_peers;          /* ranks this rank exchanges with */
  int affine;           /* 1: every element affine and the affine-element operator
                           variant is on (option affine): six metric constants per
                           element replace the per-node G */
} sem_mesh_info_t;
sem_status sem_mesh_info(sem_mesh_t m, sem_mesh_info_t* info);

/* Set (or read back) the mesh's options.  Not collective; every rank should
 * use the same options.  Setting affine after sem_geom_factors runs the
 * detection immediately (synchronous). */
sem_status sem_mesh_set_options(sem_mesh_t m, const sem_options_t* opt);
sem_status sem_mesh_get_options(sem_mesh_t m, sem_options_t* opt);

/* Topological global node ids, host int64 [E_local][n3] (for tests): two
 * local nodes carry the same id iff they are the same global node. */
sem_status sem_mesh_global_ids(sem_mesh_t m, int64_t* ids);

/* Geometric factors [reading R4] from the mesh coordinates, on device:
 * G_ab = w_i w_j w_k J (grad r_a . grad r_b), ab = 11,22,33,12,13,23, and
 * B = w_i w_j w_k J.  EINVAL if J <= 0 anywhere (message names the element).
 * Synchronous. */
sem_status sem_geom_factors(sem_mesh_t m);

/* Copy G (device double [E][6][n3], order G11,G22,G33,G12,G13,G23) and B
 * (device double [E][n3]) out of the mesh (either may be NULL).  For parity
 * tests.  Synchronous. */
sem_status sem_geom_get(sem_mesh_t m, double* G, double* B);

/* Multiplicity weights mult = 1/m (device double [E][n3]) and mask (device
 * double [E][n3], 0 at masked nodes else 1) [readings R7, R8]. Synchronous. */
sem_status sem_mult_mask_get(sem_mesh_t m, double* mult, double* mask);

/* ---------------------------------------------------------------------- */
/* Operators.  h1, h2: device double [E][n3] or NULL -> constants h1c, h2c
 * [reading R6].  u and w must not alias.                                   */

/* Local (unassembled) operator [reading R5]: w = A_e u element by element,
 *   w = D^T q_r + D^T q_s + D^T q_t + h2 B u,  q_a = h1 sum_b G_ab (D_b u). */
sem_status sem_ax(sem_mesh_t m, const double* u, double* w, const double* h1,
                  const double* h2, double h1c, double h2c, sem_stream_t stream);

/* Gather-scatter on a local field (device double [E][n3], in place):
 *   SEM_GS_ADD  -- dssum [R7]: every copy <- sum of all copies of its global
 *                  node, summed in ascending element order; across ranks the
 *                  per-rank partial sums are added in ascending rank order.
 *                  Collective when the mesh has a communicator.
 *   SEM_GS_MASK -- u <- 0 at masked nodes [R8]. */
sem_status sem_gs_op(sem_mesh_t m, double* u, int op, sem_stream_t stream);

/* Fused w = mask . dssum(A_e u): the benchmarked operator ("Ax+dssum").
 * The operator kernel over all elements, then one gather-scatter kernel over
 * the shared nodes (precomputed copy offsets); with a communicator the
 * boundary elements run first and the interface exchange overlaps the
 * interior launch.  Same results as sem_ax + sem_gs_op(ADD) +
 * sem_gs_op(MASK), bit for bit. */
sem_status sem_ax_dssum(sem_mesh_t m, const double* u, double* w, const double* h1,
                        const double* h2, double h1c, double h2c, sem_stream_t stream);

/* Assembled right-hand side b = mask . dssum(B f) [reading R11]; f, b
 * device double [E][n3] (may alias).  Collective with a communicator. */
sem_status sem_rhs(sem_mesh_t m, const double* f, double* b, sem_stream_t stream);

/* Jacobi inverse diagonal [reading R9]: dinv = 1 / dssum(diag A_e), 1 at
 * masked nodes; device double [E][n3].  Collective with a communicator. */
sem_status sem_jacobi(sem_mesh_t m, const double* h1, const double* h2, double h1c,
                      double h2c, double* dinv, sem_stream_t stream);

/* Jacobi-preconditioned CG [reading R10] for A x = b with
 * A = mask . dssum . A_e (Helmholtz h1/h2, or Poisson h1 = 1, h2 = 0).
 *   b     device [E][n3], assembled and continuous (see sem_rhs); not modified
 *         (the solver masks it, and projects out the mean when the system is
 *         singular: no masked node anywhere and h2 == 0).
 *   x     device [E][n3], output (x0 = 0).
 *   tol   relative tolerance on the mult-weighted residual norm
 *         ||r_k|| <= tol ||b||; tol = 0 runs exactly maxit iterations.
 *   iters, rel_res, converged: host outputs.
 * Collective with a communicator; synchronises `stream`. */
sem_status sem_cg_solve(sem_mesh_t m, const double* b, double* x, const double* h1,
                        const double* h2, double h1c, double h2c, double tol, int maxit,
                        int* iters, double* rel_res, int* converged, sem_stream_t stream);

/* Restarted GMRES(restart) with right Jacobi preconditioning M = diag(dinv)
 * for the same system ("restarted GMRES for the pressure
 * solves"; reading R14 in DESIGN.md: Saad 2003 Alg. 9.5 with
 * Givens rotations; the Arnoldi step by classical Gram-Schmidt with one
 * re-orthogonalisation).  Same conventions as sem_cg_solve: b device
 * [E][n3] assembled and continuous (masked; projected when singular), x0 = 0,
 * mult-weighted inner products, stopping rule |g_{j+1}| <= tol ||b|| on the
 * Arnoldi residual estimate, tol = 0 runs exactly maxit Arnoldi steps.
 *   restart  Krylov basis length per cycle, 1..30 (the mesh keeps restart+1
 *            basis vectors of E*n3 doubles on the device)
 *   iters    Arnoldi steps done; rel_res: TRUE residual ||b - A x|| / ||b||
 *            at the end (one extra operator application per cycle)
 * Preconditioner: sem_options_t.gmres_precond.  With SEM_PC_HSMG the method
 * is flexible GMRES with one sem_hsmg_apply V-cycle per step (constant
 * coefficients only: h1, h2 must be NULL, else SEM_EINVAL; restart+1 more
 * basis vectors on the device).
 * Collective with a communicator; synchronises `stream` once per cycle.
 * SEM_EBREAKDOWN on a zero Givens pivot. */
sem_status sem_gmres_solve(sem_mesh_t m, const double* b, double* x, const double* h1,
                           const double* h2, double h1c, double h2c, double tol, int maxit,
                           int restart, int* iters, double* rel_res, int* converged,
                           sem_stream_t stream);

/* One hybrid-Schwarz multigrid V-cycle z = M r, the pressure preconditioner
 * of the paper's solver ("restarted GMRES for the
 * pressure solves with a hybrid-Schwarz multigrid preconditioner"; reading
 * R16 in DESIGN.md): levels of order N, N/2 (if > 1) and 1 on the same
 * elements (the fine element map evaluated at each level's GLL nodes);
 * on every level but the coarsest an averaged additive Schwarz smoother
 * (element-local fast-diagonalisation solves of the separable box
 * operator, summed by dssum and divided by the multiplicity) and the
 * restricted residual; on order 1 at most hsmg_coarse_iters Jacobi-PCG steps
 * (tol 1e-12); then the interpolated corrections added back level by level.
 *   r     device [E][n3], assembled (continuous) and masked residual
 *   z     device [E][n3], output (continuous, masked); must not alias r
 *   h1c, h2c  constant coefficients of the Helmholtz operator (R6)
 * The first call builds the levels (collective with a communicator: every
 * rank must make it).  Collective with a communicator; asynchronous on
 * `stream` (no host synchronisation). */
sem_status sem_hsmg_apply(sem_mesh_t m, const double* r, double* z, double h1c, double h2c,
                          sem_stream_t stream);

/* One first-order velocity-pressure splitting time step of the
 * incompressible Navier-Stokes equations ("the
 * exact splitting of the velocity and pressure follows ... Karniadakis
 * (1991)"; reading R15 in DESIGN.md: BDF1 / EXT1, periodic meshes):
 *   c_i = dssum(W J (u.grad)u_i)                 explicit convection
 *   u~_i = (dssum(B u_i) - dt c_i) / dssum(B)    predictor
 *   A p = dssum((grad v, u~)) / dt               pressure Poisson (PCG)
 *   (nu A + B/dt) u_i = dssum(B u~_i / dt - W J dp/dx_i)   velocity (PCG x 3)
 *   u   device [3][E][n3], the continuous velocity; overwritten by u^{n+1}
 *   p   device [E][n3], output pressure (mean-zero)
 *   dt, nu > 0 (nu = 1/Re); tol, maxit: of each PCG solve
 *   iters host int[4] (may be NULL): pressure, then the three velocity solves
 * EINVAL on meshes with Dirichlet faces (wall conditions of the splitting are
 * out of scope).  Collective with a communicator; synchronises `stream`. */
sem_status sem_pnpn_step(sem_mesh_t m, double* u, double* p, double dt, double nu, double tol,
                         int maxit, int* iters, sem_stream_t stream);

/* Same solve with b and x in HOST memory: the host<->device copies happen
 * inside the call on `stream` (end-to-end path).  h1/h2 device or NULL. */
sem_status sem_cg_solve_host(sem_mesh_t m, const double* b_host, double* x_host,
                             const double* h1, const double* h2, double h1c, double h2c,
                             double tol, int maxit, int* iters, double* rel_res,
                             int* converged, sem_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Instrumentation: when enabled, sem_ax_dssum and sem_cg_solve record CUDA
 * events around every launch of the fused operator kernel on its stream.
 * sem_profile_get returns (host outputs, each may be NULL) the number of
 * timed operator launches and their summed device time in ms since the last
 * sem_profile_enable, and the total number of CUDA kernels the library has
 * launched for this mesh since its creation (all kernels, any call).
 * Synchronises the recorded events. */
sem_status sem_profile_enable(sem_mesh_t m, int on);
sem_status sem_profile_get(sem_mesh_t m, int64_t* launches, double* ms,
                           int64_t* kernel_launches);

#ifdef __cplusplus
}
#endif
#endif /* SEM_B200_H */
