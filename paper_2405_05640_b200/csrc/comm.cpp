// Multi-GPU plumbing: NCCL communicator bootstrap, scalar allreduce and the
// interface exchange of the gather-scatter ("unit-depth
// communication"; PAPER.md:74 elements "distributed among the MPI ranks").
#include <cuda_runtime.h>

#include <string.h>

#include <string>

#include "internal.h"

namespace sem {

sem_status comm_setup_mesh(sem_mesh* m) {
  (void)m;
  return fail(SEM_EINVAL, "multi-GPU meshes are not implemented yet");
}

sem_status comm_allreduce_sum(sem_mesh* m, double* d, int n, cudaStream_t s) {
#ifdef SEM_WITH_NCCL
  ncclResult_t r = ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclSum, m->comm->nccl, s);
  if (r != ncclSuccess) return fail(SEM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  return SEM_OK;
#else
  (void)m; (void)d; (void)n; (void)s;
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

sem_status comm_gs_exchange(sem_mesh* m, double* u, cudaStream_t s) {
  (void)m; (void)u; (void)s;
  return SEM_OK;
}

void comm_mesh_free(sem_mesh* m) { (void)m; }

}  // namespace sem

using namespace sem;

extern "C" {

sem_status sem_comm_unique_id(void* id128) {
  if (!id128) return fail(SEM_EINVAL, "sem_comm_unique_id: NULL buffer");
#ifdef SEM_WITH_NCCL
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclResult_t r = ncclGetUniqueId((ncclUniqueId*)id128);
  if (r != ncclSuccess) return fail(SEM_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  return SEM_OK;
#else
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

sem_status sem_comm_create(const void* id128, int rank, int nranks, int device, sem_comm_t* out) {
  if (!id128 || !out) return fail(SEM_EINVAL, "sem_comm_create: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SEM_EINVAL, "sem_comm_create: bad rank/nranks");
  *out = nullptr;
#ifdef SEM_WITH_NCCL
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) return fail(SEM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce));
  sem_comm* c = new sem_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(SEM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  return SEM_OK;
#else
  (void)device;
  return fail(SEM_ENCCL, "built without NCCL");
#endif
}

void sem_comm_destroy(sem_comm_t c) {
  if (!c) return;
#ifdef SEM_WITH_NCCL
  if (c->nccl) ncclCommDestroy(c->nccl);
#endif
  delete c;
}

}  // extern "C"
