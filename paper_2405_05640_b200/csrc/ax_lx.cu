// One order of the operator kernel (ax_kernel.cuh): compiled once per lx
// with -DSEM_AX_LX=lx (build.py), so the orders compile in parallel.
#include "ax_kernel.cuh"

#ifndef SEM_AX_LX
#error "compile with -DSEM_AX_LX=<lx>"
#endif

namespace sem {
template cudaError_t ax_upload_basis_lx<SEM_AX_LX>(const double*, const double*);
template cudaError_t ax_launch_lx<SEM_AX_LX>(const sem_mesh*, const AxKP&, int, bool, int64_t, cudaStream_t);
template cudaError_t ax_affine_detect_lx<SEM_AX_LX>(const sem_mesh*, double*, int*, cudaStream_t);
template int ax_occupancy_lx<SEM_AX_LX>();
}  // namespace sem
