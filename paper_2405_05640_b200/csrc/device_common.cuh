// Device helpers shared by the kernel translation units (header-only,
// internal linkage).  See kernels.cu / ax.cu.
#pragma once
#include <stdint.h>

#include "internal.h"

#define SEM_COUNT_LAUNCH(m) (const_cast<sem_mesh*>(m)->nlaunch++)
// run CALL with the compile-time LX of the runtime order LXV (2..12)
#define SEM_LX_DISPATCH(LXV, CALL)                  \
  switch (LXV) {                                    \
    case 2: { constexpr int LX = 2; CALL; } break;  \
    case 3: { constexpr int LX = 3; CALL; } break;  \
    case 4: { constexpr int LX = 4; CALL; } break;  \
    case 5: { constexpr int LX = 5; CALL; } break;  \
    case 6: { constexpr int LX = 6; CALL; } break;  \
    case 7: { constexpr int LX = 7; CALL; } break;  \
    case 8: { constexpr int LX = 8; CALL; } break;  \
    case 9: { constexpr int LX = 9; CALL; } break;  \
    case 10: { constexpr int LX = 10; CALL; } break; \
    case 11: { constexpr int LX = 11; CALL; } break; \
    case 12: { constexpr int LX = 12; CALL; } break; \
    default: return cudaErrorInvalidValue;          \
  }

// OUT = EXPR evaluated with the compile-time LX of the runtime order LXV
#define SEM_LX_DISPATCH_INT(LXV, OUT, EXPR)               \
  switch (LXV) {                                          \
    case 2: { constexpr int LX = 2; OUT = EXPR; } break;  \
    case 3: { constexpr int LX = 3; OUT = EXPR; } break;  \
    case 4: { constexpr int LX = 4; OUT = EXPR; } break;  \
    case 5: { constexpr int LX = 5; OUT = EXPR; } break;  \
    case 6: { constexpr int LX = 6; OUT = EXPR; } break;  \
    case 7: { constexpr int LX = 7; OUT = EXPR; } break;  \
    case 8: { constexpr int LX = 8; OUT = EXPR; } break;  \
    case 9: { constexpr int LX = 9; OUT = EXPR; } break;  \
    case 10: { constexpr int LX = 10; OUT = EXPR; } break; \
    case 11: { constexpr int LX = 11; OUT = EXPR; } break; \
    case 12: { constexpr int LX = 12; OUT = EXPR; } break; \
    default: break;                                       \
  }

namespace sem {
namespace {

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + 1D bulk async copy (TMA engine), L2 policy
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// expected transaction bytes without an arrival (the arrival comes later)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global load / store with an L2 eviction-priority policy
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_hint_rw(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// gpu-scope release store / acquire load (per-position completion flags of
// the fused gather-scatter)
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// 16-byte asynchronous global -> shared copies (LDGSTS), completed by
// cp.async.wait_all in the issuing thread
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// programmatic dependent launch (sm_90+): wait for the previous kernel of the
// stream (its memory visible), and allow the next one to launch early
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Local node offset of canonical node n of an entity copy (slot, orient);
// device twin of copy_node_offset() in topo.cpp.
template <int LX>
__device__ __forceinline__ int node_offset(int slot, int orient, int n) {
  constexpr int N = LX - 1, M = LX - 2, MD = M > 0 ? M : 1;
  int i, j, k;
  if (slot < kEdgeSlot0) {
    const int a = n % MD, b = n / MD;
    const int du = (orient & 4) ? b : a, dv = (orient & 4) ? a : b;
    const int u = 1 + ((orient & 1) ? M - 1 - du : du);
    const int v = 1 + ((orient & 2) ? M - 1 - dv : dv);
    const int side = (slot & 1) ? N : 0, ax = slot >> 1;
    i = ax == 0 ? side : u;
    j = ax == 0 ? u : (ax == 1 ? side : v);
    k = ax == 2 ? side : v;
  } else if (slot < kVertSlot0) {
    const int ed = slot - kEdgeSlot0, ax = ed >> 2, q = ed & 3;
    const int t = 1 + ((orient & 1) ? M - 1 - n : n);
    const int p = (q & 1) * N, r = (q >> 1) * N;
    i = ax == 0 ? t : p;
    j = ax == 0 ? p : (ax == 1 ? t : r);
    k = ax == 2 ? t : r;
  } else {
    const int c = slot - kVertSlot0;
    i = (c & 1) * N;
    j = ((c >> 1) & 1) * N;
    k = (c >> 2) * N;
  }
  return i + LX * (j + LX * k);
}

// The "x-planes last" element layout of the operator output in the CG
// (DESIGN.md §4).  Rows r = j + lx k of an element are taken in groups of
// four; a group stores the interior nodes 0 < i < lx-1 of its rows (row
// after row), then their i = 0 nodes, then their i = lx-1 nodes.  The
// x-face nodes then come in 32-byte runs (one sector each) instead of one
// per 64-byte row, and at lx = 8 a warp of the operator (four rows of one
// plane) still writes one contiguous 256-byte block.
template <int LX>
__device__ __forceinline__ int xlast_pos(int q) {
  constexpr int NT = LX * LX;
  const int i = q % LX, r = q / LX, g = r >> 2, rr = r & 3;
  const int gs = min(4, NT - 4 * g), gb = 4 * g * LX;
  return (i >= 1 && i <= LX - 2) ? gb + rr * (LX - 2) + (i - 1) : gb + gs * (LX - 2) + (i == LX - 1 ? gs : 0) + rr;
}

// deterministic block sum of NV values (fixed tree); result valid in thread 0
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* s_red /* >= 32*NV */) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nt = blockDim.x * blockDim.y * blockDim.z;
  const int nw = (nt + 31) >> 5;
  const int lane = tid & 31;
  const int active = min(32, nt - (tid & ~31));  // lanes present in this warp
  const unsigned wmask = active == 32 ? 0xffffffffu : ((1u << active) - 1u);
#pragma unroll
  for (int q = 0; q < NV; ++q)
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_down_sync(wmask, v[q], o);
      if (lane + o < active) v[q] += t;
    }
  if ((tid & 31) == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) s_red[q * 32 + (tid >> 5)] = v[q];
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += s_red[q * 32 + w];
      v[q] = s;
    }
  }
}

// Partials written per block, the last block to arrive (ticket) sums them in
// block order -> deterministic.  part: [nblk][NV]; out: NV doubles.
// nblk_in > 0: only blocks [0, nblk_in) take part (the others must not call)
template <int NV>
__device__ __forceinline__ void grid_sum_last_block(double (&v)[NV], double* part, unsigned* ticket,
                                                    double* out, double* s_red, int* s_flag, unsigned nblk_in = 0) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nt = blockDim.x * blockDim.y * blockDim.z;
  const unsigned nblk = nblk_in ? nblk_in : gridDim.x;
  block_sum<NV>(v, s_red);
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) part[(size_t)blockIdx.x * NV + q] = v[q];
    __threadfence();
    const unsigned t = atomicInc(ticket, nblk - 1);
    *s_flag = (t == nblk - 1);
  }
  __syncthreads();
  if (*s_flag) {
    __threadfence();
    double acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
    for (unsigned b = tid; b < nblk; b += nt) {
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[q] += __ldcg(&part[(size_t)b * NV + q]);
    }
    __syncthreads();
    block_sum<NV>(acc, s_red);
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < NV; ++q) out[q] = acc[q];
    }
  }
}

}  // namespace
}  // namespace sem
