// The finalizer of the fused gather-scatter (DESIGN.md "Fused
// gather-scatter"; readings R7, R8): k_gs_fin runs beside the persistent
// operator launch on a second stream, one warp per CTA, and finishes every
// shared entity of the launch segment as soon as the operator has published
// the completion flags of all positions holding its copies.  Only this kernel
// waits (the operator never does), so the two cannot deadlock whether or not
// they are co-resident.
#pragma once
#include <stdint.h>

#include "device_common.cuh"

namespace sem {

// Finish the groups of one finalizer list (FinDesc): per group, sum the m
// copies in ascending element order (from L2: ld.cg) and store the sum -- 0
// if masked -- to every copy, once every position holding a copy has
// released its completion flag (acquire).  Called by all NT threads of the
// CTA.  Latency-bound by construction (descriptor -> offsets -> values), so
// every thread handles its groups in rounds of KG with all loads of a round in
// flight, the offsets of the first round are requested before the flag wait,
// and the persistent operator calls it while its element's operands are in
// flight.
constexpr int kFinKG = 2;  // groups per thread per round
// sdesc != nullptr: the descriptor was prefetched into shared memory.
__device__ __forceinline__ void fin_run(const FinArgs& F, double* __restrict__ w, int64_t q, int list,
                                        unsigned long long ep, unsigned* err, int tid, int NT,
                                        const uint4* sdesc = nullptr) {
  const uint4* dp = reinterpret_cast<const uint4*>(F.desc + 2 * q + list);
  const uint4 d0 = sdesc ? sdesc[0] : __ldg(dp), d1 = sdesc ? sdesc[1] : __ldg(dp + 1);
  int cnt[kFinMaxM];
  cnt[0] = d0.z & 0xffff;
  cnt[1] = d0.z >> 16;
  cnt[2] = d0.w & 0xffff;
  cnt[3] = d0.w >> 16;
  cnt[4] = d1.x & 0xffff;
  cnt[5] = d1.x >> 16;
  cnt[6] = d1.y & 0xffff;
  cnt[7] = d1.y >> 16;
  const int ndep = d1.z & 0xffff;
  // class c (m = c + 1) holds groups [cum[c], cum[c+1]) at words wb[c] + (g - cum[c]) m
  int cum[kFinMaxM + 1];
  uint32_t wb[kFinMaxM];
  cum[0] = 0;
  uint32_t off = d0.x;
#pragma unroll
  for (int c = 0; c < kFinMaxM; ++c) {
    off = (off + 3) & ~3u;
    wb[c] = off;
    off += (uint32_t)cnt[c] * (c + 1);
    cum[c + 1] = cum[c] + cnt[c];
  }
  const int tot = cum[kFinMaxM];
  if (tot == 0) return;
  bool waited = false;
  for (int g0 = 0; g0 < tot; g0 += kFinKG * NT) {
    uint32_t o[kFinKG][kFinMaxM];
    int mg[kFinKG];
#pragma unroll
    for (int r = 0; r < kFinKG; ++r) {
      const int g = g0 + tid + r * NT;
      // class of group g by a select chain (no dynamically indexed arrays:
      // they would live in local memory)
      int m = 1, c0 = 0;
      uint32_t base = wb[0];
#pragma unroll
      for (int cc = 1; cc < kFinMaxM; ++cc)
        if (g >= cum[cc]) {
          m = cc + 1;
          c0 = cum[cc];
          base = wb[cc];
        }
      mg[r] = (g < tot) ? m : 0;
      const uint32_t* src = F.idx + base + (uint32_t)(g - c0) * m;
#pragma unroll
      for (int k = 0; k < kFinMaxM; ++k) o[r][k] = (k < mg[r]) ? __ldg(src + k) : 0u;
    }
    if (!waited) {  // the copies' positions must have released their flags
      waited = true;
      if (tid < 32) {
        const unsigned wmask = NT >= 32 ? 0xffffffffu : ((1u << NT) - 1u);  // lanes present
        for (int k = tid; k < ndep; k += 32) {
          const unsigned long long* f = F.flag + F.dep[d0.y + k];
          long long t0 = 0;
          while (ld_acquire_gpu(f) < ep) {
            if (t0 == 0) t0 = clock64();
            else if (clock64() - t0 > (1ll << 31)) {  // ~1 s: record and go on (never hang)
              atomicOr(err, 1u);
              break;
            }
          }
        }
        __syncwarp(wmask);
      }
      __syncthreads();
    }
    double v[kFinKG][kFinMaxM];
#pragma unroll
    for (int r = 0; r < kFinKG; ++r) {
      const bool masked = (o[r][0] & kFinMasked) != 0;
      o[r][0] &= ~kFinMasked;
#pragma unroll
      for (int k = 0; k < kFinMaxM; ++k) v[r][k] = (k < mg[r] && !masked) ? __ldcg(w + o[r][k]) : 0.0;
      if (masked) mg[r] = -mg[r];
    }
#pragma unroll
    for (int r = 0; r < kFinKG; ++r) {
      const int m = mg[r] < 0 ? -mg[r] : mg[r];
      double s = 0.0;
      if (mg[r] > 0) {
#pragma unroll
        for (int k = 0; k < kFinMaxM; ++k)
          if (k < m) s += v[r][k];
      }
#pragma unroll
      for (int k = 0; k < kFinMaxM; ++k)
        if (k < m) w[o[r][k]] = s;
    }
  }
}


// One warp per CTA, persistent: items (owner positions, ascending) by ticket.
// skip != nullptr and *skip: the paired operator launch did nothing (CG done,
// GMRES cycle end), so neither does this one (the epochs stay paired).
__global__ void __launch_bounds__(32, 32) k_gs_fin(const FinArgs F, double* __restrict__ w, int64_t q0, int64_t count,
                                                   LaunchCtl* ctl, unsigned* err, const int* skip) {
  const int lane = threadIdx.x;
  if (skip && *skip) return;
  const unsigned long long ep = __ldcg(&ctl->epoch) + 1;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(&ctl->ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((int64_t)t >= count) break;
    fin_run(F, w, q0 + (int64_t)t, 0, ep, err, lane, 32);
  }
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(&ctl->exitcnt, 1u) == gridDim.x - 1) {
      ctl->exitcnt = 0;
      ctl->ticket = 0;
      ctl->epoch = ep;
      __threadfence();
    }
  }
}

}  // namespace sem
