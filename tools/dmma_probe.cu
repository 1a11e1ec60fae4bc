// DMMA experiment ("tensor cores only if an fp64 DMMA
// formulation of the derivative contractions is shown to beat the CUDA-core
// path"; round-1 review item 5).  Measures the three tensor-product
// derivative contractions of one lx = 8 element (ur = D_r u, us = D_s u,
// ut = D_t u over the 8x8x8 tile), the compute core of the operator, with
// the element tile resident in shared memory and the inputs L2-resident, so
// the kernels are bound by the SM (shared-memory pipe, fp64 pipe), not by
// HBM:
//   cuda : the operator's mapping -- thread (i,j) owns column (i,j,:), D rows
//          in registers, the r/s contractions from shared memory (LDS.128
//          along r), t from registers; 2 warps per element;
//   dmma : mma.sync.aligned.m8n8k4 f64 (DMMA): each direction is
//          C(8 x 64) = D(8 x 8) U(8 x 64) = 8 N-tiles x 2 K-steps = 16 MMAs,
//          B fragments loaded from the shared tile; 2 warps per element.
// Both write a checksum per element (ur + us + ut summed over the tile, in
// their own order) so nothing is dead code; the checksums agree to rounding.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
//   tools/dmma_probe      (prints the time per element of each kernel)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int LX = 8, N3 = 512, NT = 64;
__constant__ double cD[LX * LX];

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// u: [nsrc][512] (small, L2-resident); element e reads tile e % nsrc
__global__ void __launch_bounds__(NT, 7) k_cuda(const double* __restrict__ u, int nsrc, double* out, int reps) {
  __shared__ __align__(16) double su[N3];
  const int i = threadIdx.x, j = threadIdx.y, tid = i + LX * j;
  const double* ue = u + (size_t)(blockIdx.x % nsrc) * N3;
  for (int t = tid; t < N3; t += NT) su[t] = ue[t];
  __syncthreads();
  double Da[LX], Db[LX], uc[LX];
#pragma unroll
  for (int l = 0; l < LX; ++l) {
    Da[l] = cD[i * LX + l];
    Db[l] = cD[j * LX + l];
    uc[l] = su[tid + NT * l];
  }
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    // the operands change every repetition, so no contraction is hoisted
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      Da[l] *= 1.0000000001;
      Db[l] *= 1.0000000001;
      uc[l] *= 1.0000000001;
    }
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
      for (int l = 0; l < LX; l += 2) {
        const double2 v = *reinterpret_cast<const double2*>(su + l + LX * j + NT * k);
        ur = fma(Da[l], v.x, ur);
        ur = fma(Da[l + 1], v.y, ur);
      }
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        us = fma(Db[l], su[i + LX * l + NT * k], us);
        ut = fma(cD[k * LX + l], uc[l], ut);
      }
      acc += ur + us + ut;
    }
  }
  out[(size_t)blockIdx.x * NT + tid] = acc;
}

__global__ void __launch_bounds__(NT, 7) k_dmma(const double* __restrict__ u, int nsrc, double* out, int reps) {
  __shared__ __align__(16) double su[N3];
  const int tid = threadIdx.x + LX * threadIdx.y, lane = tid & 31, warp = tid >> 5;
  const double* ue = u + (size_t)(blockIdx.x % nsrc) * N3;
  for (int t = tid; t < N3; t += NT) su[t] = ue[t];
  __syncthreads();
  // A fragments (D rows, K halves): A[row = lane/4][col = lane%4 + 4h]
  const double a0 = cD[(lane >> 2) * LX + (lane & 3)], a1 = cD[(lane >> 2) * LX + (lane & 3) + 4];
  const int bl = lane & 3, bn = lane >> 2;  // B fragment: row (l) = lane%4 (+4h), column = lane/4
  double acc = 0.0;
  double a0r = a0, a1r = a1;
  for (int r = 0; r < reps; ++r) {
    a0r *= 1.0000000001;  // (as in k_cuda: nothing can be hoisted)
    a1r *= 1.0000000001;
    // each warp: 4 of the 8 N-tiles of each direction
#pragma unroll
    for (int tt = 0; tt < 4; ++tt) {
      const int c = (warp * 4 + tt) * 8 + bn;  // the column (of 64) this lane feeds
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0;
      // r: column c = (j,k) -> u[l + 8c]
      dmma(d0, d1, a0r, su[bl + 8 * c], d0, d1);
      dmma(d0, d1, a1r, su[bl + 4 + 8 * c], d0, d1);
      // s: column c = (i,k) = (c%8, c/8) -> u[i + 8l + 64k]
      dmma(e0, e1, a0r, su[(c & 7) + 8 * bl + 64 * (c >> 3)], e0, e1);
      dmma(e0, e1, a1r, su[(c & 7) + 8 * (bl + 4) + 64 * (c >> 3)], e0, e1);
      // t: column c = (i,j) -> u[c + 64l]
      dmma(f0, f1, a0r, su[c + 64 * bl], f0, f1);
      dmma(f0, f1, a1r, su[c + 64 * (bl + 4)], f0, f1);
      acc += d0 + d1 + e0 + e1 + f0 + f1;
    }
  }
  out[(size_t)blockIdx.x * NT + tid] = acc;
}

int main() {
  const int E = 148 * 7 * 64, nsrc = 64, reps = 16;
  std::vector<double> D(LX * LX), hu((size_t)nsrc * N3);
  for (int k = 0; k < LX * LX; ++k) D[k] = 0.01 * ((k * 37) % 17 - 8);
  for (size_t k = 0; k < hu.size(); ++k) hu[k] = 1e-3 * (double)((k * 7919) % 1000);
  cudaMemcpyToSymbol(cD, D.data(), sizeof(double) * LX * LX);
  double *du, *o1, *o2;
  cudaMalloc(&du, sizeof(double) * hu.size());
  cudaMalloc(&o1, sizeof(double) * (size_t)E * NT);
  cudaMalloc(&o2, sizeof(double) * (size_t)E * NT);
  cudaMemcpy(du, hu.data(), sizeof(double) * hu.size(), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, double* o, const char* name) {
    for (int w = 0; w < 3; ++w) kern<<<E, dim3(LX, LX)>>>(du, nsrc, o, reps);
    cudaEventRecord(a);
    for (int w = 0; w < 10; ++w) kern<<<E, dim3(LX, LX)>>>(du, nsrc, o, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms / 10.0 * 1e6 / ((double)E * reps);  // ns per element-contraction set
    const double flops = 3.0 * 2 * 512 * 8 * (double)E * reps / (ms / 10.0 * 1e-3);
    printf("{\"kernel\": \"%s\", \"ns_per_element\": %.3f, \"contraction_tflops\": %.2f, \"err\": \"%s\"}\n", name,
           per, flops / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run(k_cuda, o1, "cuda-core (operator mapping)");
  run(k_dmma, o2, "dmma m8n8k4");
  // checksum agreement (sum over all outputs)
  std::vector<double> h1((size_t)E * NT), h2((size_t)E * NT);
  cudaMemcpy(h1.data(), o1, sizeof(double) * h1.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), o2, sizeof(double) * h2.size(), cudaMemcpyDeviceToHost);
  double s1 = 0, s2 = 0;
  for (size_t k = 0; k < h1.size(); ++k) {
    s1 += h1[k];
    s2 += h2[k];
  }
  printf("{\"checksum_cuda\": %.15e, \"checksum_dmma\": %.15e, \"rel_diff\": %.3e}\n", s1, s2,
         std::abs(s1 - s2) / std::abs(s1));
  // the CUDA-core kernel also scales u by (1 + 1e-10) per repetition: the
  // checksums differ by ~reps * 1e-10 relative (a consistency check only)
  return 0;
}
