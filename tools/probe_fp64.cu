// Probe: fp64 FMA throughput and a plain fp64 streaming copy on the B200 box.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void read_kernel(const double2* __restrict__ a, double* out, size_t n) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; int blocks = sms * 8, threads = 256;
  fma_kernel<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0); fma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 64 * iters * (double)blocks * threads;
  printf("SMs %d  fp64 FMA: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965GHz)\n", sms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / 1.965e9);
  size_t n = (size_t)1 << 28;  // 4 GiB of double2? 2^28 * 16 B = 4 GiB
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  for (int g : {1, 2, 4, 8}) {
    int grid = sms * g;
    copy_kernel<<<grid, 512>>>(a, b, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copy_kernel<<<grid, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid=%d*SM: %.1f GB/s\n", g, 5 * 2.0 * n * 16 / ms / 1e6);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) read_kernel<<<grid, 512>>>(a, out, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read grid=%d*SM: %.1f GB/s\n", g, 5.0 * n * 16 / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
