// Microbenchmark: FP64 dependent-chain latency and MUFU.RSQ64H latency on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double *out, long long *cyc, int iters, double a) {
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, 1e-9);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lat_rsq(double *out, long long *cyc, int iters) {
  double x = threadIdx.x * 1e-3 + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
      x = y + 1.5;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: many independent chains per thread, many warps
__global__ void k_thr(double *out, int iters, double a) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, 1e-9);
  double s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *out; long long *cyc, h;
  cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 8);
  int iters = 1000;
  k_lat<<<1, 32>>>(out, cyc, iters, 0.999); cudaDeviceSynchronize();
  k_lat<<<1, 32>>>(out, cyc, iters, 0.999); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (iters * 16));
  k_lat_rsq<<<1, 32>>>(out, cyc, iters); cudaDeviceSynchronize();
  k_lat_rsq<<<1, 32>>>(out, cyc, iters); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("MUFU.RSQ64H + DADD dependent latency: %.2f cycles\n", (double)h / (iters * 16));
  // issue throughput per SM with w warps of 8 chains
  for (int w = 1; w <= 32; w *= 2) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int blocks = 148;
    k_thr<<<blocks, 32 * w>>>(out, 2000, 0.999);
    cudaEventRecord(a); k_thr<<<blocks, 32 * w>>>(out, 2000, 0.999); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * blocks * 32.0 * w * 2000 * 8;
    printf("warps/SM %2d x 8 chains: %.2f TFLOP/s fp64\n", w, flops / ms / 1e9);
  }
  return 0;
}
