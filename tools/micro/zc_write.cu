// SM stores straight into page-locked host memory (zero-copy over PCIe):
// bandwidth vs grid size, against the copy engine (cudaMemcpyAsync D2H).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_zc(const double2 *src, double2 *dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_busy(double *out, int iters) {
  double a = threadIdx.x;
  for (int i = 0; i < iters; ++i) a = fma(a, 0.999999, 1e-9);
  if (a == 1.2345) out[0] = a;
}

int main() {
  const long long bytes = 8ll << 30, n = bytes / 16;
  double2 *d, *h;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("copy engine D2H: %.1f GB/s\n", bytes / ms / 1e6);
  }
  int grids[] = {4, 8, 16, 32, 64, 148, 296, 1184};
  for (int threads : {256, 1024})
    for (int g : grids) {
      cudaEventRecord(a);
      k_zc<<<g, threads>>>(d, h, n);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("zero-copy %4d CTAs x %4d: %.1f GB/s (%s)\n", g, threads, bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  // concurrent with a compute kernel filling the other SMs
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  double *o;
  cudaMalloc(&o, 8);
  for (int g : {16, 32}) {
    cudaEventRecord(a, s1);
    k_zc<<<g, 1024, 0, s1>>>(d, h, n);
    cudaEventRecord(b, s1);
    k_busy<<<148 * 8, 256, 0, s2>>>(o, 2000000);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("zero-copy %d CTAs beside a busy grid: %.1f GB/s\n", g, bytes / ms / 1e6);
    cudaDeviceSynchronize();
  }
  return 0;
}
