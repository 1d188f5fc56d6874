// Accuracy of the MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and of one/two
// refinement variants over r^2 in [1e-12, 1e4] (the quadrature range).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(int n, double *err) {
  double e0 = 0, e1 = 0, e2 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = exp(-27.6 + 36.8 * (i + 0.5) / n);  // 1e-12 .. 1e4
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double ref = 1.0 / sqrt(x);
    const double e = fma(-x, y * y, 1.0);
    const double y1 = fma(0.5 * y, e, y);                      // first order
    const double y2 = fma(fma(e, 0.375, 0.5), y * e, y);       // second order
    e0 = fmax(e0, fabs(y - ref) / ref);
    e1 = fmax(e1, fabs(y1 - ref) / ref);
    e2 = fmax(e2, fabs(y2 - ref) / ref);
  }
  atomicMax((unsigned long long *)&err[0], __double_as_longlong(e0));
  atomicMax((unsigned long long *)&err[1], __double_as_longlong(e1));
  atomicMax((unsigned long long *)&err[2], __double_as_longlong(e2));
}
int main() {
  double *d, h[3];
  cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
  k<<<1184, 256>>>(1 << 28, d);
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("max rel err: seed %.3e (2^%.1f)  first-order %.3e  second-order %.3e\n", h[0],
         log2(h[0]), h[1], h[2]);
  return 0;
}
