// Ceiling of the ACA P0 quadrature (p0_quad, local-frame float64 Laplace SLP)
// in isolation: the k_aca_p0 loop structure (lane element in registers, fixed
// elements staged 8 at a time in shared memory) without residual / pivot
// epilogue or factor loads.  Prints the FP64-pipe utilisation implied by the
// SASS count of 9 FP64 instructions + 1 MUFU per quadrature-point pair.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -DMINB=4 tools/micro/quad_bench.cu -o var/quad_bench
#include <cstdio>
#include <vector>

#include "../../paper_1711_01897_b200/csrc/aca_impl.cuh"

#ifndef MINB
#define MINB 4
#endif
using namespace hb;

__global__ void __launch_bounds__(128, MINB)
    k_quad(RuleTab<double> R, const FixRec<double> *fix, int nfix, int njobs, double *out) {
  __shared__ FixRec<double> sr[4][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double y[18], ny[6], nl[4] = {0, 0, 1, 1e-3};
  const double base = 0.5 + 0.001 * lane + 0.01 * wid;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    y[3 * i] = base + 0.0003 * i;
    y[3 * i + 1] = 0.2 - 0.0002 * i;
    y[3 * i + 2] = 0.1 * lane * 1e-3;
    ny[i] = y[3 * i] * y[3 * i] + y[3 * i + 1] * y[3 * i + 1] + y[3 * i + 2] * y[3 * i + 2];
  }
  double acc = 0.0;
  for (int seg = 0; seg < njobs; seg += 8) {
    if (lane < 8) sr[wid][lane] = fix[(blockIdx.x * 7 + seg + lane) % nfix];
    __syncwarp();
    for (int q = 0; q < 8; ++q) {
      const FixRec<double> *const F1[1] = {&sr[wid][q]};
      double v[1];
      p0_quad<double, false, HBEM_SLP, false, true, 1>(R, F1, y, ny, nl, v);
      acc += v[0];
    }
    __syncwarp();
  }
  out[blockIdx.x * 128 + threadIdx.x] = acc;
}

int main() {
  const int nfix = 1024, njobs = 256;
  std::vector<FixRec<double>> h(nfix);
  for (int f = 0; f < nfix; ++f) {
    for (int o = 0; o < 6; ++o) {
      double x0 = -1.0 - 0.001 * f - 0.01 * o, x1 = 0.3 + 0.0001 * o, x2 = 0.05;
      h[f].p[o][0] = -2 * x0; h[f].p[o][1] = -2 * x1; h[f].p[o][2] = -2 * x2;
      h[f].p[o][3] = x0 * x0 + x1 * x1 + x2 * x2;
    }
    h[f].n[0] = 0; h[f].n[1] = 0; h[f].n[2] = 1; h[f].n[3] = 1e-3;
    h[f].ev = make_int4(3 * f, 3 * f + 1, 3 * f + 2, f);
  }
  RuleTab<double> R{};
  const double w[6] = {0.1116907948390057, 0.1116907948390057, 0.1116907948390057,
                       0.0549758718276609, 0.0549758718276609, 0.0549758718276609};
  for (int o = 0; o < 6; ++o)
    for (int i = 0; i < 6; ++i) R.w2[o][i] = w[o] * w[i];
  FixRec<double> *d;
  double *out;
  cudaMalloc(&d, nfix * sizeof(FixRec<double>));
  cudaMemcpy(d, h.data(), nfix * sizeof(FixRec<double>), cudaMemcpyHostToDevice);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = sms * MINB * 8;
  cudaMalloc(&out, (size_t)grid * 128 * 8);
  k_quad<<<grid, 128>>>(R, d, nfix, njobs, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k_quad<<<grid, 128>>>(R, d, nfix, njobs, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warp_jobs = (double)reps * grid * 4 * njobs;
  const double dp_warp_instr = warp_jobs * 36 * 9;
  // FP64 pipe: 16 lanes per SMSP per clock -> one warp instruction per 2 clocks
  const double cap = (double)sms * 4 * (clk * 1e3) / 2 * (ms * 1e-3);
  printf("MINB=%d grid=%d: %.3f ms, %.3e entries/s, FP64-pipe utilisation %.1f%% (at %d MHz)\n",
         MINB, grid, ms / reps, warp_jobs * 32 / (ms * 1e-3), 100 * dp_warp_instr / cap, clk / 1000);
  return 0;
}
