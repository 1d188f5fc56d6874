// Which allocation calls wait for in-flight device work? A 300 ms kernel runs
// on a non-blocking stream while the host times each call.
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  cudaFree(0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  size_t step = 2ull << 30;
  CUdeviceptr base;
  cuMemAddressReserve(&base, 64ull << 30, 0, 0, 0);
  void *pinned;
  cudaHostAlloc(&pinned, 1 << 30, 0);
  void *dbuf;
  cudaMalloc(&dbuf, 1 << 30);
  for (int rep = 0; rep < 2; ++rep) {
    const long long cyc = 600000000ll;  // ~0.3 s at 1.9 GHz
    double t;
    auto spin = [&]() { k_spin<<<1, 1, 0, s>>>(cyc); cudaMemcpyAsync(pinned, dbuf, 1 << 30, cudaMemcpyDeviceToHost, s); };
    spin();
    t = now();
    CUmemGenericAllocationHandle h;
    cuMemCreate(&h, step, &prop, 0);
    printf("cuMemCreate      %.4f s\n", now() - t);
    t = now();
    cuMemMap(base + rep * step, step, 0, h, 0);
    printf("cuMemMap         %.4f s\n", now() - t);
    t = now();
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cuMemSetAccess(base + rep * step, step, &acc, 1);
    printf("cuMemSetAccess   %.4f s\n", now() - t);
    cudaStreamSynchronize(s);
    spin();
    t = now();
    void *p;
    cudaMalloc(&p, 1ull << 30);
    printf("cudaMalloc 1 GB  %.4f s\n", now() - t);
    t = now();
    void *p2;
    cudaMalloc(&p2, 1 << 20);
    printf("cudaMalloc 1 MB  %.4f s\n", now() - t);
    t = now();
    cudaFree(p2);
    printf("cudaFree 1 MB    %.4f s\n", now() - t);
    cudaStreamSynchronize(s);
  }
  return 0;
}
