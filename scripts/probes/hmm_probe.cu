// Probe: can the GPU read/write the process's pageable (malloc) memory
// directly (HMM / pageable memory access), and at what rate?
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
__global__ void copy_k(double* __restrict__ dst, const double* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  int pma = 0, pmaHPT = 0, cma = 0, hnrm = 0;
  cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, 0);
  cudaDeviceGetAttribute(&pmaHPT, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
  cudaDeviceGetAttribute(&cma, cudaDevAttrConcurrentManagedAccess, 0);
  cudaDeviceGetAttribute(&hnrm, cudaDevAttrHostNativeAtomicSupported, 0);
  std::printf("pageableMemoryAccess %d usesHostPageTables %d concurrentManagedAccess %d hostNativeAtomic %d\n", pma, pmaHPT, cma, hnrm);
  if (!pma) return 0;
  const size_t n = 43200112 / 8;
  double* dev; cudaMalloc(&dev, n * 8);
  std::vector<double> init(n); for (size_t i = 0; i < n; ++i) init[i] = i * 0.5;
  cudaMemcpy(dev, init.data(), n * 8, cudaMemcpyHostToDevice);
  double* host = (double*)std::malloc(n * 8);
  std::memset(host, 0, n * 8);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 1) {
      cudaError_t e1 = cudaMemAdvise(host, n * 8, cudaMemAdviseSetPreferredLocation, cudaCpuDeviceId);
      cudaError_t e2 = cudaMemAdvise(host, n * 8, cudaMemAdviseSetAccessedBy, 0);
      std::printf("advise: %s %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
    }
    for (int rep = 0; rep < 6; ++rep) {
      if (mode == 2) for (size_t i = 0; i < n; i += 512) host[i] = 0;  // CPU touches the pages between calls
      double t0 = now();
      copy_k<<<148 * 8, 256, 0, s>>>(host, dev, n);
      cudaError_t e = cudaStreamSynchronize(s);
      double t1 = now();
      double sum = 0; for (size_t i = 0; i < n; i += 4099) sum += host[i] - i * 0.5;
      std::printf("mode %d rep %d: D2H by kernel store %.3f ms (%.1f GB/s) %s check %g\n", mode, rep, (t1 - t0) * 1e3,
                  n * 8 / (t1 - t0) / 1e9, cudaGetErrorString(e), sum);
    }
  }
  // H2D: kernel reads pageable memory
  for (int rep = 0; rep < 4; ++rep) {
    double t0 = now();
    copy_k<<<148 * 8, 256, 0, s>>>(dev, host, n);
    cudaError_t e = cudaStreamSynchronize(s);
    double t1 = now();
    std::printf("H2D by kernel load %.3f ms (%.1f GB/s) %s\n", (t1 - t0) * 1e3, n * 8 / (t1 - t0) / 1e9, cudaGetErrorString(e));
  }
  // pinned reference
  double* pin; cudaMallocHost(&pin, n * 8);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    cudaMemcpyAsync(pin, dev, n * 8, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
    double t1 = now();
    std::printf("pinned cudaMemcpy D2H %.3f ms (%.1f GB/s)\n", (t1 - t0) * 1e3, n * 8 / (t1 - t0) / 1e9);
    t0 = now();
    copy_k<<<148 * 8, 256, 0, s>>>(pin, dev, n); cudaStreamSynchronize(s);
    t1 = now();
    std::printf("pinned kernel-store D2H %.3f ms (%.1f GB/s)\n", (t1 - t0) * 1e3, n * 8 / (t1 - t0) / 1e9);
  }
  return 0;
}
