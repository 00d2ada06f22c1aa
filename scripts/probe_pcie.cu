// PCIe probe for the e2e path: pinned cudaMemcpyAsync H2D / D2H rates at the config-1 byte
// counts (one stream, split streams), and SM-driven zero-copy stores into mapped pinned memory.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void zc_store(const double2* __restrict__ src, double2* dst, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void zc_load(const double2* src, double2* __restrict__ dst, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  const long n = 1058841L * 2;  // u + r
  const size_t by = n * 8;
  double *h, *h2, *d, *d2;
  CK(cudaHostAlloc((void**)&h, by, cudaHostAllocMapped));
  CK(cudaHostAlloc((void**)&h2, by, cudaHostAllocMapped));
  CK(cudaMalloc((void**)&d, by));
  CK(cudaMalloc((void**)&d2, by));
  cudaMemset(d, 0, by);
  cudaStream_t s, s1;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaEvent_t a, b, f;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&f);
  auto tm = [&](auto fn, const char* name, size_t bytes) {
    fn(); cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int r = 0; r < 20; ++r) fn();
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
    printf("%-40s %8.1f us %7.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  for (size_t sz : {by / 2, by}) {
    char nm[64];
    snprintf(nm, 64, "D2H memcpy %.1f MB", sz / 1e6); tm([&] { cudaMemcpyAsync(h, d, sz, cudaMemcpyDeviceToHost, s); }, nm, sz);
    snprintf(nm, 64, "H2D memcpy %.1f MB", sz / 1e6); tm([&] { cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s); }, nm, sz);
  }
  tm([&] {
    cudaEventRecord(f, s); cudaStreamWaitEvent(s1, f, 0);
    cudaMemcpyAsync(h, d, by / 2, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h2, d + n / 2, by / 2, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(f, s1); cudaStreamWaitEvent(s, f, 0);
  }, "D2H 2 streams (u || r)", by);
  tm([&] {
    cudaEventRecord(f, s); cudaStreamWaitEvent(s1, f, 0);
    cudaMemcpyAsync(d, h, by / 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(h2, d2, by / 2, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(f, s1); cudaStreamWaitEvent(s, f, 0);
  }, "H2D 8.5MB || D2H 17MB", by / 4 + by / 2);
  double* hd; CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  for (int grid : {148, 296, 592, 1184}) {
    char nm[64];
    snprintf(nm, 64, "zero-copy store grid %d", grid);
    tm([&] { zc_store<<<grid, 256, 0, s>>>((const double2*)d, (double2*)hd, n / 2); }, nm, by);
    snprintf(nm, 64, "zero-copy load grid %d", grid);
    tm([&] { zc_load<<<grid, 256, 0, s>>>((const double2*)hd, (double2*)d, n / 2); }, nm, by);
  }
  return 0;
}
