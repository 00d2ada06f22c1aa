// Dependent-chain latencies on B200 (one warp): DFMA, DMUL, LDS.64, and a DFMA+DMUL Thomas step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_latency scripts/probe_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double x = threadIdx.x * 1e-9 + 1.0, a = 0.999999, b = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * a;
  long long t2 = clock64();
  int idx = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < n; ++i) {
    double v = sm[idx];
    idx = (int)v & 1023;  // dependent address
    acc += v;
  }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = (b - a * x) * a;  // Thomas forward step (DFMA + DMUL)
  long long t4 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) {  // step with the pivot loaded from shared each time (independent)
    y = (b - a * y) * sm[(i * 8 + threadIdx.x) & 1023];
  }
  long long t5 = clock64();
  out[threadIdx.x] = x + acc + y;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8 * 8);
  const int n = 4096;
  for (int r = 0; r < 2; ++r) {
    lat_kernel<<<1, 32>>>(out, cyc, n);
    cudaDeviceSynchronize();
  }
  printf("DFMA chain %.2f cyc, DMUL chain %.2f, LDS dependent %.2f, thomas step %.2f, thomas+LDS %.2f\n",
         cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n, cyc[3] / (double)n, cyc[4] / (double)n);
  return 0;
}
