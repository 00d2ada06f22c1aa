// Launch-floor probe: device time per launch of near-empty kernels in a CUDA graph, to
// separate fixed per-kernel cost from work in the latency-bound config-1 iteration.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_launch scripts/probe_launch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 12345) p[0] = 1;
}
__global__ void smem_kernel(int* p) {
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && sm[(threadIdx.x + 1) % blockDim.x] < -1) p[0] = 1;
}
__global__ void stream_kernel(const double* __restrict__ a, double* __restrict__ b, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i] * 2.0;
}
__global__ void lastblock_kernel(unsigned* counter, double* part) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = blockIdx.x;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    double s = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += part[i];
    if (s < -1) part[0] = s;
    if (threadIdx.x == 0) *counter = 0;
  }
}

template <class F>
float graph_time(F launch, int reps) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < reps; ++i) launch(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1000.f / (5 * reps);
}

int main() {
  const int R = 200;
  int* p = nullptr;
  cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("empty <<<1,32>>>            %.2f us\n", graph_time([&](cudaStream_t s) { empty_kernel<<<1, 32, 0, s>>>(p); }, R));
  printf("empty <<<1323,128>>>        %.2f us\n", graph_time([&](cudaStream_t s) { empty_kernel<<<1323, 128, 0, s>>>(p); }, R));
  printf("empty <<<100,256>>>         %.2f us\n", graph_time([&](cudaStream_t s) { empty_kernel<<<100, 256, 0, s>>>(p); }, R));
  printf("smem183K <<<100,256>>>      %.2f us\n",
         graph_time([&](cudaStream_t s) { smem_kernel<<<100, 256, 183 * 1024, s>>>(p); }, R));
  printf("smem183K alternating empty  %.2f us (pair)\n", 2 * graph_time([&](cudaStream_t s) {
           static int k = 0;
           if (k++ & 1) smem_kernel<<<100, 256, 183 * 1024, s>>>(p);
           else empty_kernel<<<1323, 128, 0, s>>>(p);
         }, R));
  const long n = 1 << 20;
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  printf("stream 1M doubles (L2)      %.2f us\n",
         graph_time([&](cudaStream_t s) { stream_kernel<<<(n + 255) / 256, 256, 0, s>>>(a, b, n); }, R));
  unsigned* cnt;
  double* part;
  cudaMalloc(&cnt, 4);
  cudaMemset(cnt, 0, 4);
  cudaMalloc(&part, 65536 * 8);
  printf("lastblock <<<1323,128>>>    %.2f us\n",
         graph_time([&](cudaStream_t s) { lastblock_kernel<<<1323, 128, 0, s>>>(cnt, part); }, R));
  printf("lastblock <<<148,256>>>     %.2f us\n",
         graph_time([&](cudaStream_t s) { lastblock_kernel<<<148, 256, 0, s>>>(cnt, part); }, R));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
