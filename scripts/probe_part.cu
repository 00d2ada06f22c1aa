// Probe: cycles of one partitioned warp line solve (slabstep2d.cu part_solve_line) in isolation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2303_01163_b200/csrc -o probe_part scripts/probe_part.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "plan.hpp"
using namespace asdsm_b200;
template <int SEG>
__device__ __noinline__ void part_solve_line(double* line, const double* T, int n, int P, int last, double l,
                                                double r) {
  constexpr int M = SEG + 1;
  const int q = threadIdx.x & 31;
  const int R = P - 1;
  const bool full = q < P - 1;
  const int Li = full ? SEG : (q == P - 1 ? last : 0);
  const int base = q * M;
  double y[SEG];
#pragma unroll
  for (int t = 0; t < SEG; ++t) y[t] = t < Li ? line[base + t] : 0.0;
  const double fs = q < R ? line[base + M - 1] : 0.0;
  // pivots (shared, broadcast) are read straight into the chain: zero past the segment
  y[0] = y[0] * (Li > 0 ? T[0] : 0.0);
  double ylast = y[0];  // y of the segment's last row (static indices keep y in registers)
#pragma unroll
  for (int t = 1; t < SEG; ++t) {
    y[t] = (y[t] - l * y[t - 1]) * (t < Li ? T[t] : 0.0);
    if (t < Li) ylast = y[t];
  }
#pragma unroll
  for (int t = SEG - 2; t >= 0; --t) y[t] = y[t] - (r * (t < Li ? T[t] : 0.0)) * y[t + 1];
  const double ynext0 = __shfl_down_sync(0xffffffffu, y[0], 1);
  double rho = q < R ? fs - l * ylast - r * ynext0 : 0.0;
  double c1[5], c2[5];
#pragma unroll
  for (int lev = 0; lev < 5; ++lev) {
    c1[lev] = T[part_off_k1(SEG) + lev * 32 + q];
    c2[lev] = T[part_off_k2(SEG) + lev * 32 + q];
  }
#pragma unroll
  for (int lev = 0; lev < 5; ++lev) {
    const int s = 1 << lev;
    const double up = __shfl_up_sync(0xffffffffu, rho, s);
    const double dn = __shfl_down_sync(0xffffffffu, rho, s);
    if (q < R) {
      double v = rho;
      if (q - s >= 0) v = v - c1[lev] * up;
      if (q + s < R) v = v - c2[lev] * dn;
      rho = v;
    }
  }
  const double xs = q < R ? rho * T[part_off_ib(SEG) + q] : 0.0;

  double xl = __shfl_up_sync(0xffffffffu, xs, 1);
  if (q == 0) xl = 0.0;
  const double xr = full ? xs : 0.0;
  const double* g = T + (full ? part_off_g(SEG) : part_off_gl(SEG));
  const double* h = T + part_off_h(SEG);
#pragma unroll
  for (int t = 0; t < SEG; ++t) {  // all table reads before the first store (shared may alias)
    double v = y[t] - g[t] * xl;
    if (full) v = v - h[t] * xr;
    y[t] = v;
  }
#pragma unroll
  for (int t = 0; t < SEG; ++t)
    if (t < Li) line[base + t] = y[t];
  if (q < R) line[base + M - 1] = xs;
}


__global__ void probe(double* out, long long* cyc, int reps) {
  __shared__ double line[1056];
  __shared__ double T[4 * 32 + 352];
  for (int i = threadIdx.x; i < 1056; i += blockDim.x) line[i] = 1.0 + 1e-3 * i;
  for (int i = threadIdx.x; i < 4 * 32 + 352; i += blockDim.x) T[i] = 0.25 + 1e-4 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) part_solve_line<32>(line, T, 1029, 32, 6, -1.0, -1.0);
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  out[threadIdx.x] = line[threadIdx.x];
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1056 * 8); cudaMallocManaged(&cyc, 8);
  for (int k = 0; k < 3; ++k) { probe<<<1, 32>>>(out, cyc, 20); cudaDeviceSynchronize(); }
  printf("part_solve_line<32>: %lld cycles per line (1 warp, warm, 20 reps)\n", cyc[0]);
  probe<<<1, 32>>>(out, cyc, 1);
  cudaDeviceSynchronize();
  printf("part_solve_line<32>: %lld cycles (1 rep, after warm launches)\n", cyc[0]);
  double* junk; cudaMalloc(&junk, 256 << 20); cudaMemset(junk, 1, 256 << 20); cudaDeviceSynchronize();
  probe<<<1, 32>>>(out, cyc, 1);
  cudaDeviceSynchronize();
  printf("part_solve_line<32>: %lld cycles (1 rep, after a 256 MB L2 flush)\n", cyc[0]);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
