// Probe: cycles of one spline line (slabstep2d.cu spline_line) by one thread, in isolation.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kStepMaxNc = 24;
// One clamped-spline line (spline.cpp: zero-clamped natural spline through y[0..nc+1] with
// y[0] = y[nc+1] = 0), whole line in one thread: rhs, elimination, back substitution (the
// precomputed w / diag / upper terms; reciprocal multiplies), then the (y_c, c1, c2, c3)
// segments.  Compact loops (runtime nc) over a per-line shared scratch row.
__device__ __forceinline__ void spline_line(const double* y, int nc, const double* tab, const double* rr,
                                            double* seg, double* mm) {
  const int ni = nc, n = nc + 2;
  const double* w = tab + n + 2 * ni;
  const double* up = w + 2 * ni;
  double prev = 0.0;
  for (int i = 0; i < ni; ++i) {  // rhs and forward elimination in one pass (into mm[i + 1])
    double rhs = __dsub_rn(__dmul_rn(__dsub_rn(y[i + 2], y[i + 1]), rr[kStepMaxNc + i]),
                           __dmul_rn(__dsub_rn(y[i + 1], y[i]), rr[i]));
    if (i > 0) rhs = __dsub_rn(rhs, __dmul_rn(w[i], prev));
    mm[i + 1] = rhs;
    prev = rhs;
  }
  mm[0] = 0.0;
  mm[n - 1] = 0.0;
  if (ni > 0) {
    double nxt = __dmul_rn(mm[ni], rr[2 * kStepMaxNc + ni - 1]);
    mm[ni] = nxt;
    for (int i = ni - 1; i >= 1; --i) {
      nxt = __dmul_rn(__dsub_rn(mm[i], __dmul_rn(up[i - 1], nxt)), rr[2 * kStepMaxNc + i - 1]);
      mm[i] = nxt;
    }
  }
  for (int c = 0; c <= nc; ++c) {
    const double h = __dsub_rn(tab[c + 1], tab[c]);
    seg[4 * c + 0] = y[c];
    seg[4 * c + 1] = __dsub_rn(__dmul_rn(__dsub_rn(y[c + 1], y[c]), rr[3 * kStepMaxNc + c]),
                               __dmul_rn(__dmul_rn(h, __dadd_rn(__dmul_rn(2.0, mm[c]), mm[c + 1])), 1.0 / 6.0));
    seg[4 * c + 2] = __dmul_rn(mm[c], 0.5);
    seg[4 * c + 3] = __dmul_rn(__dsub_rn(mm[c + 1], mm[c]), rr[4 * kStepMaxNc + c]);
  }
}


__global__ void probe(double* out, long long* cyc, int reps) {
  __shared__ double y[32], mm[32], seg[128], tab[200], rr[200];
  for (int i = threadIdx.x; i < 200; i += blockDim.x) { tab[i] = 0.1 * i + 0.01; rr[i] = 1.0 + 0.001 * i; }
  for (int i = threadIdx.x; i < 32; i += blockDim.x) y[i] = 0.5 + 0.01 * i;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0)
    for (int r = 0; r < reps; ++r) spline_line(y, 9, tab, rr, seg, mm);
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  out[threadIdx.x] = seg[threadIdx.x];
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1056 * 8); cudaMallocManaged(&cyc, 8);
  for (int k = 0; k < 3; ++k) { probe<<<1, 32>>>(out, cyc, 20); cudaDeviceSynchronize(); }
  printf("spline_line nc=9: %lld cycles (warm, 20 reps)\n", cyc[0]);
  probe<<<1, 32>>>(out, cyc, 1); cudaDeviceSynchronize();
  printf("spline_line nc=9: %lld cycles (1 rep)\n", cyc[0]);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
