// Warp-partitioned tridiagonal line solve (SepSolver::part tables, plan.cpp
// build_partition_tables): every lane Thomas-eliminates a segment of SEG rows in registers, the
// separators form a tridiagonal system solved by a 5-level shuffle PCR, and every lane
// reconstructs its segment from the two separator values.  Shared by the 2D slab step
// (slabstep2d.cu) and the generic separable line solve (sepsolve.cu).
#pragma once
#include "plan.hpp"

namespace asdsm_b200 {

// One line of mode space (length n, in shared memory, in place) by one warp; T = this mode's
// SepSolver::part table (in shared memory).  Every lane runs exactly SEG steps: rows past its
// segment have pivot 0, so they stay 0 and decouple.
template <int SEG>
__device__ __forceinline__ void part_solve_line(double* line, const double* T, int n, int P, int last, double l,
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

}  // namespace asdsm_b200
