// Natural cubic spline through zero-clamped knots, bitwise the reference's CubicSpline
// (proj/src/spline.cpp:9-76): knots (0, c*n*h for c = 1..nc, 1), values (0, y_1..y_nc, 0).
#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

__device__ __forceinline__ double knot(const MeshDev& m, int axis, int c) {
  if (c == 0) return 0.0;
  if (c == m.nc[axis] + 1) return 1.0;
  return static_cast<double>(static_cast<i64>(c) * m.n[axis]) * m.h[axis];
}

// Natural cubic spline second derivatives through (0,0), (knot_c, v_c), (1,0)
// (zero_clamped_spline + CubicSpline ctor, spline.cpp:9-37, 58-76).  y has nc+2 entries.
__device__ inline void spline_second_derivs(const MeshDev& m, int axis, const double* y, double* mm, double* diag,
                                     double* upper, double* rhs) {
  const int n = m.nc[axis] + 2;
  for (int i = 0; i < n; ++i) mm[i] = 0.0;
  if (n == 2) return;
  const int ni = n - 2;
  for (int i = 0; i < ni; ++i) {
    const double x0 = knot(m, axis, i), x1 = knot(m, axis, i + 1), x2 = knot(m, axis, i + 2);
    const double hl = __dsub_rn(x1, x0);
    const double hr = __dsub_rn(x2, x1);
    diag[i] = __dadd_rn(hl, hr) / 3.0;
    upper[i] = hr / 6.0;
    rhs[i] = __dsub_rn(__dsub_rn(y[i + 2], y[i + 1]) / hr, __dsub_rn(y[i + 1], y[i]) / hl);
  }
  for (int i = 1; i < ni; ++i) {
    const double lower = __dsub_rn(knot(m, axis, i + 1), knot(m, axis, i)) / 6.0;
    const double w = lower / diag[i - 1];
    diag[i] = __dsub_rn(diag[i], __dmul_rn(w, upper[i - 1]));
    rhs[i] = __dsub_rn(rhs[i], __dmul_rn(w, rhs[i - 1]));
  }
  mm[ni] = rhs[ni - 1] / diag[ni - 1];
  for (int i = ni - 1; i >= 1; --i) mm[i] = __dsub_rn(rhs[i - 1], __dmul_rn(upper[i - 1], mm[i + 1])) / diag[i - 1];
}

// CubicSpline::operator() (spline.cpp:39-56) at fine index fi (1-based) along `axis` for a
// line whose knot values are y(c), c = 0..nc+1 (y(0) = y(nc+1) = 0), second derivatives mm.
template <typename Y>
__device__ __forceinline__ double spline_eval(const MeshDev& m, int axis, Y y, const double* mm, int fi) {
  const double x = static_cast<double>(fi) * m.h[axis];
  int i = fi / m.n[axis];
  if (i > m.nc[axis]) i = m.nc[axis];
  const double xi = knot(m, axis, i), xi1 = knot(m, axis, i + 1);
  const double y0 = y(i), y1 = y(i + 1), m0 = mm[i], m1 = mm[i + 1];
  const double h = __dsub_rn(xi1, xi);
  const double t = __dsub_rn(x, xi);
  const double c1 = __dsub_rn(__dsub_rn(y1, y0) / h, __dmul_rn(h, __dadd_rn(__dmul_rn(2.0, m0), m1)) / 6.0);
  const double c2 = m0 / 2.0;
  const double c3 = __dsub_rn(m1, m0) / __dmul_rn(6.0, h);
  return __dadd_rn(y0, __dmul_rn(t, __dadd_rn(c1, __dmul_rn(t, __dadd_rn(c2, __dmul_rn(t, c3))))));
}

// The per-interval coefficients spline_eval forms, (y_i, c1, c2, c3) for i = 0..nc, so that a
// line evaluated at many points pays the divisions once (bitwise the same values).  Tables are
// interval-major: interval i of a line sits at seg + i * ss (ss = 4 x the family's line count),
// so the lines of neighbouring points read neighbouring 32-byte entries.
template <typename Y>
__device__ inline void spline_segments(const MeshDev& m, int axis, Y y, const double* mm, double* seg, i64 ss) {
  const int nc = m.nc[axis];
  for (int i = 0; i <= nc; ++i) {
    const double xi = knot(m, axis, i), xi1 = knot(m, axis, i + 1);
    const double y0 = y(i), y1 = y(i + 1), m0 = mm[i], m1 = mm[i + 1];
    const double h = __dsub_rn(xi1, xi);
    seg[ss * i] = y0;
    seg[ss * i + 1] = __dsub_rn(__dsub_rn(y1, y0) / h, __dmul_rn(h, __dadd_rn(__dmul_rn(2.0, m0), m1)) / 6.0);
    seg[ss * i + 2] = m0 / 2.0;
    seg[ss * i + 3] = __dsub_rn(m1, m0) / __dmul_rn(6.0, h);
  }
}

// spline_eval from the segment table of the line
__device__ __forceinline__ double spline_eval_seg(const MeshDev& m, int axis, const double* __restrict__ seg, i64 ss,
                                                  int fi) {
  const double x = static_cast<double>(fi) * m.h[axis];
  int i = fi / m.n[axis];
  if (i > m.nc[axis]) i = m.nc[axis];
  const double t = __dsub_rn(x, knot(m, axis, i));
  const double4 c = *reinterpret_cast<const double4*>(seg + ss * i);
  return __dadd_rn(c.x, __dmul_rn(t, __dadd_rn(c.y, __dmul_rn(t, __dadd_rn(c.z, __dmul_rn(t, c.w))))));
}

}  // namespace asdsm_b200
