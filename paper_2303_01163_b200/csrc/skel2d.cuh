// 2D skeleton fast path: cross values, corrections and spline segment coefficients
// (solver.cpp:166-187 with CubicSpline, spline.cpp:9-56) computed by ONE block, using the
// data-independent spline terms precomputed on the host.  Header-only so the slab
// back-transform's last block can run it right after the norms are known.
#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

constexpr int kSkelMaxKnots = 24;  // 2D fast path: coarse counts <= 22 (shared-memory staging)

// Spline tables of both axes staged in shared memory by the calling block (every access of
// the per-line recurrences would otherwise be an exposed L2 round trip).
constexpr int kSkelTabMax = 6 * kSkelMaxKnots;

// per-line: second derivatives via the pre-eliminated tridiagonal system, then per-segment
// (y_c, c1, c2, c3); y has nc+2 entries (y[0] = y[nc+1] = 0).
__device__ inline void skel_line_segments(const double* tab, int nc, const double* y, double* seg) {
  const int n = nc + 2, ni = nc;
  const double* x = tab;
  const double* hl = tab + n;
  const double* hr = hl + ni;
  const double* w = hr + ni;
  const double* dg = w + ni;
  const double* up = dg + ni;
  double rhs[kSkelMaxKnots], m[kSkelMaxKnots];
  for (int i = 0; i < n; ++i) m[i] = 0.0;
  for (int i = 0; i < ni; ++i) rhs[i] = __dsub_rn(__dsub_rn(y[i + 2], y[i + 1]) / hr[i], __dsub_rn(y[i + 1], y[i]) / hl[i]);
  for (int i = 1; i < ni; ++i) rhs[i] = __dsub_rn(rhs[i], __dmul_rn(w[i], rhs[i - 1]));
  if (ni > 0) {
    m[ni] = rhs[ni - 1] / dg[ni - 1];
    for (int i = ni - 1; i >= 1; --i) m[i] = __dsub_rn(rhs[i - 1], __dmul_rn(up[i - 1], m[i + 1])) / dg[i - 1];
  }
  for (int c = 0; c <= nc; ++c) {
    const double h = __dsub_rn(x[c + 1], x[c]);
    seg[4 * c + 0] = y[c];
    seg[4 * c + 1] = __dsub_rn(__dsub_rn(y[c + 1], y[c]) / h, __dmul_rn(h, __dadd_rn(__dmul_rn(2.0, m[c]), m[c + 1])) / 6.0);
    seg[4 * c + 2] = m[c] / 2.0;
    seg[4 * c + 3] = __dsub_rn(m[c + 1], m[c]) / __dmul_rn(6.0, h);
  }
}

// evaluation at fine index fi (1-based) along an axis with factor n: same as CubicSpline()
__device__ __forceinline__ double skel_seg_eval(const double* tab, const double* seg, int nc, int n, double hfine,
                                                int fi) {
  int c = fi / n;
  if (c > nc) c = nc;
  const double x = static_cast<double>(fi) * hfine;
  const double t = __dsub_rn(x, tab[c]);
  const double* s = seg + 4 * c;
  return __dadd_rn(s[0], __dmul_rn(t, __dadd_rn(s[1], __dmul_rn(t, __dadd_rn(s[2], __dmul_rn(t, s[3]))))));
}

// the whole cc + spline phase, executed by all threads of one block
__device__ inline void skel2d_ccspline_block(const Skel2DArgs& a) {
  const MeshDev& m = a.m;
  const int nc0 = m.nc[0], nc1 = m.nc[1];
  __shared__ double se1[kSkelMaxKnots * kSkelMaxKnots], se2[kSkelMaxKnots * kSkelMaxKnots];
  const bool in_smem = nc0 * nc1 <= kSkelMaxKnots * kSkelMaxKnots;
  const double nfc = a.norm_fc ? *a.norm_fc : 1.0;
  const double ncf = a.norm_cf ? *a.norm_cf : 1.0;
  __shared__ double stab[2][kSkelTabMax];
  const int tl0 = (nc0 + 2) + 5 * nc0, tl1 = (nc1 + 2) + 5 * nc1;
  for (int q = threadIdx.x; q < tl0; q += blockDim.x) cp_async8(&stab[0][q], a.sp_tab[0] + q);
  for (int q = threadIdx.x; q < tl1; q += blockDim.x) cp_async8(&stab[1][q], a.sp_tab[1] + q);
  cp_async_wait_all();
  for (int t = threadIdx.x; t < nc0 * nc1; t += blockDim.x) {
    const int I = t % nc0, J = t / nc0;
    double u1 = a.u_fc[static_cast<i64>((I + 1) * m.n[0] - 1) + static_cast<i64>(m.nf[0]) * J];
    double u2 = a.u_cf[I + static_cast<i64>(nc0) * ((J + 1) * m.n[1] - 1)];
    if (a.norm_fc) {
      u1 = u1 / nfc;
      u2 = u2 / ncf;
    }
    double uh;
    if (a.u_cc) uh = __dsub_rn(__dadd_rn(u1, u2), a.u_cc[t]);
    else uh = (a.coin[0] == 0) ? u2 : u1;
    const double d1 = __dsub_rn(uh, u1), d2 = __dsub_rn(uh, u2);
    a.e1[t] = d1;
    a.e2[t] = d2;
    if (in_smem) {
      se1[t] = d1;
      se2[t] = d2;
    }
  }
  __syncthreads();
  const double* E1 = in_smem ? se1 : a.e1;
  const double* E2 = in_smem ? se2 : a.e2;
  // Phase 2, split so only the two short recurrences per line are sequential:
  //  2a one thread per (line, i): rhs_i = (y[i+2]-y[i+1])/hr_i - (y[i+1]-y[i])/hl_i
  //  2b one thread per line: forward elimination and back substitution (spline.cpp:29-36)
  //  2c one thread per (line, segment): (y_c, c1, c2, c3) (spline.cpp:47-55)
  constexpr int KM = kSkelMaxKnots;
  __shared__ double srhs[2 * KM][KM];  // [line][i]   (lines: nc1 along x, then nc0 along y)
  __shared__ double smm[2 * KM][KM];   // [line][c]   second derivatives
  const int nlines = nc0 + nc1;
  auto yval = [&](int line, int c) -> double {  // y[c], c = 0..nc+1
    if (line < nc1) return (c == 0 || c == nc0 + 1) ? 0.0 : E1[(c - 1) + static_cast<i64>(nc0) * line];
    const int I = line - nc1;
    return (c == 0 || c == nc1 + 1) ? 0.0 : E2[I + static_cast<i64>(nc0) * (c - 1)];
  };
  for (int t = threadIdx.x; t < nc1 * nc0 + nc0 * nc1; t += blockDim.x) {
    const int line = t < nc1 * nc0 ? t / nc0 : nc1 + (t - nc1 * nc0) / nc1;
    const int nc = line < nc1 ? nc0 : nc1;
    const int i = t < nc1 * nc0 ? t % nc0 : (t - nc1 * nc0) % nc1;
    const double* tab = stab[line < nc1 ? 0 : 1];
    const double* hl = tab + nc + 2;
    const double* hr = hl + nc;
    srhs[line][i] = __dsub_rn(__dsub_rn(yval(line, i + 2), yval(line, i + 1)) / hr[i],
                              __dsub_rn(yval(line, i + 1), yval(line, i)) / hl[i]);
  }
  __syncthreads();
  for (int line = threadIdx.x; line < nlines; line += blockDim.x) {
    const int nc = line < nc1 ? nc0 : nc1, ni = nc, n = nc + 2;
    const double* tab = stab[line < nc1 ? 0 : 1];
    const double* w = tab + n + 2 * ni;
    const double* dg = w + ni;
    const double* up = dg + ni;
    double* rhs = srhs[line];
    double* m = smm[line];
    for (int i = 1; i < ni; ++i) rhs[i] = __dsub_rn(rhs[i], __dmul_rn(w[i], rhs[i - 1]));
    m[0] = 0.0;
    m[n - 1] = 0.0;
    if (ni > 0) {
      m[ni] = rhs[ni - 1] / dg[ni - 1];
      for (int i = ni - 1; i >= 1; --i) m[i] = __dsub_rn(rhs[i - 1], __dmul_rn(up[i - 1], m[i + 1])) / dg[i - 1];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nc1 * (nc0 + 1) + nc0 * (nc1 + 1); t += blockDim.x) {
    int line, c;
    if (t < nc1 * (nc0 + 1)) {
      line = t / (nc0 + 1);
      c = t % (nc0 + 1);
    } else {
      line = nc1 + (t - nc1 * (nc0 + 1)) / (nc1 + 1);
      c = (t - nc1 * (nc0 + 1)) % (nc1 + 1);
    }
    const double* x = stab[line < nc1 ? 0 : 1];
    const double* m = smm[line];
    const double y0 = yval(line, c), y1 = yval(line, c + 1);
    const double h = __dsub_rn(x[c + 1], x[c]);
    double* seg = line < nc1 ? a.seg1 + static_cast<i64>(line) * 4 * (nc0 + 1) + 4 * c
                             : a.seg2 + static_cast<i64>(line - nc1) * 4 * (nc1 + 1) + 4 * c;
    seg[0] = y0;
    seg[1] = __dsub_rn(__dsub_rn(y1, y0) / h, __dmul_rn(h, __dadd_rn(__dmul_rn(2.0, m[c]), m[c + 1])) / 6.0);
    seg[2] = m[c] / 2.0;
    seg[3] = __dsub_rn(m[c + 1], m[c]) / __dmul_rn(6.0, h);
  }
}

}  // namespace asdsm_b200
