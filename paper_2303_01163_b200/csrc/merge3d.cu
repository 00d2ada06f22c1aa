// 3D skeleton merge (merge_3d, proj/src/solver.cpp:297-410) on the device.
//
// Inputs: the three slab solutions u[a] (kind coarse along a), optional coarse solution
// u_ccc (smooth mode) or the seeded draws (error mode).  Stages, each a data-parallel
// kernel over the lines / points it touches:
//   M1 triple level: s_a = P(slab a -> triple) u[a], u_hat, per-pair corr = u_hat - base_t
//   M2 pair targets T_ab on the pair kinds: base + spline_f(corr), pinned to u_hat at stations
//   M3 per-plane Boolean-sum corrections of every slab (correct_slab_plane, solver.cpp:204-293)
//   M4 inclusion-exclusion scatter onto the fine skeleton points, in the reference's
//      scatter_add order (slabs 0,1,2; -T01, -T02, -T12; +u_hat).
// All arithmetic is non-contracted and ordered as in the reference.
#include "merge3d.cuh"
#include "spline.cuh"

#include <algorithm>

namespace asdsm_b200 {

namespace {

constexpr int kMaxKnots = 64;

struct Ext3 {
  int e[3];
  __device__ __forceinline__ i64 lin(int i0, int i1, int i2) const {
    return i0 + static_cast<i64>(e[0]) * (i1 + static_cast<i64>(e[1]) * i2);
  }
};

__device__ __forceinline__ Ext3 kind_ext(const MeshDev& m, unsigned mask) {
  Ext3 x;
  for (int a = 0; a < 3; ++a) x.e[a] = ((mask >> a) & 1u) ? m.nc[a] : m.nf[a];
  return x;
}

__device__ __forceinline__ int station(const MeshDev& m, int a, int c) { return (c + 1) * m.n[a] - 1; }

__device__ __forceinline__ int pair_slot(int a, int b) { return (a < b ? a : b) + (a < b ? b : a) - 1; }

// value of slab a at a point given by per-axis indices in each axis' own space of slab a
__device__ __forceinline__ double slab_val(const Merge3DArgs& A, int a, int i0, int i1, int i2) {
  return A.u[a][kind_ext(A.m, 1u << a).lin(i0, i1, i2)];
}

// ---- M1 ----------------------------------------------------------------------------------
__global__ void m1_kernel(Merge3DArgs A, const DevState* st) {
  if (!st->active || !st->have_e) return;
  const MeshDev& m = A.m;
  const int n = m.nc[0] * m.nc[1] * m.nc[2];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int c0 = t % m.nc[0], c1 = (t / m.nc[0]) % m.nc[1], c2 = t / (m.nc[0] * m.nc[1]);
  const int f0 = station(m, 0, c0), f1 = station(m, 1, c1), f2 = station(m, 2, c2);
  double s[3];
  s[0] = slab_val(A, 0, c0, f1, f2);
  s[1] = slab_val(A, 1, f0, c1, f2);
  s[2] = slab_val(A, 2, f0, f1, c2);
  double uh;
  if (A.u_ccc) {
    uh = __dsub_rn(__dadd_rn(__dadd_rn(s[0], s[1]), s[2]), A.u_ccc[t]) / 2.0;
  } else {
    uh = s[A.coin[0]];
  }
  A.u_hat[t] = uh;
  int p = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b, ++p) {
      double bt;
      if (A.u_ccc) bt = __dadd_rn(s[a], s[b]) / 2.0;
      else bt = A.coin[1 + p] ? s[b] : s[a];
      A.corr[p][t] = __dsub_rn(uh, bt);
    }
}

// ---- M2 ----------------------------------------------------------------------------------
// pair p = (a,b), free fine axis f; line (ca, cb): spline along f through corr(ca, cb, :).
__device__ __forceinline__ void pair_axes(int p, int& a, int& b, int& f) {
  a = p < 2 ? 0 : 1;
  b = p == 0 ? 1 : 2;
  f = 3 - a - b;
}

__global__ void m2_derivs_kernel(Merge3DArgs A, const DevState* st) {
  if (!st->active || !st->have_e) return;
  const MeshDev& m = A.m;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int base = 0;
  for (int p = 0; p < 3; ++p) {
    int a, b, f;
    pair_axes(p, a, b, f);
    const int nl = m.nc[a] * m.nc[b];
    if (t < base + nl) {
      const int l = t - base;
      const int ca = l % m.nc[a], cb = l / m.nc[a];
      double y[kMaxKnots], dg[kMaxKnots], up[kMaxKnots], rh[kMaxKnots];
      const int nc = m.nc[f];
      y[0] = 0.0;
      y[nc + 1] = 0.0;
      for (int c = 0; c < nc; ++c) {
        int idx[3];
        idx[a] = ca;
        idx[b] = cb;
        idx[f] = c;
        y[c + 1] = A.corr[p][idx[0] + static_cast<i64>(m.nc[0]) * (idx[1] + static_cast<i64>(m.nc[1]) * idx[2])];
      }
      spline_second_derivs(m, f, y, A.mP[p] + static_cast<i64>(l) * (nc + 2), dg, up, rh);
      return;
    }
    base += nl;
  }
}

__global__ void m2_fill_kernel(Merge3DArgs A, const DevState* st) {
  if (!st->active || !st->have_e) return;
  const MeshDev& m = A.m;
  i64 total = 0;
  for (int p = 0; p < 3; ++p) {
    int a, b, f;
    pair_axes(p, a, b, f);
    total += static_cast<i64>(m.nc[a]) * m.nc[b] * m.nf[f];
  }
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 r = t;
    int p = 0, a = 0, b = 1, f = 2;
    for (p = 0; p < 3; ++p) {
      pair_axes(p, a, b, f);
      const i64 np = static_cast<i64>(m.nc[a]) * m.nc[b] * m.nf[f];
      if (r < np) break;
      r -= np;
    }
    const unsigned pmask = (1u << a) | (1u << b);
    const Ext3 pe = kind_ext(m, pmask);
    int idx[3];
    idx[0] = static_cast<int>(r % pe.e[0]);
    idx[1] = static_cast<int>((r / pe.e[0]) % pe.e[1]);
    idx[2] = static_cast<int>(r / (static_cast<i64>(pe.e[0]) * pe.e[1]));
    const int ca = idx[a], cb = idx[b], k = idx[f];
    // projections of slab a and slab b onto the pair kind
    int ia[3], ib[3];
    ia[a] = ca; ia[b] = station(m, b, cb); ia[f] = k;
    ib[a] = station(m, a, ca); ib[b] = cb; ib[f] = k;
    const double ua = slab_val(A, a, ia[0], ia[1], ia[2]);
    const double ub = slab_val(A, b, ib[0], ib[1], ib[2]);
    double base;
    if (A.u_ccc) base = __dadd_rn(ua, ub) / 2.0;
    else base = A.coin[1 + p] ? ub : ua;
    const int nc = m.nc[f];
    const int l = ca + m.nc[a] * cb;
    const double* mm = A.mP[p] + static_cast<i64>(l) * (nc + 2);
    auto yv = [&](int c) -> double {
      if (c == 0 || c == nc + 1) return 0.0;
      int q[3];
      q[a] = ca; q[b] = cb; q[f] = c - 1;
      return A.corr[p][q[0] + static_cast<i64>(m.nc[0]) * (q[1] + static_cast<i64>(m.nc[1]) * q[2])];
    };
    double v = __dadd_rn(base, spline_eval(m, f, yv, mm, k + 1));
    if ((k + 1) % m.n[f] == 0) {
      int q[3];
      q[a] = ca; q[b] = cb; q[f] = (k + 1) / m.n[f] - 1;
      v = A.u_hat[q[0] + static_cast<i64>(m.nc[0]) * (q[1] + static_cast<i64>(m.nc[1]) * q[2])];
    }
    A.T[p][pe.lin(idx[0], idx[1], idx[2])] = v;
  }
}

// ---- M3 ----------------------------------------------------------------------------------
__device__ __forceinline__ void slab_axes(int a, int& f1, int& f2) {
  f1 = (a == 0) ? 1 : 0;
  f2 = (a == 2) ? 1 : 2;
}

// helpers reading T1 / T2 / u_hat / slab at (a: I, f1: i1, f2: i2) with each index in the
// axis space of the respective kind
__device__ __forceinline__ double at3(const double* arr, const Ext3& e, int a, int f1, int f2, int I, int i1, int i2) {
  int q[3];
  q[a] = I; q[f1] = i1; q[f2] = i2;
  return arr[e.lin(q[0], q[1], q[2])];
}

struct PlaneCtx {
  int a, f1, f2;
  Ext3 se, t1e, t2e, he;
  const double* slab;
  const double* T1;
  const double* T2;
};

__device__ __forceinline__ PlaneCtx plane_ctx(const Merge3DArgs& A, int a) {
  PlaneCtx c;
  c.a = a;
  slab_axes(a, c.f1, c.f2);
  c.se = kind_ext(A.m, 1u << a);
  c.t1e = kind_ext(A.m, (1u << a) | (1u << c.f1));
  c.t2e = kind_ext(A.m, (1u << a) | (1u << c.f2));
  c.he = kind_ext(A.m, 7u);
  c.slab = A.u[a];
  c.T1 = A.T[pair_slot(a, c.f1)];
  c.T2 = A.T[pair_slot(a, c.f2)];
  return c;
}

// family y-values (solver.cpp:239-242, 253-256, 268-271)
__device__ __forceinline__ double fam1_y(const MeshDev& m, const PlaneCtx& c, int I, int k2, int C1) {
  return __dsub_rn(at3(c.T1, c.t1e, c.a, c.f1, c.f2, I, C1, k2), at3(c.slab, c.se, c.a, c.f1, c.f2, I, station(m, c.f1, C1), k2));
}
__device__ __forceinline__ double fam2_y(const MeshDev& m, const PlaneCtx& c, int I, int k1, int C2) {
  return __dsub_rn(at3(c.T2, c.t2e, c.a, c.f1, c.f2, I, k1, C2), at3(c.slab, c.se, c.a, c.f1, c.f2, I, k1, station(m, c.f2, C2)));
}
__device__ __forceinline__ double fam3_y(const Merge3DArgs& A, const PlaneCtx& c, int I, int C2, int C1) {
  return __dsub_rn(at3(A.u_hat, c.he, c.a, c.f1, c.f2, I, C1, C2),
                   at3(c.slab, c.se, c.a, c.f1, c.f2, I, station(A.m, c.f1, C1), station(A.m, c.f2, C2)));
}

// Line families per slab a (offsets in Merge3DArgs):
//   fam1: (I, k2) along f1, nc_f1 knots     fam2: (I, k1) along f2, nc_f2 knots
//   fam3a: (I, C2) along f1                 fam3b: (I, k1) along f2 through g(I, k1, :)
__global__ void m3_derivs_kernel(Merge3DArgs A, int stage, const DevState* st) {
  if (!st->active || !st->have_e) return;
  const int a = blockIdx.y;  // slab
  const MeshDev& m = A.m;
  const PlaneCtx c = plane_ctx(A, a);
  const int ncA = m.nc[a], nc1 = m.nc[c.f1], nc2 = m.nc[c.f2], nf1 = m.nf[c.f1], nf2 = m.nf[c.f2];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double y[kMaxKnots], dg[kMaxKnots], up[kMaxKnots], rh[kMaxKnots];
  auto yl = [&](int q) { return y[q]; };
  if (stage == 0) {
    const int n1 = ncA * nf2, n2 = ncA * nf1, n3 = ncA * nc2;
    if (t < n1) {
      const int I = t % ncA, k2 = t / ncA;
      y[0] = 0.0;
      y[nc1 + 1] = 0.0;
      for (int C = 0; C < nc1; ++C) y[C + 1] = fam1_y(m, c, I, k2, C);
      double* mm = A.mF1[a] + static_cast<i64>(t) * (nc1 + 2);
      spline_second_derivs(m, c.f1, y, mm, dg, up, rh);
      spline_segments(m, c.f1, yl, mm, A.sF1[a] + 4 * static_cast<i64>(t), 4 * static_cast<i64>(n1));
    } else if (t < n1 + n2) {
      const int l = t - n1;
      const int I = l % ncA, k1 = l / ncA;
      y[0] = 0.0;
      y[nc2 + 1] = 0.0;
      for (int C = 0; C < nc2; ++C) y[C + 1] = fam2_y(m, c, I, k1, C);
      double* mm = A.mF2[a] + static_cast<i64>(l) * (nc2 + 2);
      spline_second_derivs(m, c.f2, y, mm, dg, up, rh);
      spline_segments(m, c.f2, yl, mm, A.sF2[a] + 4 * static_cast<i64>(l), 4 * static_cast<i64>(n2));
    } else if (t < n1 + n2 + n3) {
      const int l = t - n1 - n2;
      const int I = l % ncA, C2 = l / ncA;
      y[0] = 0.0;
      y[nc1 + 1] = 0.0;
      for (int C = 0; C < nc1; ++C) y[C + 1] = fam3_y(A, c, I, C2, C);
      double* mm = A.mF3a[a] + static_cast<i64>(l) * (nc1 + 2);
      spline_second_derivs(m, c.f1, y, mm, dg, up, rh);
      spline_segments(m, c.f1, yl, mm, A.sF3a[a] + 4 * static_cast<i64>(l), 4 * static_cast<i64>(n3));
    }
  } else {
    // fam3b: (I, k1), y = g(I, k1, C2) = fam3a spline (I, C2) at k1
    const int n = ncA * nf1;
    if (t >= n) return;
    const int I = t % ncA, k1 = t / ncA;
    y[0] = 0.0;
    y[nc2 + 1] = 0.0;
    for (int C2 = 0; C2 < nc2; ++C2)
      y[C2 + 1] = spline_eval_seg(m, c.f1, A.sF3a[a] + 4 * static_cast<i64>(I + ncA * C2), 4 * static_cast<i64>(ncA) * nc2, k1 + 1);
    double* mm = A.mF3b[a] + static_cast<i64>(t) * (nc2 + 2);
    spline_second_derivs(m, c.f2, y, mm, dg, up, rh);
    spline_segments(m, c.f2, yl, mm, A.sF3b[a] + 4 * static_cast<i64>(t), 4 * static_cast<i64>(n));
  }
  (void)nf2;
}

// The same splines one warp per line (nc <= 30 knots per line): lanes load the knot values and
// form the right-hand sides and the segment coefficients in parallel, lane 0 runs the short
// Thomas chain; the working arrays live in shared memory (the thread-per-line kernel above keeps
// them in local memory, one dependent local access per step).  Same operations in the same order
// as spline_second_derivs / spline_segments: bitwise the same tables.
constexpr int kDerivWarps = 4;
constexpr int kWarpKnots = 32;

__device__ __forceinline__ void spline_warp(const MeshDev& m, int axis, double* ys, double* dg, double* up, double* rh,
                                            double* mmS, double* mm, double* seg, i64 ss) {
  const int lane = threadIdx.x & 31;
  const int nc = m.nc[axis], n = nc + 2, ni = n - 2;
  __syncwarp();
  if (lane < ni) {  // spline_second_derivs: rhs, diag, upper of row i
    const int i = lane;
    const double x0 = knot(m, axis, i), x1 = knot(m, axis, i + 1), x2 = knot(m, axis, i + 2);
    const double hl = __dsub_rn(x1, x0);
    const double hr = __dsub_rn(x2, x1);
    dg[i] = __dadd_rn(hl, hr) / 3.0;
    up[i] = hr / 6.0;
    rh[i] = __dsub_rn(__dsub_rn(ys[i + 2], ys[i + 1]) / hr, __dsub_rn(ys[i + 1], ys[i]) / hl);
  }
  if (lane < n) mmS[lane] = 0.0;
  __syncwarp();
  if (lane == 0 && ni > 0) {
    for (int i = 1; i < ni; ++i) {
      const double lower = __dsub_rn(knot(m, axis, i + 1), knot(m, axis, i)) / 6.0;
      const double w = lower / dg[i - 1];
      dg[i] = __dsub_rn(dg[i], __dmul_rn(w, up[i - 1]));
      rh[i] = __dsub_rn(rh[i], __dmul_rn(w, rh[i - 1]));
    }
    mmS[ni] = rh[ni - 1] / dg[ni - 1];
    for (int i = ni - 1; i >= 1; --i) mmS[i] = __dsub_rn(rh[i - 1], __dmul_rn(up[i - 1], mmS[i + 1])) / dg[i - 1];
  }
  __syncwarp();
  if (lane < n) mm[lane] = mmS[lane];
  if (lane <= nc) {  // spline_segments: interval i
    const int i = lane;
    const double xi = knot(m, axis, i), xi1 = knot(m, axis, i + 1);
    const double y0 = ys[i], y1 = ys[i + 1], m0 = mmS[i], m1 = mmS[i + 1];
    const double h = __dsub_rn(xi1, xi);
    double4 c;
    c.x = y0;
    c.y = __dsub_rn(__dsub_rn(y1, y0) / h, __dmul_rn(h, __dadd_rn(__dmul_rn(2.0, m0), m1)) / 6.0);
    c.z = m0 / 2.0;
    c.w = __dsub_rn(m1, m0) / __dmul_rn(6.0, h);
    *reinterpret_cast<double4*>(seg + ss * i) = c;
  }
}

__global__ void __launch_bounds__(32 * kDerivWarps) m3_derivs_warp_kernel(Merge3DArgs A, int stage, const DevState* st) {
  if (!st->active || !st->have_e) return;
  __shared__ double sh[kDerivWarps][5][kWarpKnots + 2];
  const int a = blockIdx.y;  // slab
  const MeshDev& m = A.m;
  const PlaneCtx c = plane_ctx(A, a);
  const int ncA = m.nc[a], nc1 = m.nc[c.f1], nc2 = m.nc[c.f2], nf1 = m.nf[c.f1], nf2 = m.nf[c.f2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * kDerivWarps + warp;
  double* ys = sh[warp][0];
  double* dg = sh[warp][1];
  double* up = sh[warp][2];
  double* rh = sh[warp][3];
  double* mmS = sh[warp][4];
  if (stage == 0) {
    const int n1 = ncA * nf2, n2 = ncA * nf1, n3 = ncA * nc2;
    if (t < n1) {
      const int I = t % ncA, k2 = t / ncA;
      if (lane < nc1 + 2) ys[lane] = (lane == 0 || lane == nc1 + 1) ? 0.0 : fam1_y(m, c, I, k2, lane - 1);
      spline_warp(m, c.f1, ys, dg, up, rh, mmS, A.mF1[a] + static_cast<i64>(t) * (nc1 + 2),
                  A.sF1[a] + 4 * static_cast<i64>(t), 4 * static_cast<i64>(n1));
    } else if (t < n1 + n2) {
      const int l = t - n1;
      const int I = l % ncA, k1 = l / ncA;
      if (lane < nc2 + 2) ys[lane] = (lane == 0 || lane == nc2 + 1) ? 0.0 : fam2_y(m, c, I, k1, lane - 1);
      spline_warp(m, c.f2, ys, dg, up, rh, mmS, A.mF2[a] + static_cast<i64>(l) * (nc2 + 2),
                  A.sF2[a] + 4 * static_cast<i64>(l), 4 * static_cast<i64>(n2));
    } else if (t < n1 + n2 + n3) {
      const int l = t - n1 - n2;
      const int I = l % ncA, C2 = l / ncA;
      if (lane < nc1 + 2) ys[lane] = (lane == 0 || lane == nc1 + 1) ? 0.0 : fam3_y(A, c, I, C2, lane - 1);
      spline_warp(m, c.f1, ys, dg, up, rh, mmS, A.mF3a[a] + static_cast<i64>(l) * (nc1 + 2),
                  A.sF3a[a] + 4 * static_cast<i64>(l), 4 * static_cast<i64>(n3));
    }
  } else {
    const int n = ncA * nf1;
    if (t >= n) return;
    const int I = t % ncA, k1 = t / ncA;
    if (lane < nc2 + 2)
      ys[lane] = (lane == 0 || lane == nc2 + 1)
                     ? 0.0
                     : spline_eval_seg(m, c.f1, A.sF3a[a] + 4 * static_cast<i64>(I + ncA * (lane - 1)),
                                       4 * static_cast<i64>(ncA) * nc2, k1 + 1);
    spline_warp(m, c.f2, ys, dg, up, rh, mmS, A.mF3b[a] + static_cast<i64>(t) * (nc2 + 2),
                A.sF3b[a] + 4 * static_cast<i64>(t), 4 * static_cast<i64>(n));
  }
  (void)nf2;
}

// corrected slab a = slab + ((s1 + s2) - s3) at every slab point (solver.cpp:289-292), each
// spline from its line's segment table
__global__ void m3_apply_kernel(Merge3DArgs A, const DevState* st) {
  if (!st->active || !st->have_e) return;
  const int a = blockIdx.y;  // slab
  const MeshDev& m = A.m;
  const PlaneCtx c = plane_ctx(A, a);
  const int ncA = m.nc[a];
  const unsigned e0 = c.se.e[0], e1 = c.se.e[1];
  const unsigned total = e0 * e1 * static_cast<unsigned>(c.se.e[2]);  // < 2^31: checked at launch
  const i64 ss1 = 4 * static_cast<i64>(ncA) * m.nf[c.f2], ss2 = 4 * static_cast<i64>(ncA) * m.nf[c.f1];
  const double* __restrict__ slab = c.slab;
  double* __restrict__ outp = A.corrected[a];
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    int q[3];
    const unsigned r = t / e0;
    q[0] = static_cast<int>(t - r * e0);
    q[2] = static_cast<int>(r / e1);
    q[1] = static_cast<int>(r - static_cast<unsigned>(q[2]) * e1);
    const int I = q[a], k1 = q[c.f1], k2 = q[c.f2];
    const double s1 = spline_eval_seg(m, c.f1, A.sF1[a] + 4 * static_cast<i64>(I + ncA * k2), ss1, k1 + 1);
    const double s2 = spline_eval_seg(m, c.f2, A.sF2[a] + 4 * static_cast<i64>(I + ncA * k1), ss2, k2 + 1);
    const double s3 = spline_eval_seg(m, c.f2, A.sF3b[a] + 4 * static_cast<i64>(I + ncA * k1), ss2, k2 + 1);
    outp[t] = __dadd_rn(slab[t], __dsub_rn(__dadd_rn(s1, s2), s3));
  }
}

// ---- M4 ----------------------------------------------------------------------------------
// Skeleton points only, enumerated plane family by plane family without duplicates:
// family 0: x-coarse planes (all y, z); family 1: y-coarse planes with x not coarse;
// family 2: z-coarse planes with x, y not coarse.
__global__ void m4_kernel(Merge3DArgs A, double* out, const DevState* st) {
  if (!st->active || !st->have_e) return;
  const MeshDev& m = A.m;
  const i64 nf0 = m.nf[0], nf1 = m.nf[1];
  // 32-bit point counts (checked at launch): 64-bit divisions were the kernel's cost
  const unsigned unf1 = m.nf[1], unf2 = m.nf[2], nc0 = m.nc[0], nc1 = m.nc[1], nc2 = m.nc[2];
  const unsigned fx = m.nf[0] - m.nc[0], fy = m.nf[1] - m.nc[1];  // non-coarse counts per axis
  const unsigned n0 = nc0 * unf1 * unf2;
  const unsigned n1 = fx * nc1 * unf2;
  const unsigned n2 = fx * fy * nc2;
  const unsigned s0 = m.n[0] - 1, s1 = m.n[1] - 1;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n0 + n1 + n2; t += gridDim.x * blockDim.x) {
    int f[3];
    if (t < n0) {
      const unsigned q = t, r = q / nc0, z = r / unf1;
      f[0] = static_cast<int>((q - r * nc0 + 1) * m.n[0] - 1);
      f[1] = static_cast<int>(r - z * unf1);
      f[2] = static_cast<int>(z);
    } else if (t < n0 + n1) {
      const unsigned q = t - n0, r = q / fx, z = r / nc1, x = q - r * fx;
      f[0] = static_cast<int>(x + x / s0);  // x-th non-coarse fine index
      f[1] = static_cast<int>((r - z * nc1 + 1) * m.n[1] - 1);
      f[2] = static_cast<int>(z);
    } else {
      const unsigned q = t - n0 - n1, r = q / fx, c = r / fy, x = q - r * fx, y = r - c * fy;
      f[0] = static_cast<int>(x + x / s0);
      f[1] = static_cast<int>(y + y / s1);
      f[2] = static_cast<int>((c + 1) * m.n[2] - 1);
    }
    bool on[3];
    int cc[3];
    int non = 0;
    for (int a = 0; a < 3; ++a) {
      on[a] = (f[a] + 1) % m.n[a] == 0;
      cc[a] = (f[a] + 1) / m.n[a] - 1;
      non += on[a];
    }
    double v = 0.0;
    for (int a = 0; a < 3; ++a) {
      if (!on[a]) continue;
      int q[3] = {f[0], f[1], f[2]};
      q[a] = cc[a];
      v = __dadd_rn(v, A.corrected[a][kind_ext(m, 1u << a).lin(q[0], q[1], q[2])]);
    }
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b) {
        if (!(on[a] && on[b])) continue;
        int q[3] = {f[0], f[1], f[2]};
        q[a] = cc[a];
        q[b] = cc[b];
        v = __dadd_rn(v, -A.T[pair_slot(a, b)][kind_ext(m, (1u << a) | (1u << b)).lin(q[0], q[1], q[2])]);
      }
    if (non == 3) v = __dadd_rn(v, A.u_hat[cc[0] + static_cast<i64>(m.nc[0]) * (cc[1] + static_cast<i64>(m.nc[1]) * cc[2])]);
    out[f[0] + nf0 * (f[1] + nf1 * static_cast<i64>(f[2]))] = v;
  }
}

unsigned nblk(i64 n, int bs, int cap = 8 * kNumSms) {
  i64 b = (n + bs - 1) / bs;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b);
}

}  // namespace

void launch_merge3d(const Merge3DArgs& A, double* out, DevState* st, cudaStream_t s) {
  const MeshDev& m = A.m;
  for (int a = 0; a < 3; ++a)
    if (m.nc[a] + 2 > kMaxKnots) throw AsdsmError(kUnsupported, "3D merge supports at most 62 coarse points per axis");
  const int ntr = m.nc[0] * m.nc[1] * m.nc[2];
  m1_kernel<<<(ntr + 127) / 128, 128, 0, s>>>(A, st);
  const int npl = m.nc[0] * m.nc[1] + m.nc[0] * m.nc[2] + m.nc[1] * m.nc[2];
  m2_derivs_kernel<<<(npl + 63) / 64, 64, 0, s>>>(A, st);
  i64 npair = 0;
  for (int p = 0; p < 3; ++p) {
    const int a = p < 2 ? 0 : 1, b = p == 0 ? 1 : 2, f = 3 - a - b;
    npair += static_cast<i64>(m.nc[a]) * m.nc[b] * m.nf[f];
  }
  m2_fill_kernel<<<nblk(npair, 256), 256, 0, s>>>(A, st);
  g_kernel_launches += 3;
  // the three slabs' corrections are independent: one launch per stage covers all of them
  int nl = 0, nl3 = 0;
  i64 ns = 0;
  for (int a = 0; a < 3; ++a) {
    const int f1 = (a == 0) ? 1 : 0, f2 = (a == 2) ? 1 : 2;
    nl = std::max(nl, m.nc[a] * (m.nf[f2] + m.nf[f1] + m.nc[f2]));
    nl3 = std::max(nl3, m.nc[a] * m.nf[f1]);
    ns = std::max(ns, static_cast<i64>(m.nc[a]) * m.nf[f1] * m.nf[f2]);
  }
  const bool per_thread = std::getenv("ASDSM_M3_THREAD_LINES") != nullptr;
  bool warp_ok = !per_thread;
  for (int q = 0; q < 3; ++q) warp_ok = warp_ok && m.nc[q] + 2 <= kWarpKnots;
  if (warp_ok) {
    m3_derivs_warp_kernel<<<dim3((nl + kDerivWarps - 1) / kDerivWarps, 3), 32 * kDerivWarps, 0, s>>>(A, 0, st);
    m3_derivs_warp_kernel<<<dim3((nl3 + kDerivWarps - 1) / kDerivWarps, 3), 32 * kDerivWarps, 0, s>>>(A, 1, st);
  } else {
    m3_derivs_kernel<<<dim3((nl + 31) / 32, 3), 32, 0, s>>>(A, 0, st);
    m3_derivs_kernel<<<dim3((nl3 + 31) / 32, 3), 32, 0, s>>>(A, 1, st);
  }
  if (ns >= (i64{1} << 31)) throw AsdsmError(kUnsupported, "3D merge: slab arrays of 2^31 points or more");
  m3_apply_kernel<<<dim3(nblk(ns, 256, 3 * kNumSms), 3), 256, 0, s>>>(A, st);
  g_kernel_launches += 3;
  const i64 nskel = static_cast<i64>(m.nc[0]) * m.nf[1] * m.nf[2] +
                   static_cast<i64>(m.nf[0] - m.nc[0]) * m.nc[1] * m.nf[2] +
                   static_cast<i64>(m.nf[0] - m.nc[0]) * (m.nf[1] - m.nc[1]) * m.nc[2];
  if (nskel >= (i64{1} << 31)) throw AsdsmError(kUnsupported, "3D merge: 2^31 skeleton points or more");
  m4_kernel<<<nblk(nskel, 256, 32 * kNumSms), 256, 0, s>>>(A, out, st);
  ++g_kernel_launches;
  ASDSM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace asdsm_b200
